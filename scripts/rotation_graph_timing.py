"""Phase timing of the CUDA-graph tournament rotations (GB_TRACE_ROTATIONS):
eager rotation 0, capture + instantiate, replays, graph destruction, against
the eager path, on the C2 graph with K = 2 * VR parts."""
import json
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
os.environ["GB_TRACE_ROTATIONS"] = "1"
import torch  # noqa: E402

import paper_2008_12336_b200 as gb  # noqa: E402
from paper_2008_12336_b200 import tournament as tn  # noqa: E402

VR = int(os.environ.get("VR", "8"))
R = int(os.environ.get("R", "8"))
g = gb.rmat_graph(20, 1 << 24, 7)
cfg = gb.TrainConfig(dim=128, negative_samples=3, seed=1, learning_rate=0.035)
M = torch.from_numpy(gb.init_embedding(g.num_vertices, 128, 1)).cuda()
for mode in ("1", "0", "1", "0"):
    os.environ["GB_ROTATION_GRAPH"] = mode
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    st = tn.train_tournament(g, M, cfg, R * 5 * 2 * VR, gather=False, num_ranks=VR)
    torch.cuda.synchronize()
    print(json.dumps({"graph": mode, "K": 2 * VR, "rotations": st["rotations"],
                      "wall_s": time.perf_counter() - t0, "train_s": st["train_s"],
                      "phases_s": st.get("phases_s")}), flush=True)
