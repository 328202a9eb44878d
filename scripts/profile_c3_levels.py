"""One training launch on a level of the C3 hierarchy (for ncu): the level's
graph from the device coarsening of the C3 shape, d=128, the default kernel
selection (uncapped), 1 edge-scaled epoch = one launch of ceil(E/V) passes.
LEVEL picks the level (C3: 0..4).  Run under
  ncu --set full -k regex:train_passes -c 1 ... python scripts/profile_c3_levels.py"""
import json
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import torch  # noqa: E402

import paper_2008_12336_b200 as gb  # noqa: E402

LEVEL = int(os.environ.get("LEVEL", "4"))
EPOCHS = int(os.environ.get("EPOCHS", "1"))
g = gb.rmat_graph(22, 126_000_000, 7, densify_ids=True)
h = gb.coarsen_all(g, threshold=100)
gl = h.graphs[LEVEL]
cfg = gb.TrainConfig(dim=128, negative_samples=3, seed=1, epoch_unit="edge-scaled")
M = torch.from_numpy(gb.init_embedding(gl.num_vertices, 128, 1)).cuda()
torch.cuda.synchronize()
t0 = time.perf_counter()
if EPOCHS > 1:  # warm-up launch
    gb.train_level(gl, M, cfg, 1, rng_stream=LEVEL)
    torch.cuda.synchronize()
    t0 = time.perf_counter()
st = gb.train_level(gl, M, cfg, EPOCHS, rng_stream=LEVEL)
torch.cuda.synchronize()
dt = time.perf_counter() - t0
print(json.dumps({"level": LEVEL, "epochs": EPOCHS, "GB_PIPE": os.environ.get("GB_PIPE"), "V": gl.num_vertices, "arcs": gl.num_edges,
                  "passes": st.passes, "updates": st.updates, "s": dt,
                  "upd_per_s": st.updates / dt}))
