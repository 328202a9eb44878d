"""Where the C4-shape link-prediction setup time goes (measurement tool):
LinkPredictionSetup.build's split / coarsen / evaluation-pair phases, plus
the numpy draw of the withheld edges inside the split."""
import json
import os
import sys
import time

# large cached blocks never split (the native allocator otherwise fragments
# at this scale; DESIGN 5b)
os.environ.setdefault("PYTORCH_CUDA_ALLOC_CONF", "max_split_size_mb:1024")
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import numpy as np  # noqa: E402
import torch  # noqa: E402

import paper_2008_12336_b200 as gb  # noqa: E402
from paper_2008_12336_b200.evaluate import LinkPredictionSetup  # noqa: E402

g = gb.rmat_graph(int(os.environ.get("SCALE", "27")), int(os.environ.get("SAMPLES", "1900000000")),
                  7, densify_ids=True)
torch.cuda.synchronize()
m = g.num_edges // 2
t0 = time.perf_counter()
np.random.default_rng(1).choice(m, size=int(round(0.2 * m)), replace=False)
t_choice = time.perf_counter() - t0
t0 = time.perf_counter()
setup = LinkPredictionSetup.build(g, eval_seed=1, evaluator="device", eval_sample=1 << 20)
torch.cuda.synchronize()
print(json.dumps({"vertices": g.num_vertices, "edges": m, "numpy_choice_s": t_choice,
                  "setup_s": time.perf_counter() - t0, "phases_s": setup.times}), flush=True)
