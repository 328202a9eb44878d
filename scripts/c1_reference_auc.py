"""Reference AUCROC on the C1 workload (run in the build container only).

Builds the C1 graph with the repo's R-MAT generator (oracle restatement, bit-
identical to the GPU generator): scale 14, 262,144 samples, seed 7, ids
densified.  Then runs the REFERENCE (mlembed, /root/reference) end to end --
run_link_prediction with the "normal" preset (e=1000, p=0.3, lr=0.035), d=32,
3 negatives, edge-scaled epochs, num_workers=1 (its deterministic mode) --
for training seeds 1..5 at eval_seed 1, and writes
tests/golden/c1_reference_auc.json.  The GPU side repeats the same protocol
in scripts/c1_gpu_auc.py.
"""
import json
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, "/root/reference/pkg/src")
os.environ.setdefault("NUMBA_CACHE_DIR", "/tmp/numba_cache")

import numpy as np  # noqa: E402
import mlembed as ml  # noqa: E402
from oracle import oracle as orc  # noqa: E402

x, a = orc.rmat_graph(14, 262144, 7, densify_ids=True)
g = ml.Graph(num_vertices=len(x) - 1, num_edges=int(x[-1]), xadj=x, adj=a)
out = {"graph": {"scale": 14, "samples": 262144, "seed": 7, "densified": True,
                 "vertices": g.num_vertices, "arcs": g.num_edges},
       "protocol": {"preset": "normal", "total_epochs": 1000, "smoothing_ratio": 0.3,
                    "learning_rate": 0.035, "dim": 32, "negative_samples": 3,
                    "epoch_unit": "edge-scaled", "eval_seed": 1, "num_workers": 1},
       "runs": []}
# usage: c1_reference_auc.py [--out PATH] [seed ...]; several processes may
# run disjoint seed sets into separate files, merged by --merge
args = sys.argv[1:]
out_path = os.path.join(ROOT, "tests", "golden", "c1_reference_auc.json")
if args[:1] == ["--merge"]:
    runs = []
    for p in args[1:]:
        with open(p) as f:
            runs += json.load(f)["runs"]
    out["runs"] = sorted({r["seed"]: r for r in runs}.values(), key=lambda r: r["seed"])
    args = []
    seeds = []
elif args[:1] == ["--out"]:
    out_path, args = args[1], args[2:]
    seeds = [int(s) for s in args] or [1, 2, 3, 4, 5]
else:
    seeds = [int(s) for s in args] or [1, 2, 3, 4, 5]
for seed in seeds:
    cfg = ml.TrainConfig(dim=32, total_epochs=1000, smoothing_ratio=0.3, learning_rate=0.035,
                         negative_samples=3, seed=seed, num_workers=1,
                         epoch_unit="edge-scaled")
    t0 = time.perf_counter()
    rep = ml.run_link_prediction(g, cfg, eval_seed=1)
    out["runs"].append({"seed": seed, "aucroc": rep.aucroc, "times": rep.times,
                        "counts": rep.counts})
    print(seed, rep.aucroc, rep.times, flush=True)
aucs = [r["aucroc"] for r in out["runs"]]
out["mean"] = float(np.mean(aucs))
out["std"] = float(np.std(aucs))
with open(out_path, "w") as f:
    json.dump(out, f, indent=1)
print("mean", out["mean"], "std", out["std"])
