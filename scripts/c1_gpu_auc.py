"""GPU AUCROC on the C1 workload, same protocol as scripts/c1_reference_auc.py
(normal preset, d=32, edge-scaled, eval_seed 1, training seeds 1..5), for a
list of in-flight caps (CAPS env; 0 = auto policy).  Prints JSON lines."""
import json
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import numpy as np  # noqa: E402

import paper_2008_12336_b200 as gb  # noqa: E402

g = gb.rmat_graph(14, 262144, 7, densify_ids=True)
caps = [int(x) for x in os.environ.get("CAPS", "0").split(",")]
seeds = [int(x) for x in os.environ.get("SEEDS", "1,2,3,4,5").split(",")]
det = os.environ.get("DETERMINISTIC", "0") == "1"
for cap in caps:
    aucs, embed = [], []
    for seed in seeds:
        cfg = gb.TrainConfig(dim=32, total_epochs=1000, smoothing_ratio=0.3, learning_rate=0.035,
                             negative_samples=3, seed=seed, epoch_unit="edge-scaled",
                             max_inflight=cap, deterministic=det)
        rep = gb.run_link_prediction(g, cfg, eval_seed=1)
        aucs.append(rep.aucroc)
        embed.append(rep.times["embed_s"])
    print(json.dumps({"cap": cap, "deterministic": det, "aucs": aucs,
                      "mean": float(np.mean(aucs)), "std": float(np.std(aucs)),
                      "embed_s": embed, "vertices": g.num_vertices, "arcs": g.num_edges}),
          flush=True)
