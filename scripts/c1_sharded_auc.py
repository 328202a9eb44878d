"""C1 AUCROC of the sharded (multi-GPU) path against the reference's own
seeds (tests/golden/c1_reference_auc.json: normal preset, edge-scaled, d=32,
the reference at num_workers=1): train_multilevel_sharded with RANKS virtual
ranks (default 4 = K=8 parts; balanced pools, 2 sharded levels, adaptive
batch), paired by training seed; also the in-memory default path."""
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import numpy as np  # noqa: E402

import paper_2008_12336_b200 as gb  # noqa: E402
from paper_2008_12336_b200.evaluate import LinkPredictionSetup, aucroc_parity_interval  # noqa: E402

RANKS = [int(x) for x in os.environ.get("RANKS", "4").split(",")]
SHARD = int(os.environ.get("SHARD", "2"))
N = int(os.environ.get("NSEEDS", "30"))
with open(os.path.join(ROOT, "tests", "golden", "c1_reference_auc.json")) as f:
    ref = json.load(f)
gp, pr = ref["graph"], ref["protocol"]
g = gb.rmat_graph(gp["scale"], gp["samples"], gp["seed"], densify_ids=gp["densified"])
setup = LinkPredictionSetup.build(g, eval_seed=pr["eval_seed"], evaluator="device")
runs = {r["seed"]: r["aucroc"] for r in ref["runs"]}
seeds = sorted(runs)[:N]
for R in [0] + RANKS:
    mine = []
    for seed in seeds:
        cfg = gb.TrainConfig(dim=pr["dim"], total_epochs=pr["total_epochs"],
                             smoothing_ratio=pr["smoothing_ratio"],
                             learning_rate=pr["learning_rate"],
                             negative_samples=pr["negative_samples"], seed=seed,
                             epoch_unit=pr["epoch_unit"])
        if R == 0:
            M = setup.embed(cfg)
        else:
            M, _ = gb.train_multilevel_sharded(setup.train_graph, cfg, hierarchy=setup.hierarchy,
                                               num_ranks=R, return_device=True,
                                               shard_levels=SHARD)
        mine.append(setup.score(M))
    d = np.array(mine) - np.array([runs[s] for s in seeds])
    print(json.dumps({"ranks": R, "mode": "in-memory" if R == 0 else f"sharded ({SHARD} levels)",
                      "n": len(seeds), "mean": float(np.mean(mine)),
                      "ref_mean": float(np.mean([runs[s] for s in seeds])),
                      "paired": aucroc_parity_interval(d)}), flush=True)
