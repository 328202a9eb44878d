"""Seed spread of single-rotation sharded training on the friendster shape
(finest level sharded, 8 ranks, edge-scaled 10 epochs): adaptive vs fixed
per-pair batch, SEEDS training seeds."""
import json
import os
import sys

os.environ.setdefault("PYTORCH_CUDA_ALLOC_CONF", "backend:cudaMallocAsync")
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import torch  # noqa: E402

import paper_2008_12336_b200 as gb  # noqa: E402
from paper_2008_12336_b200.evaluate import LinkPredictionSetup  # noqa: E402

SEEDS = [int(x) for x in os.environ.get("SEEDS", "1,2,3").split(",")]
g = gb.rmat_graph(27, 1_900_000_000, 7, densify_ids=True)
setup = LinkPredictionSetup.build(g, eval_seed=1, evaluator="device", eval_sample=1 << 20)
del g
for seed in SEEDS:
    cfg = gb.TrainConfig(dim=128, total_epochs=10, smoothing_ratio=0.3, learning_rate=0.035,
                         negative_samples=3, seed=seed, epoch_unit="edge-scaled")
    out = {"seed": seed}
    M = setup.embed(cfg)
    out["in_memory"] = setup.score(M)
    del M
    for adapt in (True, False):
        M, _ = gb.train_multilevel_sharded(setup.train_graph, cfg, hierarchy=setup.hierarchy,
                                           num_ranks=8, shard_levels=1, return_device=True,
                                           adapt_batch=adapt)
        out["sharded1_adapt" if adapt else "sharded1_fixed"] = setup.score(M)
        del M
        torch.cuda.empty_cache()
    print(json.dumps(out), flush=True)
