"""Embed wall time and AUCROC of the GPU path in several modes on one graph,
with the device evaluator (seeded eval subsample identical for all modes).

Modes (MODES env, comma list):
  det        deterministic kernels: bit-equal to the reference at
             num_workers=1, i.e. the reference's own AUCROC
  cap<N>     Hogwild with max_inflight=N (cap0 = auto policy)
  tour<R>    finest level by the part-pair tournament over R virtual ranks
  large<K>   finest level by train_large (the reference's partitioned
             trainer, bigtrain.py:343-493) with a budget giving K parts --
             the single-device form of the algorithm the tournament shards
  a suffix "b" (tour8b, large16b) uses balanced pools (TrainConfig.balanced_pools)
  a suffix "s" (cap0s, tour2s) writes sample rows back with plain stores
  (atomic_rows=False); the default is vector-reduction write-back

    GRAPH=c1|c3 MODES=det,cap0 SEEDS=1 UNIT=vertex-pass EPOCHS=1000 \\
        EVAL_SAMPLE=1000000 python scripts/auc_modes.py
"""
import json
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import numpy as np  # noqa: E402
import torch  # noqa: E402

import paper_2008_12336_b200 as gb  # noqa: E402
from paper_2008_12336_b200 import evaluate as ev  # noqa: E402

graph = os.environ.get("GRAPH", "c1")
if graph == "c1":
    g = gb.rmat_graph(14, 262144, 7, densify_ids=True)
    dim = 32
else:
    g = gb.rmat_graph(22, 126_000_000, 7, densify_ids=True)
    dim = 128
dim = int(os.environ.get("DIM", dim))
modes = os.environ.get("MODES", "det,cap0").split(",")
seeds = [int(x) for x in os.environ.get("SEEDS", "1").split(",")]
unit = os.environ.get("UNIT", "edge-scaled")
epochs = int(os.environ.get("EPOCHS", "1000"))
cap_sample = os.environ.get("EVAL_SAMPLE")
cap_sample = int(cap_sample) if cap_sample else None
eval_seed = 1

t0 = time.perf_counter()
split = gb.split_train_test(g, 0.2, eval_seed)
tg = split.train_graph
h = gb.coarsen_all(tg, threshold=100)
torch.cuda.synchronize()
prep_s = time.perf_counter() - t0
pos_train = ev._subsample(tg.undirected_pairs(), cap_sample, eval_seed + 3)
neg_train = gb.sample_negative_edges(tg, pos_train.shape[0], seed=eval_seed + 1)
pos_test = ev._subsample(split.test_edges, cap_sample, eval_seed + 4)
neg_test = gb.sample_negative_edges(tg, pos_test.shape[0], seed=eval_seed + 2,
                                    exclude_pairs=split.test_edges)
print(json.dumps({"graph": graph, "vertices": g.num_vertices, "arcs": g.num_edges,
                  "train_levels": [x.num_vertices for x in h.graphs], "prep_s": prep_s,
                  "eval_train_pairs": 2 * int(pos_train.shape[0]),
                  "eval_test_pairs": 2 * int(pos_test.shape[0]), "unit": unit,
                  "epochs": epochs, "dim": dim}), flush=True)
def train_multilevel_large_finest(cfg, K):
    """train_multilevel (trainer.py:252-288) with the finest level trained by
    train_large under a budget that yields K parts (coarser levels in memory,
    like train_multilevel_sharded's default shard_levels=1)."""
    from paper_2008_12336_b200 import trainer as tr
    plan = tr.epoch_plan(cfg.total_epochs, cfg.smoothing_ratio, h.depth).per_level
    M = torch.from_numpy(gb.init_embedding(h.graphs[-1].num_vertices, cfg.dim,
                                           cfg.seed)).cuda()
    for i in range(h.depth - 1, -1, -1):
        g_i, e_i = h.graphs[i], int(plan[i])
        if e_i > 0:
            if i == 0:
                bud = gb.MemoryBudget(1)
                row = bud.parts_resident * cfg.dim * 4 + bud.pools_resident * 2 * bud.batch_size * 4
                bud = gb.MemoryBudget(-(-g_i.num_vertices // K) * row)
                gb.train_large(g_i, M, cfg, e_i, bud, rng_stream=i)
            else:
                gb.train_level(g_i, M, cfg, e_i, rng_stream=i)
        if i > 0:
            M = gb.expand_embedding(M, h.mappings[i - 1])
    return M


for mode_s in modes:
    balanced = mode_s.endswith("b")  # tour<R>b / large<K>b: balanced pools
    mode = mode_s[:-1] if balanced else mode_s
    atomic = not mode.endswith("s")
    mode = mode if atomic else mode[:-1]
    for seed in seeds:
        cfg = gb.TrainConfig(dim=dim, total_epochs=epochs, smoothing_ratio=0.3,
                             learning_rate=0.035, negative_samples=3, seed=seed,
                             epoch_unit=unit, deterministic=mode == "det",
                             max_inflight=int(mode[3:]) if mode.startswith("cap") else 0,
                             atomic_rows=atomic, balanced_pools=balanced)
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        if mode.startswith("tour"):
            M, _ = gb.train_multilevel_sharded(tg, cfg, hierarchy=h, num_ranks=int(mode[4:]),
                                               return_device=True)
        elif mode.startswith("large"):
            M = train_multilevel_large_finest(cfg, int(mode[5:]))
        else:
            M = gb.train_multilevel(tg, cfg, hierarchy=h, return_device=True)
        torch.cuda.synchronize()
        embed_s = time.perf_counter() - t0
        t0 = time.perf_counter()
        f_train = gb.hadamard_features_device(M, *ev._balanced(pos_train, neg_train))
        f_test = gb.hadamard_features_device(M, *ev._balanced(pos_test, neg_test))
        model = gb.train_logreg_device(f_train, gb.LogRegConfig(seed=eval_seed))
        auc = gb.auc_roc_device(gb.predict_scores_device(model, f_test.rows), f_test.labels)
        eval_s = time.perf_counter() - t0
        print(json.dumps({"mode": mode_s, "seed": seed, "aucroc": auc, "embed_s": embed_s,
                          "eval_s": eval_s}), flush=True)
        del M, f_train, f_test
        torch.cuda.empty_cache()
