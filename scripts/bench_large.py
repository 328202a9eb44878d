"""Partitioned trainer with host staging (train_large, bigtrain.py:343-493)
on one B200: the embedding matrix lives in pinned host memory, a
MemoryBudget forces K parts with P resident device slots, parts are switched
by async copies.  Reports updates/s, switches and staged bytes, next to the
oracle's pool/pair kernels timed on a sample of the same pairs on the host
cores (the reference's CPU path).

    SCALE=24 SAMPLES=250000000 DIM=256 BUDGET_GB=3 python scripts/bench_large.py
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

scale = int(os.environ.get("SCALE", "22"))
samples = int(os.environ.get("SAMPLES", str(60_000_000)))
dim = int(os.environ.get("DIM", "256"))
budget_gb = float(os.environ.get("BUDGET_GB", "1.0"))
cpu_s = float(os.environ.get("CPU_SECONDS", "15"))

g = gb.rmat_graph(scale, samples, 7, densify_ids=True)
V = g.num_vertices
budget = gb.MemoryBudget(resident_bytes=int(budget_gb * 2**30), parts_resident=3,
                         pools_resident=4, batch_size=5)
plan = gb.plan_partitions(V, dim, budget)
cfg = gb.TrainConfig(dim=dim, negative_samples=3, seed=1, learning_rate=0.035)
e_i = plan.K * budget.batch_size  # one rotation: round(e_i / (B*K)) = 1
M = gb.init_embedding(V, dim, 1)
print(json.dumps({"vertices": V, "arcs": g.num_edges, "dim": dim, "K": plan.K,
                  "part_rows": plan.max_rows, "matrix_gib": M.nbytes / 2**30,
                  "budget_gib": budget_gb}), flush=True)
walls, loops = [], []
for rep in range(2):  # the first call also pays CUDA/stream warm-up
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    st = gb.train_large(g, M, cfg, e_i, budget)
    torch.cuda.synchronize()
    walls.append(time.perf_counter() - t0)
    loops.append(st["train_s"])  # rotation loop only (no page-locking of M)
wall = min(walls)
upd = st["pos_updates"] + st["neg_updates"]
part_bytes = plan.max_rows * dim * 4
staged = (st["switches"] * 2 + budget.parts_resident) * part_bytes
line = {"train_large_s": wall, "walls": walls, "loop_s": loops, "updates": upd,
        "upd_per_s": upd / wall, "loop_upd_per_s": upd / min(loops), "switches": st["switches"],
        "rotations": st["rotations"], "staged_bytes_upper": staged,
        "staging_gbs": staged / wall / 1e9, "pairs": plan.K * (plan.K + 1) // 2}

# CPU beside it: the oracle's fill_pool_side + train_pool_side on the first
# pairs of the same schedule, all host threads, bounded sample
from oracle import oracle as orc  # noqa: E402
x, a = g.device_csr()
x = x.cpu().numpy()
a = a[: g.num_edges].cpu().numpy()
threads = orc.max_threads()
Mc = gb.init_embedding(V, dim, 1)
cpu_upd, t0 = 0, time.perf_counter()
for pos, (pa, pb) in enumerate(gb.rotation_pairs(plan.K)):
    la, ha = plan.part_range(pa)
    lb, hb = plan.part_range(pb)
    seed = gb.bigtrain._derived_seed(cfg.seed, 0, pos)
    A = Mc[la:ha]
    tj = orc.fill_pool_side(x, a, la, ha, lb, hb, 5, seed, 0)
    Bm = A if pa == pb else Mc[lb:hb]
    cpu_upd += 4 * orc.train_pool_side(A, Bm, tj, lb, hb - lb, 3, 0.035, seed, 2,
                                       nthreads=threads)
    if pa != pb:
        tk = orc.fill_pool_side(x, a, lb, hb, la, ha, 5, seed, 1)
        cpu_upd += 4 * orc.train_pool_side(Bm, A, tk, la, ha - la, 3, 0.035, seed, 3,
                                           nthreads=threads)
    if time.perf_counter() - t0 > cpu_s:
        break
cpu_el = time.perf_counter() - t0
line["cpu_baseline"] = {"upd_per_s": cpu_upd / cpu_el, "threads": threads,
                        "pairs_timed": pos + 1, "kind": "port (oracle/gosh_oracle.c)"}
print(json.dumps(line), flush=True)
