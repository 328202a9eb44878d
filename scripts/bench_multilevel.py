"""Full multilevel GOSH on a com-orkut-shaped R-MAT (C3) or the C1 graph, on
one GPU: coarsening ladder + per-level training time (GPU box).

    python scripts/bench_multilevel.py [c3|c1] [epochs]

CPU=1 adds the reference's CPU path timed on this box's host cores (the
oracle's C restatement: sequential coarsen_all = the reference's parity
path, then train_level per level with all host threads).  Levels whose CPU
training would exceed CPU_LEVEL_S seconds are timed on a bounded number of
passes and extrapolated at the measured rate (reported as such).

Mirrors train_multilevel (trainer.py:252-288) step by step so each level can
be timed; prints one JSON line per level and a summary line."""
import json
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import numpy as np  # noqa: E402
import torch  # noqa: E402

import paper_2008_12336_b200 as gb  # noqa: E402

which = sys.argv[1] if len(sys.argv) > 1 else "c3"
epochs = int(sys.argv[2]) if len(sys.argv) > 2 else 1000
if which == "c3":
    scale, samples, dim = 22, 126_000_000, 128
else:
    scale, samples, dim = 14, 262_144, 32
t0 = time.perf_counter()
g = gb.rmat_graph(scale, samples, 7, densify_ids=True)
torch.cuda.synchronize()
t_graph = time.perf_counter() - t0
print(json.dumps({"graph": which, "vertices": g.num_vertices, "arcs": g.num_edges,
                  "undirected_edges": g.num_edges // 2, "build_s": t_graph}), flush=True)
cfg = gb.TrainConfig(dim=dim, total_epochs=epochs, smoothing_ratio=0.3, learning_rate=0.035,
                     negative_samples=3, seed=1,
                     epoch_unit=os.environ.get("UNIT", "edge-scaled"),
                     max_inflight=int(os.environ.get("CAP", "0")))
t0 = time.perf_counter()
h = gb.coarsen_all(g, threshold=100)
torch.cuda.synchronize()
t_coarsen = time.perf_counter() - t0
print(json.dumps({"coarsen_s": t_coarsen, "levels": [x.num_vertices for x in h.graphs],
                  "level_ms": h.level_ms, "rounds": h.rounds, "stalled": h.stalled}),
      flush=True)
plan = gb.epoch_plan(cfg.total_epochs, cfg.smoothing_ratio, h.depth).per_level
M = torch.from_numpy(gb.init_embedding(h.graphs[-1].num_vertices, dim, cfg.seed)).cuda()
total_upd, t_train = 0, 0.0
for i in range(h.depth - 1, -1, -1):
    gi = h.graphs[i]
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    st = gb.train_level(gi, M, cfg, int(plan[i]), rng_stream=i)
    torch.cuda.synchronize()
    dt = time.perf_counter() - t0
    t_train += dt
    total_upd += st.updates
    print(json.dumps({"level": i, "V": gi.num_vertices, "E": gi.num_edges, "epochs": int(plan[i]),
                      "passes": st.passes, "updates": st.updates, "s": dt,
                      "upd_per_s": st.updates / dt if dt else None,
                      "cap": gb.trainer.inflight_cap(cfg, gi.num_vertices)}), flush=True)
    if i > 0:
        M = gb.expand_embedding(M, h.mappings[i - 1])
torch.cuda.synchronize()
print(json.dumps({"summary": which, "embed_s": t_coarsen + t_train, "coarsen_s": t_coarsen,
                  "train_s": t_train, "updates": total_upd,
                  "upd_per_s": total_upd / t_train}), flush=True)

if os.environ.get("CPU") == "1":
    sys.path.insert(0, ROOT)
    from oracle import oracle as orc
    threads = orc.max_threads()
    budget_s = float(os.environ.get("CPU_LEVEL_S", "20"))
    x0, a0 = g.device_csr()
    x0 = x0.cpu().numpy()
    a0 = a0[: g.num_edges].cpu().numpy()
    t0 = time.perf_counter()
    graphs, maps, stalled = orc.coarsen_all(x0, a0, 100)
    cpu_coarsen = time.perf_counter() - t0
    assert [len(x) - 1 for x, _ in graphs] == [x.num_vertices for x in h.graphs]
    cpu_train, cpu_upd = 0.0, 0
    Mc = orc.init_embedding(len(graphs[-1][0]) - 1, dim, cfg.seed)
    for i in range(len(graphs) - 1, -1, -1):
        x, a = graphs[i]
        V, E = len(x) - 1, int(x[-1])
        ppe = orc.passes_per_epoch(V, E, cfg.epoch_unit)
        e_i = int(plan[i])
        non_iso = int((np.diff(x) > 0).sum())
        passes_total = e_i * ppe
        # calibrate: one pass, then as many as fit the level budget
        t0 = time.perf_counter()
        orc.train_pass(x, a, Mc, cfg.learning_rate, 3, cfg.seed, i, 0, nthreads=threads)
        one = max(time.perf_counter() - t0, 1e-6)
        n_run = int(min(passes_total, max(1, budget_s / one)))
        t0 = time.perf_counter()
        for p in range(1, n_run):
            orc.train_pass(x, a, Mc, cfg.learning_rate, 3, cfg.seed, i, p, nthreads=threads)
        el = one + time.perf_counter() - t0
        rate = n_run * non_iso * 4 / el
        upd = passes_total * non_iso * 4
        est = upd / rate
        cpu_train += est
        cpu_upd += upd
        print(json.dumps({"cpu_level": i, "V": V, "passes": passes_total, "passes_timed": n_run,
                          "upd_per_s": rate, "s_est": est, "threads": threads}), flush=True)
        if i > 0:
            Mc = orc.expand(Mc, maps[i - 1][0])
    print(json.dumps({"cpu_summary": which, "threads": threads, "coarsen_s": cpu_coarsen,
                      "train_s_est": cpu_train, "embed_s_est": cpu_coarsen + cpu_train,
                      "updates": cpu_upd, "kind": "port (oracle/gosh_oracle.c)",
                      "gpu_embed_s": t_coarsen + t_train,
                      "speedup_est": (cpu_coarsen + cpu_train) / (t_coarsen + t_train)}),
          flush=True)

