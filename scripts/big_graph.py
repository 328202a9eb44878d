"""Large synthetic graphs on ONE B200: build (R-MAT -> CSR -> densify),
coarsen, full multilevel training, and the single-level pass on the finest
level measured against the HBM roofline.  Prints JSON lines with timings and
peak device memory per phase.

    SCALE=26 SAMPLES=2000000000 python scripts/big_graph.py      # C4 shape
    SCALE=24 SAMPLES=500000000  python scripts/big_graph.py      # 1/4 C4

C4 in BASELINE.json is friendster-shaped (65.6M vertices, 1.8B undirected
edges, d=128) on 8 GPUs; this is the same shape on one GPU (the matrix,
33.6 GB, and the CSR, ~15 GB, fit in 180 GB of HBM).
"""
import json
import os
import sys
import time

# Transient workspaces here are tens of GiB; with torch's default caching
# allocator a long-lived tensor placed inside a freed workspace segment pins
# it (112 GiB reserved-but-unusable at scale 27).  The driver's stream-ordered
# pool has no such fragmentation and allocates as fast.
os.environ.setdefault("PYTORCH_CUDA_ALLOC_CONF", "backend:cudaMallocAsync")

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import numpy as np  # noqa: E402
import torch  # noqa: E402

import paper_2008_12336_b200 as gb  # noqa: E402
from paper_2008_12336_b200 import _lib  # noqa: E402

scale = int(os.environ.get("SCALE", "24"))
samples = int(os.environ.get("SAMPLES", str(500_000_000)))
dim = int(os.environ.get("DIM", "128"))
epochs = int(os.environ.get("EPOCHS", "200"))  # epochs_large (cli.py:62) for V >= 10M
unit = os.environ.get("UNIT", "vertex-pass")
passes_bench = int(os.environ.get("BENCH_PASSES", "10"))


def mem():
    return round(torch.cuda.max_memory_allocated() / 2**30, 2)


def out(**kw):
    kw["peak_gib"] = mem()
    print(json.dumps(kw), flush=True)


torch.cuda.set_device(0)
if os.environ.get("RESERVE", "0") == "1":  # map HBM once (memory.py; opt-in)
    out(phase="reserve", **gb.reserve_device_memory(fraction=0.92))
t0 = time.perf_counter()
g = gb.rmat_graph(scale, samples, 7, densify_ids=True)
torch.cuda.synchronize()
out(phase="build", scale=scale, samples=samples, vertices=g.num_vertices, arcs=g.num_edges,
    undirected_edges=g.num_edges // 2, s=time.perf_counter() - t0)
torch.cuda.empty_cache()

t0 = time.perf_counter()
h = gb.coarsen_all(g, threshold=100)
torch.cuda.synchronize()
out(phase="coarsen", levels=[x.num_vertices for x in h.graphs],
    arcs=[x.num_edges for x in h.graphs], level_ms=h.level_ms, stalled=h.stalled,
    s=time.perf_counter() - t0)
torch.cuda.empty_cache()

# single-level pass on the finest level: roofline fraction at this size
xadj, adj = g.device_csr()
sources, non_iso = g.active_sources()
V = g.num_vertices
M = torch.empty((V, dim), dtype=torch.float32, device="cuda")
M.uniform_(-0.5 / dim, 0.5 / dim, generator=torch.Generator(device="cuda").manual_seed(1))
lrs = torch.tensor([0.035], dtype=torch.float32, device="cuda")
status = _lib.new_status()
cap = gb.trainer.inflight_cap(gb.TrainConfig(dim=dim), V)
flags = _lib.GB_TRAIN_FAST_SIGMOID | _lib.GB_TRAIN_ATOMIC
st = torch.cuda.current_stream()


def launch(p):
    _lib.call("gb_train_passes", V, _lib.ptr(xadj), _lib.ptr(adj), _lib.ptr(sources), non_iso,
              _lib.ptr(M), dim, 3, 1, 0, p, 1, 1 << 40, _lib.ptr(lrs), flags, cap,
              _lib.ptr(status), st.cuda_stream)


for p in range(3):
    launch(p)
torch.cuda.synchronize()
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
e0.record(st)
for p in range(passes_bench):
    launch(3 + p)
e1.record(st)
torch.cuda.synchronize()
ms = e0.elapsed_time(e1) / passes_bench
bps = 8 * dim * 5 + 12
peak = json.load(open(os.path.join(ROOT, "MEASURED_PEAKS.json")))["hbm_gbs"] if os.path.exists(
    os.path.join(ROOT, "MEASURED_PEAKS.json")) else 6650.0
achieved = non_iso * bps / (ms / 1e3) / 1e9
out(phase="pass", non_isolated=non_iso, ms_per_pass=ms, upd_per_s=non_iso * 4 / (ms / 1e3),
    achieved_gbs=achieved, peak_gbs=peak, frac=achieved / peak, bytes_per_source=bps)
del M
torch.cuda.empty_cache()

# full multilevel embedding (train_multilevel's loop, timed per level)
cfg = gb.TrainConfig(dim=dim, total_epochs=epochs, smoothing_ratio=0.3, learning_rate=0.035,
                     negative_samples=3, seed=1, epoch_unit=unit)
plan = gb.epoch_plan(cfg.total_epochs, cfg.smoothing_ratio, h.depth).per_level
Mh = torch.from_numpy(gb.init_embedding(h.graphs[-1].num_vertices, dim, cfg.seed)).cuda()
t_all = time.perf_counter()
for i in range(h.depth - 1, -1, -1):
    t0 = time.perf_counter()
    s_ = gb.train_level(h.graphs[i], Mh, cfg, int(plan[i]), rng_stream=i)
    torch.cuda.synchronize()
    dt = time.perf_counter() - t0
    out(phase="level", level=i, V=h.graphs[i].num_vertices, epochs=int(plan[i]),
        passes=s_.passes, updates=s_.updates, s=dt, upd_per_s=s_.updates / dt if dt else None)
    if i > 0:
        Mh = gb.expand_embedding(Mh, h.mappings[i - 1])
torch.cuda.synchronize()
out(phase="train_multilevel", s=time.perf_counter() - t_all, unit=unit, epochs=epochs)
