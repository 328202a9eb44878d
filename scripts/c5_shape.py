"""The C5 graph on ONE B200 (BASELINE.json configs[4]: R-MAT 2^28 ids, ~4B
undirected edges): the row-block CSR build (samples regenerated per block,
bounded key scratch), id densification, the row-block coarsening ladder, and
a d=128 training pass over the finest level at the HBM roofline.  C5's own
d=256 matrix (256 GiB) needs the 8-GPU tournament or host-staged parts; the
graph side, which is what no single GPU could build one-shot (~190 GB of sort
keys), runs here.  Prints JSON lines per phase with the peak device memory.
"""
import json
import os
import sys
import time

# native caching allocator with large blocks never split: fresh tens-of-GiB
# allocations get their own segments (no fragmentation for the 116 GB matrix,
# no on-the-spot pool mapping as under cudaMallocAsync; DESIGN 5b)
os.environ.setdefault("PYTORCH_CUDA_ALLOC_CONF", "max_split_size_mb:1024")
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import torch  # noqa: E402

import paper_2008_12336_b200 as gb  # noqa: E402
from paper_2008_12336_b200 import _lib  # noqa: E402

SCALE = int(os.environ.get("SCALE", "28"))
SAMPLES = int(os.environ.get("SAMPLES", str(4_300_000_000)))
BLOCK = int(os.environ.get("BLOCK_KEYS", str(1 << 30)))
DIM = int(os.environ.get("DIM", "128"))
PASSES = int(os.environ.get("PASSES", "3"))


def gib():
    return round(torch.cuda.max_memory_allocated() / 2**30, 2)


def main():
    if os.environ.get("RESERVE", "0") == "1":  # map HBM once (memory.py; opt-in)
        print(json.dumps({"phase": "reserve", **gb.reserve_device_memory(fraction=0.92)}),
              flush=True)
    t0 = time.perf_counter()
    g = gb.rmat_graph(SCALE, SAMPLES, 7, densify_ids=True, max_block_keys=BLOCK)
    torch.cuda.synchronize()
    print(json.dumps({"phase": "build", "scale": SCALE, "samples": SAMPLES,
                      "max_block_keys": BLOCK, "vertices": g.num_vertices, "arcs": g.num_edges,
                      "undirected_edges": g.num_edges // 2, "s": time.perf_counter() - t0,
                      "peak_gib": gib()}), flush=True)
    t0 = time.perf_counter()
    h = gb.coarsen_all(g, threshold=100, max_block_keys=BLOCK)
    torch.cuda.synchronize()
    print(json.dumps({"phase": "coarsen", "levels": [x.num_vertices for x in h.graphs],
                      "arcs": [x.num_edges for x in h.graphs], "stalled": bool(h.stalled),
                      "s": time.perf_counter() - t0, "peak_gib": gib()}), flush=True)
    del h  # keep only the finest level on the device
    import gc
    gc.collect()
    torch.cuda.empty_cache()
    xadj, adj = g.device_csr()
    sources, n_src = g.active_sources()
    M = torch.rand((g.num_vertices, DIM), device="cuda")
    M.sub_(0.5).div_(DIM)  # in place: at d=256 the matrix is 116 GB
    lrs = torch.full((1,), 0.035, dtype=torch.float32, device="cuda")
    status = _lib.new_status()
    flags = _lib.GB_TRAIN_FAST_SIGMOID | _lib.GB_TRAIN_ATOMIC

    def launch(p):
        _lib.call("gb_train_passes", g.num_vertices, _lib.ptr(xadj), _lib.ptr(adj),
                  _lib.ptr(sources), n_src, _lib.ptr(M), DIM, 3, 1, 0, p, 1, 1 << 40,
                  _lib.ptr(lrs), flags, 0, _lib.ptr(status), _lib.stream())

    def nonfinite():
        # the kernels' sticky flag + one scan of M (gb_nonfinite_scan): no
        # matrix-sized temporaries
        _lib.call("gb_nonfinite_scan", _lib.ptr(M), M.numel(), 0, _lib.ptr(status),
                  _lib.stream())
        return int(status[0].item())

    launch(0)
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for p in range(1, PASSES + 1):
        launch(p)
    e1.record()
    torch.cuda.synchronize()
    ms = e0.elapsed_time(e1) / PASSES
    bps = 8 * DIM * (2 + 3) + 12
    peak = float(json.load(open(os.path.join(ROOT, "MEASURED_PEAKS.json")))["hbm_gbs"]) \
        if os.path.exists(os.path.join(ROOT, "MEASURED_PEAKS.json")) else 6650.0
    print(json.dumps({"phase": "pass", "dim": DIM, "non_isolated": n_src, "ms_per_pass": ms,
                      "upd_per_s": n_src * 4 / (ms / 1000.0),
                      "achieved_gbs": n_src * bps / (ms / 1000.0) / 1e9, "peak_gbs": peak,
                      "frac": n_src * bps / (ms / 1000.0) / 1e9 / peak,
                      "matrix_gib": round(M.numel() * 4 / 2**30, 1),
                      "nonfinite_flag": nonfinite(), "peak_gib": gib()}), flush=True)


if __name__ == "__main__":
    main()
