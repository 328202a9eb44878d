"""The C5 configuration end to end on ONE B200 (BASELINE.json configs[4]: R-MAT
2^28 ids, ~4.2B undirected edges, d=256): row-block CSR build, row-block
coarsening ladder, then train_multilevel at d=256 with the CLI's
large-graph defaults (200 epochs, vertex-pass) -- coarse levels released as
the ladder descends, so the finest matrix (121M x 256 floats = 116 GB) and
its CSR (34 GB) share the 180 GB of HBM.  The matrix stays on the device
(return_device).  Prints JSON lines per phase with peak device memory."""
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
DIM = int(os.environ.get("DIM", "256"))
EPOCHS = int(os.environ.get("EPOCHS", "200"))


def gib():
    return round(torch.cuda.max_memory_allocated() / 2**30, 2)


def main():
    if os.environ.get("RESERVE", "0") == "1":  # map HBM once (memory.py; opt-in)
        print(json.dumps({"phase": "reserve", **gb.reserve_device_memory(fraction=0.92)}),
              flush=True)
    t0 = time.perf_counter()
    g = gb.rmat_graph(SCALE, SAMPLES, 7, densify_ids=True, max_block_keys=BLOCK)
    torch.cuda.synchronize()
    t_build = time.perf_counter() - t0
    t0 = time.perf_counter()
    h = gb.coarsen_all(g, threshold=100, max_block_keys=BLOCK)
    torch.cuda.synchronize()
    t_coarsen = time.perf_counter() - t0
    levels = [x.num_vertices for x in h.graphs]
    print(json.dumps({"phase": "graph", "vertices": g.num_vertices, "arcs": g.num_edges,
                      "build_s": t_build, "coarsen_s": t_coarsen, "levels": levels,
                      "peak_gib": gib()}), flush=True)
    cfg = gb.TrainConfig(dim=DIM, total_epochs=EPOCHS, smoothing_ratio=0.3, learning_rate=0.035,
                         negative_samples=3, seed=1, epoch_unit="vertex-pass")
    plan = gb.epoch_plan(EPOCHS, 0.3, h.depth).per_level
    updates = sum(int(plan[i]) * int(x.active_sources()[1]) * 4 for i, x in enumerate(h.graphs))
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    M = gb.train_multilevel(g, cfg, hierarchy=h, return_device=True, release_levels=True)
    torch.cuda.synchronize()
    embed_s = time.perf_counter() - t0
    status = _lib.new_status()
    _lib.call("gb_nonfinite_scan", _lib.ptr(M), M.numel(), 0, _lib.ptr(status), _lib.stream())
    print(json.dumps({"phase": "train_multilevel", "dim": DIM, "epochs": EPOCHS,
                      "plan": [int(x) for x in plan], "updates": updates, "embed_s": embed_s,
                      "upd_per_s": updates / embed_s,
                      "matrix_gib": round(M.numel() * 4 / 2**30, 1),
                      "nonfinite_flag": int(status[0].item()), "peak_gib": gib()}), flush=True)


if __name__ == "__main__":
    main()
