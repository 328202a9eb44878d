"""Where coarsening time goes on a large R-MAT (measurement tool): build the
graph, then time coarsen_all's phases per level with CUDA-synchronised wall
clocks (order, collapse, coarse CSR).  SCALE / SAMPLES as in big_graph.py; BLOCK
= max_block_keys for the row-block builds (C5: SCALE=28 SAMPLES=4300000000
BLOCK=1073741824)."""
import json
import os
import sys
import time

os.environ.setdefault("PYTORCH_CUDA_ALLOC_CONF", "backend:cudaMallocAsync")
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import torch  # noqa: E402

import paper_2008_12336_b200 as gb  # noqa: E402
from paper_2008_12336_b200 import coarsen as cz  # noqa: E402

scale = int(os.environ.get("SCALE", "26"))
samples = int(os.environ.get("SAMPLES", "1000000000"))
block = int(os.environ["BLOCK"]) if os.environ.get("BLOCK") else None  # max_block_keys (C5)

def mempool_release_threshold(set_max=False):
    """The default CUDA mempool's release threshold (torch's cudaMallocAsync
    backend allocates from it): 0 returns freed memory to the OS at every
    synchronisation, so the next large allocation maps it again."""
    import ctypes
    torch.cuda.init()
    lib = ctypes.CDLL("libcudart.so.12")
    pool = ctypes.c_void_p()
    assert lib.cudaDeviceGetDefaultMemPool(ctypes.byref(pool), torch.cuda.current_device()) == 0
    val = ctypes.c_uint64()
    if set_max:
        val.value = 2**64 - 1
        assert lib.cudaMemPoolSetAttribute(pool, 4, ctypes.byref(val)) == 0
    assert lib.cudaMemPoolGetAttribute(pool, 4, ctypes.byref(val)) == 0
    return val.value


print(json.dumps({"release_threshold": mempool_release_threshold(bool(os.environ.get("RELEASE")))}),
      flush=True)
if os.environ.get("WARM_GIB"):  # map the pool once up front (kept with RELEASE=1)
    t_w = time.perf_counter()
    warm = torch.empty(int(float(os.environ["WARM_GIB"]) * 2**30), dtype=torch.uint8, device="cuda")
    del warm
    torch.cuda.synchronize()
    print(json.dumps({"warm_gib": float(os.environ["WARM_GIB"]),
                      "warm_s": time.perf_counter() - t_w}), flush=True)
t0 = time.perf_counter()
g = gb.rmat_graph(scale, samples, 7, densify_ids=True, max_block_keys=block)
g.device_csr()  # the CSR is built on first use
torch.cuda.synchronize()
print(json.dumps({"phase": "build", "V": g.num_vertices, "E": g.num_edges,
                  "s": time.perf_counter() - t0}), flush=True)
t_all = time.perf_counter()
cur = g
lvl = 0
scratch: dict = {}  # as coarsen_all: block buffers shared by the levels
while cur.num_vertices > 100:
    t = [time.perf_counter()]
    order = cz._degree_order_dev(cur)
    torch.cuda.synchronize(); t.append(time.perf_counter())
    m, r = cz._collapse_dev(cur, order)
    torch.cuda.synchronize(); t.append(time.perf_counter())
    if m.num_clusters > cz.STALL_RATIO * cur.num_vertices:
        break
    t_hist = time.perf_counter()
    nxt = cz.build_coarse_graph(cur, m, max_block_keys=block, scratch=scratch)
    torch.cuda.synchronize(); t.append(time.perf_counter())
    print(json.dumps({"level": lvl, "V": cur.num_vertices, "E": cur.num_edges,
                      "clusters": m.num_clusters, "coarse_E": nxt.num_edges, "rounds": r,
                      "order_ms": 1e3 * (t[1] - t[0]), "collapse_ms": 1e3 * (t[2] - t[1]),
                      "coarse_csr_ms": 1e3 * (t[3] - t[2])}), flush=True)
    cur = nxt
    lvl += 1
print(json.dumps({"phase": "coarsen_total", "s": time.perf_counter() - t_all,
                  "peak_gib": round(torch.cuda.max_memory_allocated() / 2**30, 2)}), flush=True)
