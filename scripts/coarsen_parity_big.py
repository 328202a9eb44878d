"""Bit-exact coarsening at scale (GPU box): the device hierarchy of a large
R-MAT graph against the CPU oracle's sequential coarsen_all (the reference's
num_workers=1 parity path, coarsen.py:284-311), level by level -- maps,
cluster counts, coarse CSR.  Optionally the CSR build too (CPU generator +
csr_from_arcs vs the device R-MAT + CSR).

    SCALE=22 SAMPLES=126000000 CSR=1 python scripts/coarsen_parity_big.py"""
import json
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import numpy as np  # noqa: E402
import torch  # noqa: E402

import paper_2008_12336_b200 as gb  # noqa: E402
from oracle import oracle as orc  # noqa: E402

scale = int(os.environ.get("SCALE", "22"))
samples = int(os.environ.get("SAMPLES", "126000000"))
seed = int(os.environ.get("SEED", "7"))
t0 = time.perf_counter()
G = gb.rmat_graph(scale, samples, seed, densify_ids=True)
torch.cuda.synchronize()
gpu_build = time.perf_counter() - t0
x, a = G.xadj, G.adj
rec = {"scale": scale, "samples": samples, "vertices": G.num_vertices, "arcs": G.num_edges,
       "gpu_build_s": gpu_build}
if os.environ.get("CSR") == "1":
    t0 = time.perf_counter()
    cx, ca = orc.rmat_graph(scale, samples, seed, densify_ids=True)
    rec["cpu_build_s"] = time.perf_counter() - t0
    rec["csr_equal"] = bool(np.array_equal(cx, x) and np.array_equal(ca, a))
t0 = time.perf_counter()
h = gb.coarsen_all(G, threshold=100)
torch.cuda.synchronize()
rec["gpu_coarsen_s"] = time.perf_counter() - t0
t0 = time.perf_counter()
graphs, maps, stalled = orc.coarsen_all(x, a, 100)
rec["cpu_coarsen_s"] = time.perf_counter() - t0
rec["levels_gpu"] = [g.num_vertices for g in h.graphs]
rec["levels_cpu"] = [len(gx) - 1 for gx, _ in graphs]
ok = h.depth == len(graphs) and bool(h.stalled) == bool(stalled)
for L in range(1, min(h.depth, len(graphs))):
    cm, nc = maps[L - 1]
    m = h.mappings[L - 1]
    gl = h.graphs[L]
    ok &= (np.array_equal(m.map, cm) and int(m.num_clusters) == int(nc)
           and np.array_equal(gl.xadj, graphs[L][0]) and np.array_equal(gl.adj, graphs[L][1]))
rec["hierarchy_bit_exact"] = bool(ok)
print(json.dumps(rec), flush=True)
