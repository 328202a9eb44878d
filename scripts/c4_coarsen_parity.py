"""Bit-exact coarsening at the C4 (friendster) shape against the oracle.

R-MAT scale 27, 1.9B samples, ids densified (61.1M vertices, 3.74G arcs),
built on the device (gb_csr_build: bit-exact against the oracle's and the
reference's CSR at smaller scales, tests/test_gpu_parity.py and
tests/test_config_scale.py).  The device coarsens it (coarsen_all), the
CSR is downloaded and the oracle's sequential coarsen_all (oracle/
gosh_oracle.c, pinned bit-for-bit to the reference's coarsen_all(num_workers=1)
by the golden tests) coarsens the same arrays on the host; every level's
vertex / arc / cluster counts and xadj / adj / map checksums must be equal.
Writes tests/golden/coarsen_c4_hashes.json (the oracle's side) for the
driver-run GPU test.  Needs ~110 GB of host RAM and ~30 min of host CPU.
"""
import json
import os
import sys
import time

os.environ.setdefault("PYTORCH_CUDA_ALLOC_CONF", "backend:cudaMallocAsync")
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import torch  # noqa: E402

import paper_2008_12336_b200 as gb  # noqa: E402
from oracle import oracle as orc  # noqa: E402
from paper_2008_12336_b200.graph import array_checksum  # noqa: E402

SCALE = int(os.environ.get("SCALE", "27"))
SAMPLES = int(os.environ.get("SAMPLES", "1900000000"))
NAME = os.environ.get("NAME", "c4")
OUT = os.environ.get("OUT", os.path.join(ROOT, "gpurun_out", f"coarsen_{NAME}_hashes.json"))

t0 = time.perf_counter()
g = gb.rmat_graph(SCALE, SAMPLES, 7, densify_ids=True)
h = gb.coarsen_all(g, threshold=100)
torch.cuda.synchronize()
t_gpu = time.perf_counter() - t0
dev = []
for L, gl in enumerate(h.graphs):
    x, a = gl.device_csr()
    e = {"level": L, "vertices": gl.num_vertices, "arcs": gl.num_edges,
         "xadj": str(array_checksum(x)), "adj": str(array_checksum(a[: gl.num_edges]))}
    if L < len(h.mappings):
        e["map"] = str(array_checksum(h.mappings[L].device_map()))
        e["clusters"] = h.mappings[L].num_clusters
    dev.append(e)
print(json.dumps({"phase": "device", "s": t_gpu, "levels": [e["vertices"] for e in dev]}),
      flush=True)
xh, ah = g.xadj, g.adj
del h, g
torch.cuda.empty_cache()
t0 = time.perf_counter()
graphs, maps, stalled = orc.coarsen_all(xh, ah, 100)
t_orc = time.perf_counter() - t0
mine = []
for L, (x, a) in enumerate(graphs):
    e = {"level": L, "vertices": len(x) - 1, "arcs": int(x[-1]),
         "xadj": str(orc.checksum(x)), "adj": str(orc.checksum(a))}
    if L < len(maps):
        e["map"] = str(orc.checksum(maps[L][0]))
        e["clusters"] = int(maps[L][1])
    mine.append(e)
equal = mine == dev
print(json.dumps({"phase": "oracle", "s": t_orc, "levels": [e["vertices"] for e in mine],
                  "bit_exact": equal}), flush=True)
out = {"graph": {"scale": SCALE, "samples": SAMPLES, "seed": 7, "densified": True,
                 "generator": "device rmat_graph (CSR bit-exact vs oracle/reference at "
                              "smaller scales)"},
       "threshold": 100, "stalled": bool(stalled), "depth": len(mine), "levels": mine,
       "checksum": "sum_i mix64((i * 0x9E3779B97F4A7C15) ^ int64(x[i])) mod 2^64",
       "source": "oracle coarsen_all (pinned to the reference's coarsen_all(num_workers=1)) "
                 "on the box's host; the device hierarchy was identical" if equal else
                 "MISMATCH against the device hierarchy",
       "seconds": {"device_build_and_coarsen": t_gpu, "oracle_coarsen": t_orc}}
with open(OUT, "w") as f:
    json.dump(out, f, indent=1)
