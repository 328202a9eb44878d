"""Config-scale coarsening goldens (run in the build container only).

Builds the C3-shaped graph (R-MAT scale 22, 126M samples, seed 7, ids
densified -- the bench's C3) with the oracle's generator, which is pinned
bit-for-bit to the device generator and, at small scale, to the reference's
from_edges (tests/golden/rmat.npz).  Then runs the REFERENCE's
coarsen_all(num_workers=1) (/root/reference/pkg/src/mlembed/coarsen.py:284-311,
its deterministic ladder) on that CSR and records, per level, the vertex and
arc counts and position-keyed checksums (oracle.checksum == device
gb_checksum) of xadj, adj and the level's map -- the arrays are GBs, so the
fixture holds their checksums.  The oracle's own coarsen_all is run beside it
as a cross-check.  Writes tests/golden/coarsen_<name>_hashes.json (c3; and
"s24": scale 24, 400M samples -- 9.7M vertices, 769M arcs, 6 levels).
"""
import json
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, ROOT)
sys.path.insert(0, "/root/reference/pkg/src")
os.environ.setdefault("NUMBA_CACHE_DIR", "/tmp/numba_cache")

import mlembed as ml  # noqa: E402
from oracle import oracle as orc  # noqa: E402

# python make_coarsen_hashes.py [scale samples name]   (default: the C3 shape)
SCALE, SAMPLES, SEED = 22, 126_000_000, 7
NAME = "c3"
if len(sys.argv) > 3:
    SCALE, SAMPLES, NAME = int(sys.argv[1]), int(sys.argv[2]), sys.argv[3]


def level_hashes(graphs, maps):
    out = []
    for L, (x, a) in enumerate(graphs):
        e = {"level": L, "vertices": len(x) - 1, "arcs": int(x[-1]),
             "xadj": str(orc.checksum(x)), "adj": str(orc.checksum(a))}
        if L < len(maps):
            e["map"] = str(orc.checksum(maps[L][0]))
            e["clusters"] = int(maps[L][1])
        out.append(e)
    return out


t0 = time.perf_counter()
x, a = orc.rmat_graph(SCALE, SAMPLES, SEED, densify_ids=True)
t_gen = time.perf_counter() - t0
print("graph", len(x) - 1, int(x[-1]), f"{t_gen:.1f}s", flush=True)
g = ml.Graph(num_vertices=len(x) - 1, num_edges=int(x[-1]), xadj=x, adj=a)
t0 = time.perf_counter()
h = ml.coarsen_all(g, threshold=100, num_workers=1)
t_ref = time.perf_counter() - t0
ref = level_hashes([(gi.xadj, gi.adj) for gi in h.graphs],
                   [(m.map, m.num_clusters) for m in h.mappings])
print("reference coarsen_all", f"{t_ref:.1f}s", [e["vertices"] for e in ref], flush=True)
t0 = time.perf_counter()
graphs, maps, stalled = orc.coarsen_all(x, a, 100)
t_orc = time.perf_counter() - t0
mine = level_hashes(graphs, maps)
assert mine == ref, "oracle and reference hierarchies differ"
assert bool(stalled) == bool(h.stalled)
out = {"graph": {"scale": SCALE, "samples": SAMPLES, "seed": SEED, "densified": True,
                 "generator": "oracle.rmat_graph (== device rmat_graph)"},
       "threshold": 100, "stalled": bool(h.stalled), "depth": len(ref), "levels": ref,
       "checksum": "sum_i mix64((i * 0x9E3779B97F4A7C15) ^ int64(x[i])) mod 2^64",
       "source": "reference mlembed.coarsen_all(num_workers=1); oracle coarsen_all identical",
       "seconds": {"generate": t_gen, "reference_coarsen": t_ref, "oracle_coarsen": t_orc}}
with open(os.path.join(ROOT, "tests", "golden", f"coarsen_{NAME}_hashes.json"), "w") as f:
    json.dump(out, f, indent=1)
print(json.dumps(out["seconds"]))
