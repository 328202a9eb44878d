"""Dense small level like C3's coarsest (V=2128, ~2.7M arcs, d=128): capped
training throughput vs in-flight cap and lane layout (GPU box).  With
NCU=1 runs a single short launch for ncu."""
import json
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import torch  # noqa: E402

import paper_2008_12336_b200 as gb  # noqa: E402
from paper_2008_12336_b200 import _lib  # noqa: E402

V = int(os.environ.get("V", "2128"))
p = float(os.environ.get("P", "0.6"))
dim = int(os.environ.get("DIM", "128"))
g = torch.Generator(device="cuda").manual_seed(0)
m = int(V * V * p / 2)
src = torch.randint(0, V, (m,), device="cuda", generator=g)
dst = torch.randint(0, V, (m,), device="cuda", generator=g)
G = gb.graph._csr_device(V, src, dst, _lib.GB_CSR_DROP_SELF | _lib.GB_CSR_SYMMETRIZE, False)
xadj, adj = G.device_csr()
srcs, n_src = G.active_sources()
M = torch.from_numpy(gb.init_embedding(V, dim, 1)).cuda()
lrs = torch.tensor([0.01], dtype=torch.float32, device="cuda")
st = _lib.new_status()
passes = int(os.environ.get("PASSES", "200"))
caps = [int(x) for x in os.environ.get("CAPS", "16,32,64,128,256,1024").split(",")]
for cap in caps:
    def run(n):
        _lib.call("gb_train_passes", V, _lib.ptr(xadj), _lib.ptr(adj), _lib.ptr(srcs), n_src,
                  _lib.ptr(M), dim, 3, 1, 0, 0, n, 1 << 40, _lib.ptr(lrs),
                  _lib.GB_TRAIN_FAST_SIGMOID | _lib.GB_TRAIN_ATOMIC, cap, _lib.ptr(st),
                  _lib.stream())
    if os.environ.get("NCU"):
        run(20)
        run(20)
        torch.cuda.synchronize()
        continue
    run(5)
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    run(passes)
    torch.cuda.synchronize()
    dt = time.perf_counter() - t0
    upd = passes * n_src * 4
    print(json.dumps({"V": V, "arcs": G.num_edges, "cap": cap,
                      "lanes": os.environ.get("GB_GROUP_LANES", "auto"),
                      "pipe": os.environ.get("GB_PIPE", "auto"), "upd_per_s": upd / dt,
                      "us_per_source_per_group": dt / (passes * n_src) * min(cap, n_src) * 1e6}),
          flush=True)
