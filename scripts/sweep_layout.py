"""Sweep the training kernel's lane layout and in-flight cap on C2 (GPU box).
Prints one JSON line per setting: kernel ms per pass, updates/s, GB/s."""
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import numpy as np  # noqa: E402
import torch  # noqa: E402

import paper_2008_12336_b200 as gb  # noqa: E402
from paper_2008_12336_b200 import _lib  # noqa: E402

dim = int(os.environ.get("DIM", "128"))
G = gb.rmat_graph(20, 1 << 24, 7)
xadj, adj = G.device_csr()
src, n_src = G.active_sources()
M = torch.from_numpy(gb.init_embedding(G.num_vertices, dim, 1)).cuda()
lrs = torch.tensor([0.035], dtype=torch.float32, device="cuda")
st = _lib.new_status()
bps = 8 * dim * 5 + 12
lanes = [int(x) for x in os.environ.get("LANES", "8,16,32").split(",")]
caps = [int(x) for x in os.environ.get("CAPS", "0").split(",")]
p = 0
for g in lanes:
    os.environ["GB_GROUP_LANES"] = str(g)
    for cap in caps:
        def launch():
            global p
            _lib.call("gb_train_passes", G.num_vertices, _lib.ptr(xadj), _lib.ptr(adj),
                      _lib.ptr(src), n_src, _lib.ptr(M), dim, 3, 1, 0, p, 1, 1 << 40,
                      _lib.ptr(lrs), int(os.environ.get('FLAGS', '4')), cap, _lib.ptr(st), _lib.stream())
            p += 1
        for _ in range(3):
            launch()
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        n = 20
        e0.record()
        for _ in range(n):
            launch()
        e1.record()
        torch.cuda.synchronize()
        ms = e0.elapsed_time(e1) / n
        print(json.dumps({"lanes": g, "cap": cap, "dim": dim, "ms": ms,
                          "upd_per_s": n_src * 4 / ms * 1e3,
                          "GBps": n_src * bps / ms / 1e6}), flush=True)
