"""Where the C3 end-to-end embed time goes (train_multilevel(host Graph) ->
numpy): CSR upload, coarsening, each level's training, expands, matrix
download -- synchronised phase timings of the same calls train_multilevel
makes, CLI defaults (vertex-pass, 1000 epochs)."""
import json
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import numpy as np  # noqa: E402
import torch  # noqa: E402

import paper_2008_12336_b200 as gb  # noqa: E402
from paper_2008_12336_b200.evaluate import LinkPredictionSetup  # noqa: E402

UNIT = os.environ.get("UNIT", "vertex-pass")
g = gb.rmat_graph(22, 126_000_000, 7, densify_ids=True)
setup = LinkPredictionSetup.build(g, eval_seed=1, evaluator="device", eval_sample=1 << 20)
tg = setup.train_graph
xh, ah = tg.xadj, tg.adj
del g
cfg = gb.TrainConfig(dim=128, total_epochs=1000, smoothing_ratio=0.3, learning_rate=0.035,
                     negative_samples=3, seed=1, epoch_unit=UNIT)
for rep in range(3):
    ph = {}

    def mark(name, t):
        torch.cuda.synchronize()
        now = time.perf_counter()
        ph[name] = ph.get(name, 0.0) + now - t
        return now

    t0 = t = time.perf_counter()
    fresh = gb.Graph(tg.num_vertices, tg.num_edges, xadj=xh, adj=ah)
    fresh.device_csr()
    t = mark("csr_upload", t)
    h = gb.coarsen_all(fresh, threshold=100)
    t = mark("coarsen", t)
    plan = gb.epoch_plan(cfg.total_epochs, cfg.smoothing_ratio, h.depth).per_level
    M = torch.from_numpy(gb.init_embedding(h.graphs[-1].num_vertices, cfg.dim, cfg.seed)).cuda()
    t = mark("init", t)
    for i in range(h.depth - 1, -1, -1):
        if plan[i] > 0:
            gb.train_level(h.graphs[i], M, cfg, int(plan[i]), rng_stream=i)
        t = mark(f"train_L{i}", t)
        if i > 0:
            M = gb.expand_embedding(M, h.mappings[i - 1])
            t = mark("expand", t)
    from paper_2008_12336_b200._staging import device_to_numpy
    out = device_to_numpy(M)  # train_multilevel's download
    t = mark("download", t)
    ph["total"] = time.perf_counter() - t0
    print(json.dumps({"rep": rep, "unit": UNIT, "phases_s": {k: round(v, 4) for k, v in ph.items()},
                      "plan": [int(x) for x in plan],
                      "levels": [x.num_vertices for x in h.graphs]}), flush=True)
    del M, out, h, fresh
