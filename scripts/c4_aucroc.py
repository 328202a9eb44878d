"""Link-prediction AUCROC on the C4 (friendster-shaped) graph on ONE B200.

BASELINE.json configs[3]: friendster-shaped R-MAT (65.6M vertices, 1.8B
edges), d=128, multilevel.  Here: R-MAT scale 27, 1.9B samples, ids
densified (61.1M vertices, 1.87B undirected edges), the reference's
link-prediction protocol (test fraction 0.2, eval seed 1; evaluate.py:184-250)
with the device split, coarsening and evaluator (1M+1M pair subsample), the
CLI's large-graph defaults (cli.py:59-78, 162: 200 epochs, vertex-pass) and,
with RUNS containing "edge", an edge-scaled run of EDGE_EPOCHS epochs.
Prints JSON lines: setup phases, then per run embed seconds, updates/s and
AUCROC.  The CPU reference cannot run this size in reasonable time (its
sequential coarsening alone is hours at 3.7B arcs), so there is no reference
AUCROC to pair it with; C1 and C3 carry the parity comparison.
"""
from __future__ import annotations

import json
import os
import sys
import time

os.environ.setdefault("PYTORCH_CUDA_ALLOC_CONF", "backend:cudaMallocAsync")
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import torch  # noqa: E402

import paper_2008_12336_b200 as gb  # noqa: E402
from paper_2008_12336_b200.evaluate import LinkPredictionSetup  # noqa: E402

SCALE = int(os.environ.get("SCALE", "27"))
SAMPLES = int(os.environ.get("SAMPLES", "1900000000"))
RUNS = os.environ.get("RUNS", "vertex").split(",")
EDGE_EPOCHS = int(os.environ.get("EDGE_EPOCHS", "10"))


def gib():
    return round(torch.cuda.max_memory_allocated() / 2**30, 2)


def main():
    t0 = time.perf_counter()
    g = gb.rmat_graph(SCALE, SAMPLES, 7, densify_ids=True)
    torch.cuda.synchronize()
    print(json.dumps({"phase": "build", "scale": SCALE, "samples": SAMPLES,
                      "vertices": g.num_vertices, "arcs": g.num_edges,
                      "s": time.perf_counter() - t0, "peak_gib": gib()}), flush=True)
    t0 = time.perf_counter()
    setup = LinkPredictionSetup.build(g, eval_seed=1, evaluator="device", eval_sample=1 << 20)
    del g
    torch.cuda.synchronize()
    h = setup.hierarchy
    print(json.dumps({"phase": "split+coarsen+pairs", "s": time.perf_counter() - t0,
                      "train_vertices": setup.train_graph.num_vertices,
                      "train_arcs": setup.train_graph.num_edges,
                      "levels": [x.num_vertices for x in h.graphs], "peak_gib": gib()}),
          flush=True)
    for run in RUNS:
        unit, epochs = ("edge-scaled", EDGE_EPOCHS) if run == "edge" else ("vertex-pass", 200)
        cfg = gb.TrainConfig(dim=128, total_epochs=epochs, smoothing_ratio=0.3,
                             learning_rate=0.035, negative_samples=3, seed=1, epoch_unit=unit)
        plan = gb.epoch_plan(epochs, 0.3, h.depth).per_level
        updates = 0
        for i, gi in enumerate(h.graphs):
            updates += (int(plan[i]) * gb.trainer.passes_per_epoch(gi, cfg)
                        * int(gi.active_sources()[1]) * 4)
        torch.cuda.synchronize()
        t1 = time.perf_counter()
        M = setup.embed(cfg)
        torch.cuda.synchronize()
        embed_s = time.perf_counter() - t1
        t2 = time.perf_counter()
        auc = setup.score(M)
        print(json.dumps({"phase": "embed", "unit": unit, "epochs": epochs, "embed_s": embed_s,
                          "updates": updates, "upd_per_s": updates / embed_s, "aucroc": auc,
                          "eval_s": time.perf_counter() - t2, "peak_gib": gib()}), flush=True)
        del M


if __name__ == "__main__":
    main()
