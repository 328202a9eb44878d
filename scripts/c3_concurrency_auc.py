"""C3 link-prediction AUCROC against the number of sources in flight.

Same protocol as scripts/c3_equal_auc.py (C3 train graph, CLI defaults,
device evaluator on a 1M+1M subsample).  Scores:
  ref_w<T>   the oracle port of the reference path with T host threads
             (T=1 is bit-identical to the reference's default num_workers=1)
  gpu        the default device path (uncapped)
  gpu_cap<N> the device path with TrainConfig.max_inflight = N on every level
  gpu_ppr[A] VERSE PPR positives (similarity="ppr", alpha 0.A, default 0.85)
MODES (comma list) picks them, e.g. MODES=ref_w1,ref_w16,gpu,gpu_cap1024.
"""
from __future__ import annotations

import dataclasses
import json
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "scripts"))

import torch  # noqa: E402

import paper_2008_12336_b200 as gb  # noqa: E402
from paper_2008_12336_b200.evaluate import LinkPredictionSetup  # noqa: E402
from c3_equal_auc import reference_embed  # noqa: E402

MODES = os.environ.get("MODES", "ref_w16,gpu,gpu_cap4096,gpu_cap1024").split(",")
SEED = int(os.environ.get("SEED", "1"))
UNIT = os.environ.get("UNIT", "vertex-pass")
EPOCHS = int(os.environ.get("EPOCHS", "1000"))


def main():
    g = gb.rmat_graph(22, 126_000_000, 7, densify_ids=True)
    setup = LinkPredictionSetup.build(g, eval_seed=1, evaluator="device", eval_sample=1 << 20)
    tg = setup.train_graph
    xh, ah = tg.xadj, tg.adj
    del g
    base = gb.TrainConfig(dim=128, total_epochs=EPOCHS, smoothing_ratio=0.3, learning_rate=0.035,
                          negative_samples=3, seed=SEED, epoch_unit=UNIT)
    for mode in MODES:
        t0 = time.perf_counter()
        if mode.startswith("ref_w"):
            M, _, _, _, _ = reference_embed(xh, ah, base, int(mode[5:]))
        elif mode.startswith("gpu_ppr"):  # VERSE PPR positives, alpha = 0.<digits>
            alpha = float("0." + mode[len("gpu_ppr"):]) if len(mode) > 7 else 0.85
            cfg = dataclasses.replace(base, similarity="ppr", ppr_alpha=alpha)
            M = setup.embed(cfg)
            torch.cuda.synchronize()
        else:
            cfg = base if mode == "gpu" else dataclasses.replace(
                base, max_inflight=int(mode[len("gpu_cap"):]))
            M = setup.embed(cfg)
            torch.cuda.synchronize()
        embed_s = time.perf_counter() - t0
        auc = setup.score(M)
        print(json.dumps({"mode": mode, "seed": SEED, "unit": UNIT, "epochs": EPOCHS,
                          "embed_s": embed_s, "aucroc": auc}), flush=True)
        del M


if __name__ == "__main__":
    main()
