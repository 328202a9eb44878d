"""C1 AUCROC over many training seeds on the GPU, for in-flight policies.

Same protocol as scripts/c1_reference_auc.py (normal preset, d=32,
edge-scaled, eval_seed 1) but the split, the hierarchy and the evaluation
pairs are built once (they do not depend on the training seed), so each seed
costs one embed plus the device evaluator.  Env:
  SEEDS   e.g. "1-30" or "1,2,3"
  POLICY  ";"-separated floor/div pairs for the in-flight cap, e.g. "256/16;64/16"
  TAG     free-form label copied into the output line
Prints one JSON line per policy with per-seed AUCs, paired differences against
tests/golden/c1_reference_auc.json and their mean/CI.
"""
import json
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import numpy as np  # noqa: E402

import paper_2008_12336_b200 as gb  # noqa: E402
from paper_2008_12336_b200.evaluate import LinkPredictionSetup, aucroc_parity_interval  # noqa: E402

C1_GRAPH = dict(scale=14, samples=262144, seed=7, densify_ids=True)


def c1_config(seed):
    return gb.TrainConfig(dim=32, total_epochs=1000, smoothing_ratio=0.3, learning_rate=0.035,
                          negative_samples=3, seed=seed, epoch_unit="edge-scaled")


def parse_seeds(s):
    out = []
    for part in s.split(","):
        if "-" in part:
            a, b = part.split("-")
            out += list(range(int(a), int(b) + 1))
        elif part:
            out.append(int(part))
    return out


def main():
    seeds = parse_seeds(os.environ.get("SEEDS", "1-30"))
    policies = [p.split("/") for p in os.environ.get("POLICY", "256/16").split(";")]
    with open(os.path.join(ROOT, "tests", "golden", "c1_reference_auc.json")) as f:
        ref = {r["seed"]: r["aucroc"] for r in json.load(f)["runs"]}
    t0 = time.perf_counter()
    g = gb.rmat_graph(C1_GRAPH["scale"], C1_GRAPH["samples"], C1_GRAPH["seed"],
                      densify_ids=True)
    setup = LinkPredictionSetup.build(g, eval_seed=1, evaluator="device")
    setup_s = time.perf_counter() - t0
    for floor, div in policies:
        gb.trainer.INFLIGHT_FLOOR, gb.trainer.INFLIGHT_DIVISOR = int(floor), int(div)
        aucs, embed = [], []
        for seed in seeds:
            t1 = time.perf_counter()
            M = setup.embed(c1_config(seed))
            embed.append(time.perf_counter() - t1)
            aucs.append(setup.score(M))
        paired = [a - ref[s] for a, s in zip(aucs, seeds) if s in ref]
        print(json.dumps({
            "tag": os.environ.get("TAG", ""), "lib": os.environ.get("GB_LIB_PATH", "in-tree"),
            "policy": f"max({floor}, V/{div})", "seeds": seeds, "aucs": aucs,
            "mean": float(np.mean(aucs)), "std": float(np.std(aucs, ddof=1)),
            "ref_mean_same_seeds": float(np.mean([ref[s] for s in seeds if s in ref])),
            "paired": aucroc_parity_interval(paired),
            "embed_s_mean": float(np.mean(embed)), "setup_s": setup_s}), flush=True)


if __name__ == "__main__":
    main()
