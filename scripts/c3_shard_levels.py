"""How many levels to shard (the multi-GPU Amdahl term) on C3.

C3 link-prediction protocol (train graph of the split, device evaluator on a
1M+1M subsample), edge-scaled 1000 epochs, d=128, seed 1.  Runs the
in-memory ladder (train_multilevel) and train_multilevel_sharded with the
finest S levels trained by the tournament over R virtual ranks (K = 2R
parts on this one GPU), S from SHARD (default 1,2,3), and prints per run the
AUCROC and per-level seconds.  The projected time on R GPUs counts each
sharded level's one-GPU time / R (the tournament has no reduction, and its
exchange is ~7% of a round at 900 GB/s) plus the unsharded
levels' time on rank 0."""
import json
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import torch  # noqa: E402

import paper_2008_12336_b200 as gb  # noqa: E402
from paper_2008_12336_b200.evaluate import LinkPredictionSetup  # noqa: E402

R = int(os.environ.get("RANKS", "8"))
SHARD = [int(x) for x in os.environ.get("SHARD", "1,2,3").split(",")]
UNIT = os.environ.get("UNIT", "edge-scaled")
EPOCHS = int(os.environ.get("EPOCHS", "1000"))


def main():
    g = gb.rmat_graph(22, 126_000_000, 7, densify_ids=True)
    setup = LinkPredictionSetup.build(g, eval_seed=1, evaluator="device", eval_sample=1 << 20)
    del g
    tg, h = setup.train_graph, setup.hierarchy
    cfg = gb.TrainConfig(dim=128, total_epochs=EPOCHS, smoothing_ratio=0.3, learning_rate=0.035,
                         negative_samples=3, seed=1, epoch_unit=UNIT)
    plan = gb.epoch_plan(cfg.total_epochs, cfg.smoothing_ratio, h.depth).per_level
    # in-memory ladder, timed per level
    M = torch.from_numpy(gb.init_embedding(h.graphs[-1].num_vertices, 128, 1)).cuda()
    level_s = {}
    t0 = time.perf_counter()
    for i in range(h.depth - 1, -1, -1):
        t1 = time.perf_counter()
        if plan[i] > 0:
            gb.train_level(h.graphs[i], M, cfg, int(plan[i]), rng_stream=i)
        torch.cuda.synchronize()
        level_s[i] = time.perf_counter() - t1
        if i > 0:
            M = gb.expand_embedding(M, h.mappings[i - 1])
    total = time.perf_counter() - t0
    print(json.dumps({"mode": "in-memory", "levels": [x.num_vertices for x in h.graphs],
                      "embed_s": total, "level_s": level_s, "aucroc": setup.score(M)}),
          flush=True)
    del M
    for S in SHARD:
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        M, stats = gb.train_multilevel_sharded(tg, cfg, hierarchy=h, num_ranks=R,
                                               shard_levels=S, return_device=True)
        torch.cuda.synchronize()
        total = time.perf_counter() - t0
        lv = {e["level"]: e["s"] for e in stats}
        sharded = [e["level"] for e in stats if e.get("sharded")]
        proj = sum(lv[i] / R if i in sharded else lv[i] for i in lv)
        print(json.dumps({"mode": f"sharded finest {S}", "ranks": R, "K": 2 * R,
                          "embed_s_one_gpu": total, "level_s": lv, "sharded_levels": sharded,
                          "projected_s_on_R_gpus": proj, "aucroc": setup.score(M)}), flush=True)
        del M


if __name__ == "__main__":
    main()
