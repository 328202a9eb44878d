"""The north star's target shape (friendster-shaped R-MAT) through the sharded
multilevel path with 8 ranks -- as virtual ranks on ONE B200 (K=16 parts,
CUDA-graph rotations) -- against the in-memory ladder: AUCROC on the
reference's link-prediction protocol (device evaluator, 1M+1M pairs) and the
per-level times, from which the 8-GPU time is projected (each sharded level's
one-GPU time / 8 + the unsharded levels).  UNIT / EPOCHS pick the schedule
(default: the CLI's large-graph 200 vertex-pass epochs)."""
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

RANKS = int(os.environ.get("RANKS", "8"))
SHARD = [int(x) for x in os.environ.get("SHARD", "1,2").split(",")]
UNIT = os.environ.get("UNIT", "vertex-pass")
EPOCHS = int(os.environ.get("EPOCHS", "200"))


def main():
    g = gb.rmat_graph(27, 1_900_000_000, 7, densify_ids=True)
    setup = LinkPredictionSetup.build(g, eval_seed=1, evaluator="device", eval_sample=1 << 20)
    del g
    tg, h = setup.train_graph, setup.hierarchy
    cfg = gb.TrainConfig(dim=128, total_epochs=EPOCHS, smoothing_ratio=0.3, learning_rate=0.035,
                         negative_samples=3, seed=1, epoch_unit=UNIT)
    plan = gb.epoch_plan(EPOCHS, 0.3, h.depth).per_level
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
                      "unit": UNIT, "epochs": EPOCHS, "embed_s": total, "level_s": level_s,
                      "aucroc": setup.score(M)}), flush=True)
    del M
    torch.cuda.empty_cache()
    for S in SHARD:
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        M, stats = gb.train_multilevel_sharded(tg, cfg, hierarchy=h, num_ranks=RANKS,
                                               shard_levels=S, return_device=True)
        torch.cuda.synchronize()
        total = time.perf_counter() - t0
        lv = {e["level"]: e["s"] for e in stats}
        sharded = [e["level"] for e in stats if e.get("sharded")]
        rot = {e["level"]: e.get("rotations") for e in stats if e.get("sharded")}
        proj = sum(lv[i] / RANKS if i in sharded else lv[i] for i in lv)
        print(json.dumps({"mode": f"sharded finest {S}", "ranks": RANKS, "K": 2 * RANKS,
                          "rotations": rot, "embed_s_one_gpu": total, "level_s": lv,
                          "projected_s_on_R_gpus": proj, "aucroc": setup.score(M)}), flush=True)
        del M
        torch.cuda.empty_cache()


if __name__ == "__main__":
    main()
