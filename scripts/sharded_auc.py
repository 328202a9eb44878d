"""AUCROC of the sharded multilevel path (finest level by the part-pair
tournament, virtual ranks on one GPU) against the in-memory path, on the C1
protocol (normal preset, d=32, edge-scaled, eval_seed 1, seeds from SEEDS).
Same split / features / logreg as run_link_prediction (evaluate.py:184-250).

    RANKS=1,2,4 SEEDS=1,2,3 python scripts/sharded_auc.py [c1|c3]"""
import json
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import numpy as np  # noqa: E402
import torch  # noqa: E402

import paper_2008_12336_b200 as gb  # noqa: E402
from paper_2008_12336_b200 import evaluate as ev  # noqa: E402

which = sys.argv[1] if len(sys.argv) > 1 else "c1"
if which == "c1":
    g = gb.rmat_graph(14, 262144, 7, densify_ids=True)
    dim = 32
else:
    g = gb.rmat_graph(22, 126_000_000, 7, densify_ids=True)
    dim = 128
ranks = [int(x) for x in os.environ.get("RANKS", "0,2,4").split(",")]
seeds = [int(x) for x in os.environ.get("SEEDS", "1,2,3").split(",")]
epochs = int(os.environ.get("EPOCHS", "1000"))
split = gb.split_train_test(g, 0.2, 1)
tg = split.train_graph
h = gb.coarsen_all(tg, threshold=100)
pos_train = tg.undirected_pairs()
neg_train = gb.sample_negative_edges(tg, pos_train.shape[0], seed=2)
pos_test = split.test_edges
neg_test = gb.sample_negative_edges(tg, pos_test.shape[0], seed=3, exclude_pairs=pos_test)
for R in ranks:
    aucs, embed = [], []
    for seed in seeds:
        cfg = gb.TrainConfig(dim=dim, total_epochs=epochs, smoothing_ratio=0.3,
                             learning_rate=0.035, negative_samples=3, seed=seed,
                             epoch_unit="edge-scaled")
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        if R == 0:
            M = gb.train_multilevel(tg, cfg, hierarchy=h)
        else:
            M, _ = gb.train_multilevel_sharded(tg, cfg, hierarchy=h, num_ranks=R)
        embed.append(time.perf_counter() - t0)
        f_train = gb.hadamard_features(M, *ev._balanced(pos_train, neg_train))
        f_test = gb.hadamard_features(M, *ev._balanced(pos_test, neg_test))
        model = gb.train_logreg(f_train, gb.LogRegConfig(seed=1))
        aucs.append(gb.auc_roc(gb.predict_scores(model, f_test.rows), f_test.labels))
    print(json.dumps({"graph": which, "ranks": R, "mode": "in-memory" if R == 0 else "tournament",
                      "aucs": aucs, "mean": float(np.mean(aucs)), "std": float(np.std(aucs)),
                      "embed_s": embed, "levels": [x.num_vertices for x in h.graphs]}),
          flush=True)
