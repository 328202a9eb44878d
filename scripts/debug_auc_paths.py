"""C1: same seed through run_link_prediction's flow and auc_modes' flow,
each embedding scored by both evaluators (diagnostic)."""
import json, os, sys, time
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import numpy as np
import torch
import paper_2008_12336_b200 as gb
from paper_2008_12336_b200 import evaluate as ev

g = gb.rmat_graph(14, 262144, 7, densify_ids=True)
split = gb.split_train_test(g, 0.2, 1)
tg = split.train_graph
h = gb.coarsen_all(tg, threshold=100)
pos_train = tg.undirected_pairs()
neg_train = gb.sample_negative_edges(tg, pos_train.shape[0], seed=2)
pos_test = split.test_edges
neg_test = gb.sample_negative_edges(tg, pos_test.shape[0], seed=3, exclude_pairs=pos_test)


def score(M):
    out = {}
    f_tr = gb.hadamard_features(M, *ev._balanced(pos_train, neg_train))
    f_te = gb.hadamard_features(M, *ev._balanced(pos_test, neg_test))
    m = gb.train_logreg(f_tr, gb.LogRegConfig(seed=1))
    out["host"] = gb.auc_roc(gb.predict_scores(m, f_te.rows), f_te.labels)
    d_tr = gb.hadamard_features_device(M, *ev._balanced(pos_train, neg_train))
    d_te = gb.hadamard_features_device(M, *ev._balanced(pos_test, neg_test))
    md = gb.train_logreg_device(d_tr, gb.LogRegConfig(seed=1))
    out["dev"] = gb.auc_roc_device(gb.predict_scores_device(md, d_te.rows), d_te.labels)
    out["w_rel"] = float(np.abs(m.weights - md.weights).max() / np.abs(m.weights).max())
    return out


for rep in range(2):
    for seed in (1, 2):
        cfg = gb.TrainConfig(dim=32, total_epochs=1000, smoothing_ratio=0.3, learning_rate=0.035,
                             negative_samples=3, seed=seed, epoch_unit="edge-scaled")
        M1 = gb.train_multilevel(tg, cfg)
        M2 = gb.train_multilevel(tg, cfg, hierarchy=h, return_device=True).cpu().numpy()
        rep_ = gb.run_link_prediction(g, cfg, eval_seed=1)
        print(json.dumps({"rep": rep, "seed": seed, "internal_coarsen": score(M1),
                          "given_hierarchy": score(M2), "run_link_prediction": rep_.aucroc}),
              flush=True)
