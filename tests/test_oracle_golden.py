"""Pin the CPU oracle (oracle/gosh_oracle.c) to golden vectors produced by
the reference itself (tests/golden/make_golden.py).  CPU only."""
from __future__ import annotations

import numpy as np
import pytest


def test_rng_matches_reference(golden, orc):
    g = golden("rng.npz")
    for z, want in zip(g["mix_in"], g["mix_out"]):
        assert orc.mix64(int(z)) == int(want)
    for seed, stream, step, v, ctr, n, key, d in g["table"].tolist():
        assert orc.stream_key(seed, stream, step, v) == key
        assert orc.draw_below(key, ctr, n) == d


def test_update_embedding_bit_exact(golden, orc):
    g = golden("update.npz")
    for k, (d, b, reuse, v, s, lr) in enumerate(g["cases"].tolist()):
        M = g[f"c{k}_before"].copy()
        orc.update_embedding(M, int(v), int(s), int(b), lr, reuse=bool(reuse))
        assert np.array_equal(M, g[f"c{k}_after"]), k


def _graphs(g):
    out = []
    i = 0
    while f"g{i}_xadj" in g:
        out.append((g[f"g{i}_xadj"], g[f"g{i}_adj"]))
        i += 1
    return out


def test_train_pass_bit_exact(golden, orc):
    g = golden("train_pass.npz")
    graphs = _graphs(g)
    for k, (gi, d, n_neg, reuse, seed, stream, lr) in enumerate(g["cases"].tolist()):
        xadj, adj = graphs[int(gi)]
        M = g[f"c{k}_M0"].copy()
        for p in range(3):
            orc.train_pass(xadj, adj, M, lr, int(n_neg), int(seed), int(stream), p,
                           reuse=bool(reuse))
        assert np.array_equal(M, g[f"c{k}_M3"]), k


def test_train_level_bit_exact(golden, orc):
    g = golden("train_pass.npz")
    graphs = _graphs(g)
    for j, (gi, d, e_i, seed, stream, edge, passes, updates) in enumerate(g["levels"].tolist()):
        xadj, adj = graphs[gi]
        M = g[f"L{j}_M0"].copy()
        st = orc.train_level(xadj, adj, M, d, e_i, 0.05, 3, seed, stream,
                             "edge-scaled" if edge else "vertex-pass")
        assert st == (passes, updates)
        assert np.array_equal(M, g[f"L{j}_M"]), j


def test_coarsening_bit_exact(golden, orc):
    g = golden("coarsen.npz")
    for i, name in enumerate(g["names"].tolist()):
        xadj, adj = g[f"g{i}_xadj"], g[f"g{i}_adj"]
        order = orc.counting_order(np.diff(xadj))
        assert np.array_equal(order, g[f"g{i}_order"]), name
        cmap, nc = orc.collapse_seq(xadj, adj, order)
        assert nc == int(g[f"g{i}_nc"]) and np.array_equal(cmap, g[f"g{i}_map"]), name
        cx, ca = orc.coarse_csr(xadj, adj, cmap, nc)
        assert np.array_equal(cx, g[f"g{i}_cxadj"]) and np.array_equal(ca, g[f"g{i}_cadj"])
        graphs, maps, stalled = orc.coarsen_all(xadj, adj, int(g[f"g{i}_thr"]))
        assert len(graphs) == int(g[f"g{i}_depth"]) and stalled == bool(g[f"g{i}_stalled"])
        for L in range(1, len(graphs)):
            assert np.array_equal(graphs[L][0], g[f"g{i}_L{L}_xadj"]), (name, L)
            assert np.array_equal(graphs[L][1], g[f"g{i}_L{L}_adj"]), (name, L)
            assert np.array_equal(maps[L - 1][0], g[f"g{i}_M{L - 1}_map"]), (name, L)


def test_csr_build_bit_exact(golden, orc):
    g = golden("csr.npz")
    for k in range(int(g["n"])):
        pairs = g[f"c{k}_pairs"]
        directed = bool(g[f"c{k}_directed"])
        x, a = orc.csr_from_arcs(int(g[f"c{k}_V"]), pairs[:, 0], pairs[:, 1], drop_self=True,
                                 symmetrize=not directed)
        assert np.array_equal(x, g[f"c{k}_xadj"]) and np.array_equal(a, g[f"c{k}_adj"]), k


def test_pool_fill_and_train_pair_bit_exact(golden, orc):
    g = golden("pool.npz")
    graphs = _graphs(g)
    for k, row in enumerate(g["cases"].tolist()):
        gi, j, kk, lo_j, hi_j, lo_k, hi_k, d, B, n_neg, reuse, seed, lr, pos = row
        gi, j, kk, lo_j, hi_j, lo_k, hi_k, d, B, n_neg, reuse, seed, pos = map(
            int, (gi, j, kk, lo_j, hi_j, lo_k, hi_k, d, B, n_neg, reuse, seed, pos))
        xadj, adj = graphs[gi]
        tj = orc.fill_pool_side(xadj, adj, lo_j, hi_j, lo_k, hi_k, B, seed, 0)
        assert np.array_equal(tj, g[f"c{k}_tj"]), k
        Mj = g[f"c{k}_Mj0"].copy()
        Mk = Mj if j == kk else g[f"c{k}_Mk0"].copy()
        got = orc.train_pool_side(Mj, Mk, tj, lo_k, hi_k - lo_k, n_neg, lr, seed, 2,
                                  reuse=bool(reuse))
        if j != kk:
            tk = orc.fill_pool_side(xadj, adj, lo_k, hi_k, lo_j, hi_j, B, seed, 1)
            assert np.array_equal(tk, g[f"c{k}_tk"]), k
            got += orc.train_pool_side(Mk, Mj, tk, lo_j, hi_j - lo_j, n_neg, lr, seed, 3,
                                       reuse=bool(reuse))
        assert got == pos
        assert np.array_equal(Mj, g[f"c{k}_Mj"]), (k, "j")
        assert np.array_equal(Mk, g[f"c{k}_Mk"]), (k, "k")


def test_derived_seed(golden, orc):
    g = golden("pool.npz")
    got = [orc.derived_seed(s, st, p) for s in (1, 7, 2**40) for st in (0, 3) for p in (0, 1, 99)]
    assert got == [int(x) for x in g["derived"]]


def test_rmat_csr_matches_reference_builder(golden, orc):
    g = golden("rmat.npz")
    for k in range(2):
        scale, n, seed = g[f"r{k}_cfg"].tolist()
        perm = orc.rmat_permutation(scale, seed)
        assert np.array_equal(perm, g[f"r{k}_perm"])
        src, dst = orc.rmat_edges(scale, n, seed, perm)
        assert np.array_equal(src, g[f"r{k}_src"]) and np.array_equal(dst, g[f"r{k}_dst"])
        x, a = orc.csr_from_arcs(1 << scale, src, dst)
        assert np.array_equal(x, g[f"r{k}_xadj"]) and np.array_equal(a, g[f"r{k}_adj"])


def test_hogwild_oracle_runs_multithreaded(orc):
    x, a = orc.rmat_graph(10, 8000, 1)
    M = orc.init_embedding(len(x) - 1, 32, 1)
    orc.train_pass(x, a, M, 0.035, 3, 1, 0, 0, nthreads=4)
    assert np.isfinite(M).all()
