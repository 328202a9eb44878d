"""Host-side logic and the C-ABI library surface; no GPU needed.

Mirrors the reference's own host-logic tests (test_trainer.py:86-131,
test_bigtrain.py:23-245, test_eval.py:129-154, test_graph.py:88-110) against
the package, plus checks that libgosh_b200.so exports every entry point the
header declares.
"""
from __future__ import annotations

import io
import math
import os
import re

import numpy as np
import pytest

import paper_2008_12336_b200 as gb
from paper_2008_12336_b200 import _lib
from paper_2008_12336_b200.bigtrain import (_derived_seed, _ensure_resident, _pick_victim,
                                            next_submatrix, switch_submatrices)
from paper_2008_12336_b200.errors import ConfigError, PlanError, SplitError

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


# -- the C ABI ------------------------------------------------------------------
def test_library_exports_every_header_symbol():
    header = open(os.path.join(ROOT, "include", "gosh_b200.h")).read()
    declared = set(re.findall(r"^\s*(?:int|const char \*)\s*(gb_\w+)\(", header, re.M))
    assert len(declared) >= 20
    L = _lib.load()
    for name in declared:
        assert hasattr(L, name), name
    assert declared == set(_lib.exported_symbols())
    assert L.gb_version() == 1


def test_library_rejects_bad_arguments_without_gpu():
    L = _lib.load()
    rc = L.gb_train_passes(10, None, None, None, 0, None, 0, 3, 1, 0, 0, 1, 1, None, 0, 0, None,
                           None)
    assert rc == _lib.GB_E_INVALID
    assert b"gb_train_passes" in L.gb_last_error()
    with pytest.raises(ValueError):
        _lib.check(rc, "gb_train_passes")


# -- epoch schedule (trainer.py:145-181) ------------------------------------------
def test_epoch_plan_reference_cases():
    assert gb.epoch_plan(10, 0.5, 3).per_level.tolist() == [2, 3, 5]
    assert gb.epoch_plan(7, 0.3, 3).per_level.tolist() == [1, 2, 4]
    assert gb.epoch_plan(9, 0.25, 1).per_level.tolist() == [9]
    assert gb.epoch_plan(100, 0.3, 3).per_level.tolist() == [20, 30, 50]
    assert gb.epoch_plan(120, 1.0, 6).per_level.tolist() == [20] * 6


def test_epoch_plan_conserves_total_and_floor():
    rng = np.random.default_rng(55)
    for _ in range(400):
        depth = int(rng.integers(1, 12))
        e = int(rng.integers(depth, 5000))
        plan = gb.epoch_plan(e, float(rng.random()), depth)
        assert plan.per_level.sum() == e and plan.per_level.min() >= 1


def test_epoch_plan_rejects_bad_inputs():
    with pytest.raises(PlanError):
        gb.epoch_plan(3, 0.5, 4)
    with pytest.raises(PlanError):
        gb.epoch_plan(10, 0.5, 0)
    with pytest.raises(ConfigError):
        gb.epoch_plan(10, 1.5, 2)


def test_epoch_shares_halve_toward_finer_levels():
    _, geo = gb.epoch_shares(1000, 0.3, 7)
    assert all(geo[i + 1] == 2.0 * geo[i] for i in range(6))


def test_lr_decay_is_linear_with_floor():
    assert gb.lr_at(0.05, 0, 100) == 0.05
    assert gb.lr_at(0.05, 50, 100) == pytest.approx(0.025)
    assert gb.lr_at(0.05, 10_000, 100) == pytest.approx(0.05 * 1e-4)


def test_init_embedding_matches_numpy_pcg64():
    M = gb.init_embedding(50, 16, seed=9)
    assert M.dtype == np.float32 and np.all(np.abs(M) <= 0.5 / 16)
    want = np.random.default_rng(9).uniform(-0.5 / 16, 0.5 / 16, size=(50, 16)).astype(np.float32)
    assert np.array_equal(M, want)


def test_sigmoid_clamps():
    assert gb.sigmoid(-50.0) == 1.0 / (1.0 + math.exp(10.0))
    assert gb.sigmoid(0.0) == 0.5


def test_train_config_validation():
    for bad in (dict(dim=0), dict(total_epochs=-1), dict(smoothing_ratio=2.0),
                dict(learning_rate=0.0), dict(negative_samples=-1), dict(num_workers=0),
                dict(epoch_unit="x"), dict(max_inflight=-1)):
        with pytest.raises(ConfigError):
            gb.TrainConfig(**bad).validate()


def test_inflight_cap_policy():
    from paper_2008_12336_b200.trainer import inflight_cap
    assert inflight_cap(gb.TrainConfig(deterministic=True), 10**6) == 1
    assert inflight_cap(gb.TrainConfig(max_inflight=7), 10**6) == 7
    # default: uncapped (the cap is at least the level's vertex count)
    for V in (10, 1000, 1 << 20):
        assert inflight_cap(gb.TrainConfig(), V) >= V


# -- partitioned-trainer host logic (bigtrain.py) -----------------------------------
def _plan_k_oracle(n, d, res, P, S, B):
    cap = res // (P * d * 4 + S * 2 * B * 4)
    return max(P, -(-n // cap))


def test_plan_partitions_reference_case_and_random():
    plan = gb.plan_partitions(1_000_000, 128, gb.MemoryBudget(512 * 1024 * 1024))
    assert plan.K == 4
    rng = np.random.default_rng(77)
    for _ in range(200):
        n, d = int(rng.integers(10, 2_000_000)), int(rng.integers(4, 256))
        P, S, B = int(rng.integers(2, 6)), int(rng.integers(1, 8)), int(rng.integers(1, 12))
        per = P * d * 4 + S * 2 * B * 4
        res = int(rng.integers(per, per * n * 2))
        plan = gb.plan_partitions(n, d, gb.MemoryBudget(res, P, S, B))
        assert plan.K == _plan_k_oracle(n, d, res, P, S, B)
        w = np.diff(plan.boundaries)
        assert plan.boundaries[-1] == n and w.min() >= 1 and w.max() - w.min() <= 1
    with pytest.raises(PlanError):
        gb.plan_partitions(1000, 128, gb.MemoryBudget(64))


def test_memory_budget_validation():
    for kw in (dict(resident_bytes=0), dict(resident_bytes=1 << 20, parts_resident=1),
               dict(resident_bytes=1 << 20, pools_resident=0),
               dict(resident_bytes=1 << 20, batch_size=0)):
        with pytest.raises(ConfigError):
            gb.MemoryBudget(**kw)


def test_rotation_pairs_recurrence():
    def unroll(K):
        pairs = [(0, 0)]
        while len(pairs) < K * (K + 1) // 2:
            a, b = pairs[-1]
            pairs.append((a, b + 1) if a > b else (a + 1, 0))
        return pairs
    for K in range(1, 12):
        assert gb.rotation_pairs(K) == unroll(K)
    with pytest.raises(ConfigError):
        gb.rotation_pairs(0)


def _state_with(parts, K=5, rows=20, dim=4):
    plan = gb.PartitionPlan(K=K, boundaries=np.linspace(0, rows, K + 1, dtype=np.int64))
    backing = np.arange(rows * dim, dtype=np.float32).reshape(rows, dim)
    st = gb.ResidencyState.create(plan, backing, parts_resident=len(parts))
    for p in parts:
        switch_submatrices(st, -1, p)
    return st


def test_residency_state_machine():
    st = _state_with([1, 2, 4])
    pairs = gb.rotation_pairs(5)
    assert next_submatrix(st, pairs.index((4, 0)), pairs) == 3
    st = _state_with([4, 3])
    assert next_submatrix(st, pairs.index((4, 2)), pairs) is None
    st = _state_with([0, 1], K=4, rows=16)
    st.view(0)[:] = 7.5
    switch_submatrices(st, 0, 2)
    assert np.all(st.backing[0:4] == 7.5) and st.resident(2) and not st.resident(0)
    with pytest.raises(ValueError):
        switch_submatrices(st, 2, 1)
    with pytest.raises(ValueError):
        switch_submatrices(st, 3, 0)
    with pytest.raises(ValueError):
        switch_submatrices(st, -1, 0)
    st.in_flight = (2, 1)
    with pytest.raises(RuntimeError):
        switch_submatrices(st, 2, 0)
    st = _state_with([0, 1, 2])
    sched = [(0, 0), (1, 0), (3, 3), (4, 3)]
    assert _pick_victim(st, sched, -1, set()) == 2
    assert _pick_victim(st, sched, -1, {2}) == 1
    assert _pick_victim(st, sched, -1, {0, 1, 2}) is None
    plan = gb.PartitionPlan(K=5, boundaries=np.linspace(0, 20, 6, dtype=np.int64))
    st = gb.ResidencyState.create(plan, np.zeros((20, 4), np.float32), parts_resident=3)
    switch_submatrices(st, -1, 0)
    _ensure_resident(st, (2, 4), gb.rotation_pairs(5), 0)
    assert st.resident(2) and st.resident(4) and st.resident(0)


def test_derived_seed_matches_reference_golden(golden):
    g = golden("pool.npz")
    got = [_derived_seed(s, st, p) for s in (1, 7, 2**40) for st in (0, 3) for p in (0, 1, 99)]
    assert got == [int(x) for x in g["derived"]]


# -- evaluation harness (evaluate.py) -------------------------------------------------
def test_auc_against_brute_force_with_ties():
    rng = np.random.default_rng(3)
    for _ in range(20):
        n = int(rng.integers(2, 60))
        s = rng.integers(0, 5, size=n).astype(np.float64)
        y = rng.integers(0, 2, size=n)
        if y.min() == y.max():
            continue
        pos, neg = s[y == 1], s[y == 0]
        brute = (2 * (pos[:, None] > neg[None, :]).sum()
                 + (pos[:, None] == neg[None, :]).sum()) / (2 * pos.size * neg.size)
        assert gb.auc_roc(s, y) == pytest.approx(brute, abs=1e-15)
    assert gb.auc_roc([0.1, 0.9], [0, 1]) == 1.0
    with pytest.raises(ValueError):
        gb.auc_roc([1.0, 2.0], [1, 1])


def _host_graph(pairs, V):
    pairs = np.asarray(pairs)
    both = np.vstack([pairs, pairs[:, ::-1]])
    key = np.unique(both[:, 0] * V + both[:, 1])
    xadj = np.zeros(V + 1, dtype=np.int64)
    xadj[1:] = np.cumsum(np.bincount(key // V, minlength=V))
    return gb.Graph(V, key.shape[0], xadj=xadj, adj=(key % V).astype(np.int32))


def test_host_graph_methods_and_validate():
    g = _host_graph([(0, 1), (1, 2), (0, 2), (3, 4), (4, 5), (3, 5), (2, 3)], 6)
    g.validate()
    assert g.degree(2) == 3 and g.neighbors(2).tolist() == [0, 1, 3]
    assert g.degrees().tolist() == [2, 2, 3, 3, 2, 2]
    assert g.has_arc(2, 3) and not g.has_arc(0, 5)
    assert g.undirected_pairs().shape == (7, 2)
    bad = gb.Graph(3, 4, xadj=np.array([0, 2, 3, 4]), adj=np.array([2, 1, 0, 1], np.int32))
    with pytest.raises(ValueError):
        bad.validate()


def test_negative_edges_avoid_graph_and_exclusions():
    g = _host_graph([(i, (i + 1) % 30) for i in range(30)], 30)
    neg = gb.sample_negative_edges(g, 200, seed=4)
    assert neg.shape == (200, 2) and np.all(neg[:, 0] != neg[:, 1])
    assert not any(g.has_arc(int(u), int(v)) for u, v in neg)
    ex = np.array([[0, 5], [7, 9]])
    neg = gb.sample_negative_edges(g, 300, seed=5, exclude_pairs=ex)
    s = {tuple(p) for p in neg.tolist()}
    assert not ({(0, 5), (5, 0), (7, 9), (9, 7)} & s)
    assert np.array_equal(gb.sample_negative_edges(g, 50, 1), gb.sample_negative_edges(g, 50, 1))


def test_logreg_deterministic_and_separates():
    rng = np.random.default_rng(0)
    X = np.vstack([rng.normal(1, 0.3, (100, 4)), rng.normal(-1, 0.3, (100, 4))]).astype(
        np.float32)
    y = np.r_[np.ones(100), np.zeros(100)].astype(np.int8)
    f = gb.FeatureSet(rows=X, labels=y)
    m1 = gb.train_logreg(f, gb.LogRegConfig(epochs=20))
    m2 = gb.train_logreg(f, gb.LogRegConfig(epochs=20))
    assert np.array_equal(m1.weights, m2.weights)
    assert gb.auc_roc(gb.predict_scores(m1, X), y) > 0.99
    with pytest.raises(ValueError):
        gb.train_logreg(gb.FeatureSet(rows=X[:5], labels=np.ones(5, np.int8)))


def test_binary_cache_round_trip(tmp_path):
    g = _host_graph([(0, 1), (1, 2), (2, 3)], 5)
    p = str(tmp_path / "g.gshg")
    gb.save_graph(g, p)
    h = gb.load_graph(p)
    assert np.array_equal(h.xadj, g.xadj) and np.array_equal(h.adj, g.adj)
    (tmp_path / "bad").write_bytes(b"XXXX0000")
    with pytest.raises(ValueError):
        gb.load_graph(str(tmp_path / "bad"))


def test_embedding_io_round_trip(tmp_path):
    M = gb.init_embedding(7, 5, 3)
    p = str(tmp_path / "m.gshe")
    gb.save_embedding(M, p)
    assert np.array_equal(gb.load_embedding(p), M)
    buf = io.StringIO()
    gb.write_embedding_tsv(M[:2], buf, orig_ids=np.array([10, 20]))
    assert buf.getvalue().startswith("10\t")


def test_edge_list_parse_errors():
    with pytest.raises(gb.EdgeListParseError) as ei:
        gb.load_edge_list(io.StringIO("1 2\n3\n"))
    assert ei.value.line_number == 2
    with pytest.raises(gb.EdgeListParseError):
        gb.load_edge_list(io.StringIO("1 2\nx y\n"))
    with pytest.raises(gb.EmptyGraphError):
        gb.load_edge_list(io.StringIO("# only a comment\n\n"))


def test_split_rejects_degenerate_fractions():
    g = _host_graph([(0, 1), (1, 2)], 3)
    with pytest.raises(SplitError):
        gb.split_train_test(g, 0.0, 1)
    with pytest.raises(SplitError):
        gb.split_train_test(g, 1.0, 1)


def test_product_package_never_imports_the_oracle():
    pkg = os.path.join(ROOT, "paper_2008_12336_b200")
    for fn in os.listdir(pkg):
        if fn.endswith(".py"):
            src = open(os.path.join(pkg, fn)).read()
            assert not re.search(r"^\s*(from|import)\s+\S*oracle", src, re.M), fn
            assert "liboracle" not in src, fn


def test_pair_side_pool_modes_and_balanced_config(monkeypatch):
    """PairSides picks the pool mode from GB_POOL_MODE (compact by default,
    materialize for deterministic runs, balanced when configured) and
    rejects unknown modes; balanced pools need the Hogwild kernels."""
    from paper_2008_12336_b200.bigtrain import PairSides
    csr = (None, None)
    st = None
    monkeypatch.delenv("GB_POOL_MODE", raising=False)
    assert PairSides(csr, gb.TrainConfig(), 0, 5, st).mode == "compact"
    assert PairSides(csr, gb.TrainConfig(deterministic=True), 0, 5, st).mode == "materialize"
    assert PairSides(csr, gb.TrainConfig(balanced_pools=True), 0, 5, st, K=4).mode == "balanced"
    monkeypatch.setenv("GB_POOL_MODE", "fused")
    assert PairSides(csr, gb.TrainConfig(), 0, 5, st).mode == "fused"
    monkeypatch.setenv("GB_POOL_MODE", "bogus")
    with pytest.raises(gb.ConfigError):
        PairSides(csr, gb.TrainConfig(), 0, 5, st)
    with pytest.raises(gb.ConfigError):
        gb.TrainConfig(balanced_pools=True, deterministic=True).validate()


def test_round2_entry_points_reject_bad_arguments_without_gpu():
    """The round-2 entry points validate their arguments before touching the
    device: null pointers / bad sizes give GB_E_INVALID and a message naming
    the call (the reference's ValueError/ConfigError checks map to these)."""
    import ctypes as C
    L = _lib.load()
    sz = C.c_size_t(0)
    n = C.c_int64(0)
    res = (C.c_int64 * 5)()
    flags = C.c_int(0)
    cases = [
        ("gb_collapse_cas", lambda: L.gb_collapse_cas(0, None, None, None, 1.0, 1, None,
                                                      C.byref(n), None, 0, None)),
        ("gb_collapse_cas_workspace", lambda: L.gb_collapse_cas_workspace(0, C.byref(sz))),
        ("gb_csr_validate", lambda: L.gb_csr_validate(-1, 0, None, None, C.byref(flags), None,
                                                      0, None)),
        ("gb_parse_edge_text", lambda: L.gb_parse_edge_text(None, 10, None, None, res, None, 0,
                                                            None)),
        ("gb_unique_ids", lambda: L.gb_unique_ids(None, 0, None, C.byref(n), 1, None, 0, None)),
        ("gb_train_passes_ppr", lambda: L.gb_train_passes_ppr(10, None, None, None, 0, None, 32,
                                                              3, 1, 0, 0, 1, 1, None, 0, 0,
                                                              None, 0.0, None)),
        ("gb_fill_pool_compact_dp", lambda: L.gb_fill_pool_compact_dp(None, None, 0, 1, 0, 1, 5,
                                                                      None, 0, None, None, None,
                                                                      None)),
        ("gb_train_pool_list_dp", lambda: L.gb_train_pool_list_dp(None, None, 32, None, None,
                                                                  None, 1, 5, 0, 1, 3, None, 2,
                                                                  0, 0, None, None)),
    ]
    for name, call in cases:
        assert call() == _lib.GB_E_INVALID, name
        assert name.encode().split(b"_workspace")[0] in L.gb_last_error(), name


def test_row_block_plans_agree():
    """The row-block planner (graph.py) on numpy and on a tensor: the same
    consecutive blocks covering every row, each within the key cap unless it
    is a single row above it."""
    import torch

    from paper_2008_12336_b200.graph import plan_row_blocks, plan_row_blocks_tensor
    rng = np.random.default_rng(5)
    for n, cap in ((1, 10), (1000, 50), (5000, 700), (777, 10_000)):
        h = rng.integers(0, 40, size=n).astype(np.int64)
        h[rng.integers(0, n, size=max(1, n // 100))] = 3 * cap  # rows above the cap
        h[: min(n, 7)] = 0
        ref = plan_row_blocks(h, cap)
        got, upper, largest = plan_row_blocks_tensor(torch.from_numpy(h), cap)
        assert got == ref, (n, cap)
        assert upper == int(h.sum())
        assert largest == max(int(h[a:b].sum()) for a, b in ref)
        assert ref[0][0] == 0 and ref[-1][1] == n
        for (a, b), (c, _) in zip(ref, ref[1:]):
            assert b == c
        for a, b in ref:
            assert h[a:b].sum() <= cap or b - a == 1
