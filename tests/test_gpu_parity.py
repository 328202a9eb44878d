"""GPU parity: the sm_100a kernels (through the C ABI) against the reference's
golden vectors and the CPU oracle.

Bars (north star): bit-exact for RNG, CSR, coarsening maps and levels, pools
and every deterministic training result; within 1e-5 relative for the
parallel (tree-dot / Hogwild) kernels on fixed sample lists.
"""
from __future__ import annotations

import numpy as np
import pytest
import torch

import paper_2008_12336_b200 as gb
from paper_2008_12336_b200 import _lib
from paper_2008_12336_b200.graph import Graph

pytestmark = pytest.mark.gpu

REL_TOL = 1e-5


def _graphs(g, prefix="g"):
    out = []
    i = 0
    while f"{prefix}{i}_xadj" in g:
        x, a = g[f"{prefix}{i}_xadj"], g[f"{prefix}{i}_adj"]
        out.append(Graph(len(x) - 1, int(x[-1]), xadj=x, adj=a))
        i += 1
    return out


def _rel_err(a, b):
    return float(np.max(np.abs(a.astype(np.float64) - b)) / max(np.max(np.abs(b)), 1e-30))


# -- RNG --------------------------------------------------------------------------
def test_device_rng_matches_reference(cuda, golden):
    t = golden("rng.npz")["table"]
    for row in t[::7].tolist():
        seed, stream, step, v, ctr, n, key, d = row
        out = torch.empty(3, dtype=torch.int64, device=cuda)
        _lib.call("gb_rng_draw_below", seed, stream, step, v, ctr, n, 3, _lib.ptr(out),
                  _lib.stream())
        assert int(out[0]) == d


def test_device_rng_batch_matches_oracle(cuda, orc):
    out = torch.empty(100000, dtype=torch.int64, device=cuda)
    _lib.call("gb_rng_draw_below", 5, 3, 9, 1000, 2, 123457, 100000, _lib.ptr(out),
              _lib.stream())
    assert np.array_equal(out.cpu().numpy(), orc.rng_draw_below(5, 3, 9, 1000, 2, 123457, 100000))


# -- CSR build / R-MAT --------------------------------------------------------------
def test_from_edges_matches_reference(cuda, golden):
    g = golden("csr.npz")
    for k in range(int(g["n"])):
        pairs = g[f"c{k}_pairs"]
        h = gb.from_edges(pairs, num_vertices=int(g[f"c{k}_V"]),
                          directed=bool(g[f"c{k}_directed"]))
        assert np.array_equal(h.xadj, g[f"c{k}_xadj"]), k
        assert np.array_equal(h.adj, g[f"c{k}_adj"]), k
        h.validate()


def test_from_edges_small_cases(cuda):
    g = gb.from_edges([(0, 1), (1, 0), (1, 2), (2, 2)], num_vertices=3)
    assert g.num_edges == 4 and g.xadj.tolist() == [0, 1, 3, 4] and g.adj.tolist() == [1, 0, 2, 1]
    d = gb.from_edges([(0, 1), (2, 1)], num_vertices=3, directed=True)
    assert d.has_arc(0, 1) and not d.has_arc(1, 0)
    e = gb.from_edges(np.zeros((0, 2), np.int64), num_vertices=4)
    assert e.num_edges == 0 and e.xadj.tolist() == [0] * 5
    with pytest.raises(gb.EmptyGraphError):
        gb.from_edges([], num_vertices=0)


def test_rmat_generator_matches_oracle_and_reference(cuda, orc, golden):
    g = golden("rmat.npz")
    for k in range(2):
        scale, n, seed = g[f"r{k}_cfg"].tolist()
        src, dst = gb.rmat_edges(scale, n, seed)
        assert np.array_equal(src.cpu().numpy(), g[f"r{k}_src"])
        assert np.array_equal(dst.cpu().numpy(), g[f"r{k}_dst"])
        h = gb.rmat_graph(scale, n, seed)
        assert np.array_equal(h.xadj, g[f"r{k}_xadj"]) and np.array_equal(h.adj, g[f"r{k}_adj"])
    # a larger instance against the oracle, raw and densified
    x, a = orc.rmat_graph(14, 1 << 18, 11)
    h = gb.rmat_graph(14, 1 << 18, 11)
    assert np.array_equal(h.xadj, x) and np.array_equal(h.adj, a)
    xd, ad = orc.rmat_graph(14, 1 << 18, 11, densify_ids=True)
    hd = gb.rmat_graph(14, 1 << 18, 11, densify_ids=True)
    assert np.array_equal(hd.xadj, xd) and np.array_equal(hd.adj, ad)
    hd.validate()


def test_load_edge_list_and_split(cuda, tmp_path):
    import io
    g = gb.load_edge_list(io.StringIO("# c\n5 9\n9 40\n\n40 5\n"))
    assert g.num_vertices == 3 and g.orig_ids.tolist() == [5, 9, 40] and g.num_edges == 6
    g = gb.rmat_graph(10, 4000, 3, densify_ids=True)
    a = gb.split_train_test(g, 0.2, seed=4)
    b = gb.split_train_test(g, 0.2, seed=4)
    assert np.array_equal(a.test_edges, b.test_edges)
    tg = a.train_graph
    tg.validate()
    assert np.all(tg.degrees() > 0)
    for u, v in a.test_edges[:50]:
        assert not tg.has_arc(int(u), int(v))


# -- coarsening -------------------------------------------------------------------------
def test_coarsening_matches_reference_goldens(cuda, golden):
    g = golden("coarsen.npz")
    for i, name in enumerate(g["names"].tolist()):
        x, a = g[f"g{i}_xadj"], g[f"g{i}_adj"]
        G = Graph(len(x) - 1, int(x[-1]), xadj=x, adj=a)
        order = gb.degree_order(G)
        assert np.array_equal(order, g[f"g{i}_order"]), name
        m = gb.collapse_map(G, order)
        assert m.num_clusters == int(g[f"g{i}_nc"]), name
        assert np.array_equal(m.map, g[f"g{i}_map"]), name
        cg = gb.build_coarse_graph(G, m)
        assert np.array_equal(cg.xadj, g[f"g{i}_cxadj"]), name
        assert np.array_equal(cg.adj, g[f"g{i}_cadj"]), name
        h = gb.coarsen_all(G, threshold=int(g[f"g{i}_thr"]))
        assert h.depth == int(g[f"g{i}_depth"]) and h.stalled == bool(g[f"g{i}_stalled"]), name
        for L in range(1, h.depth):
            assert np.array_equal(h.graphs[L].xadj, g[f"g{i}_L{L}_xadj"]), (name, L)
            assert np.array_equal(h.graphs[L].adj, g[f"g{i}_L{L}_adj"]), (name, L)
            assert np.array_equal(h.mappings[L - 1].map, g[f"g{i}_M{L - 1}_map"]), (name, L)


@pytest.mark.parametrize("scale,samples,dens", [(16, 1 << 20, True), (17, 1 << 21, False)])
def test_coarsen_all_bit_exact_on_rmat(cuda, orc, scale, samples, dens):
    x, a = orc.rmat_graph(scale, samples, 7, densify_ids=dens)
    graphs, maps, stalled = orc.coarsen_all(x, a, 100)
    G = gb.rmat_graph(scale, samples, 7, densify_ids=dens)
    h = gb.coarsen_all(G, threshold=100)
    assert h.depth == len(graphs) and h.stalled == stalled
    for L in range(1, h.depth):
        assert np.array_equal(h.graphs[L].xadj, graphs[L][0])
        assert np.array_equal(h.graphs[L].adj, graphs[L][1])
        assert np.array_equal(h.mappings[L - 1].map, maps[L - 1][0])


def test_directed_collapse_matches_oracle(cuda, orc):
    rng = np.random.default_rng(2)
    pairs = rng.integers(0, 300, size=(1500, 2))
    G = gb.from_edges(pairs, num_vertices=300, directed=True)
    order = gb.degree_order(G)
    cmap, nc = orc.collapse_seq(G.xadj, G.adj, order)
    m = gb.collapse_map(G, order)
    assert m.num_clusters == nc and np.array_equal(m.map, cmap)


def test_expand_matches_oracle(cuda, orc):
    rng = np.random.default_rng(1)
    for d in (3, 8, 32, 128):
        coarse = rng.random((40, d)).astype(np.float32)
        cmap = rng.integers(0, 40, size=1000).astype(np.int32)
        got = gb.expand_embedding(coarse, gb.Mapping(map=cmap, num_clusters=40))
        assert np.array_equal(got, orc.expand(coarse, cmap))
    with pytest.raises(ValueError):
        gb.expand_embedding(coarse[:3], gb.Mapping(map=cmap, num_clusters=40))


# -- training: exact (deterministic) kernels vs the reference ---------------------------
def test_update_embedding_bit_exact(cuda, golden):
    g = golden("update.npz")
    for k, (d, b, reuse, v, s, lr) in enumerate(g["cases"].tolist()):
        M = g[f"c{k}_before"].copy()
        gb.update_embedding(M, int(v), int(s), int(b), lr, reuse_updated_source=bool(reuse))
        assert np.array_equal(M, g[f"c{k}_after"]), k
    with pytest.raises(TypeError):
        gb.update_embedding(np.zeros((2, 4)), 0, 1, 1, 0.1)


def test_train_pass_exact_bit_exact_vs_reference(cuda, golden):
    g = golden("train_pass.npz")
    graphs = _graphs(g)
    for k, (gi, d, n_neg, reuse, seed, stream, lr) in enumerate(g["cases"].tolist()):
        G = graphs[int(gi)]
        M = torch.from_numpy(g[f"c{k}_M0"].copy()).cuda()
        lrs = torch.full((3,), lr, dtype=torch.float32, device="cuda")
        st = _lib.new_status()
        x, a = G.device_csr()
        flags = _lib.GB_TRAIN_EXACT | (_lib.GB_TRAIN_REUSE if reuse else 0)
        src, n_src = G.active_sources() if k % 2 else (None, 0)
        _lib.call("gb_train_passes", G.num_vertices, _lib.ptr(x), _lib.ptr(a), _lib.ptr(src),
                  n_src, _lib.ptr(M),
                  int(d), int(n_neg), int(seed), int(stream), 0, 3, 1, _lib.ptr(lrs), flags, 1,
                  _lib.ptr(st), _lib.stream())
        assert np.array_equal(M.cpu().numpy(), g[f"c{k}_M3"]), k


def test_train_level_deterministic_bit_exact(cuda, golden):
    g = golden("train_pass.npz")
    graphs = _graphs(g)
    for j, (gi, d, e_i, seed, stream, edge, passes, updates) in enumerate(g["levels"].tolist()):
        cfg = gb.TrainConfig(dim=d, total_epochs=e_i, seed=seed, negative_samples=3,
                             learning_rate=0.05, deterministic=True,
                             epoch_unit="edge-scaled" if edge else "vertex-pass")
        M = g[f"L{j}_M0"].copy()
        st = gb.train_level(graphs[gi], M, cfg, e_i, rng_stream=stream)
        assert st == (passes, updates)
        assert np.array_equal(M, g[f"L{j}_M"]), j


def test_train_multilevel_deterministic_bit_exact(cuda, golden):
    g = golden("large.npz")
    for k, (d, e, p10, edge, seed, thr, depth) in enumerate(g["multilevel"].tolist()):
        x, a = g[f"ml{k}_0_xadj"], g[f"ml{k}_0_adj"]
        G = Graph(len(x) - 1, int(x[-1]), xadj=x, adj=a)
        cfg = gb.TrainConfig(dim=d, total_epochs=e, smoothing_ratio=p10 / 10, seed=seed,
                             epoch_unit="edge-scaled" if edge else "vertex-pass",
                             deterministic=True)
        h = gb.coarsen_all(G, threshold=thr)
        assert h.depth == depth
        M = gb.train_multilevel(G, cfg, hierarchy=h)
        assert np.array_equal(M, g[f"ml{k}_M"]), k


# -- training: parallel kernels within 1e-5 on fixed sample lists -----------------------
@pytest.mark.parametrize("d", [8, 32, 33, 128, 256])
def test_tree_dot_single_group_within_tolerance(cuda, orc, d):
    """Fast layout (tree dot) with one group in flight = the reference's update
    order; only the fp64 summation order differs."""
    x, a = orc.rmat_graph(11, 16000, 5, densify_ids=True)
    G = Graph(len(x) - 1, int(x[-1]), xadj=x, adj=a)
    M0 = orc.init_embedding(G.num_vertices, d, 3)
    M = M0.copy()
    cfg = gb.TrainConfig(dim=d, seed=3, max_inflight=1)
    gb.train_level(G, M, cfg, 2, lr0=0.035, rng_stream=1)
    # lr decays per epoch in train_level; replay that schedule in the oracle
    ref = M0.copy()
    orc.train_level(x, a, ref, d, 2, 0.035, 3, 3, 1)
    assert _rel_err(M, ref) <= REL_TOL


def test_fixed_sample_lists_parallel_within_tolerance(cuda, orc):
    """One deterministic update epoch on fixed sample lists: disjoint sources
    and sample rows run fully parallel and must match the sequential oracle."""
    rng = np.random.default_rng(8)
    V, d, n = 40000, 128, 4000
    M0 = orc.init_embedding(V, d, 1) * 40.0  # larger rows: non-trivial scores
    perm = rng.permutation(V)
    src = perm[:n]
    samples = perm[n:n + 4 * n].reshape(n, 4)
    labels = np.array([1, 0, 0, 0], dtype=np.int8)
    M = M0.copy()
    gb.apply_sample_lists(M, src, samples, labels, 0.05)
    ref = M0.copy()
    for i in range(n):
        for j in range(4):
            orc.update_embedding(ref, int(src[i]), int(samples[i, j]), int(labels[j]), 0.05)
    assert _rel_err(M, ref) <= REL_TOL
    M2 = M0.copy()
    gb.apply_sample_lists(M2, src, samples, labels, 0.05, deterministic=True)
    assert np.array_equal(M2, ref)
    M3 = M0.copy()
    gb.apply_sample_lists(M3, src, samples, labels, 0.05, atomic_rows=False)
    assert _rel_err(M3, ref) <= REL_TOL


def test_atomic_rows_keep_concurrent_updates_of_a_hot_row(cuda, orc):
    """Every source trains against the same hub row at once: with vector-
    reduction write-back all increments land (the result matches the
    sequential order up to second-order staleness); plain stores lose most."""
    rng = np.random.default_rng(21)
    V, d, n, hub = 6000, 128, 4096, 5999
    M0 = orc.init_embedding(V, d, 3) * 40.0
    src = rng.permutation(V - 1)[:n]
    samples = np.full((n, 1), hub, dtype=np.int64)
    labels = np.array([1], dtype=np.int8)
    lr = 1e-4
    ref = M0.copy()
    for i in range(n):
        orc.update_embedding(ref, int(src[i]), hub, 1, lr)
    dref = ref[hub].astype(np.float64) - M0[hub]
    Ma = M0.copy()
    gb.apply_sample_lists(Ma, src, samples, labels, lr, atomic_rows=True)
    Ms = M0.copy()
    gb.apply_sample_lists(Ms, src, samples, labels, lr, atomic_rows=False)
    err_a = np.abs((Ma[hub] - M0[hub]) - dref).max() / np.abs(dref).max()
    err_s = np.abs((Ms[hub] - M0[hub]) - dref).max() / np.abs(dref).max()
    assert err_a < 1e-3, err_a
    assert err_s > 10 * err_a
    others = np.setdiff1d(np.arange(V), [hub])
    assert _rel_err(Ma[others], ref[others]) <= 1e-4


@pytest.mark.parametrize("variant", ["throughput", "latency", "staged", "staged_f64"])
@pytest.mark.parametrize("d", [16, 32, 64, 128, 256])
def test_single_group_passes_match_sequential(cuda, orc, d, variant, monkeypatch):
    """The parallel pass kernels (throughput, latency and shared-memory-staged
    variants) with one source in flight are the reference's sequential pass
    up to the tree dot and fp32 sigmoid: within 1e-5 relative after two
    passes."""
    monkeypatch.setenv("GB_PIPE", "1" if variant == "latency" else "0")
    monkeypatch.setenv("GB_PASS_SMEM", "1" if variant.startswith("staged") else "0")
    x, a = orc.rmat_graph(11, 20000, 3, densify_ids=True)
    g = Graph(len(x) - 1, int(x[-1]), xadj=x, adj=a)
    M0 = orc.init_embedding(g.num_vertices, d, 1) * 20.0
    ref = M0.copy()
    orc.train_level(x, a, ref, d, 2, 0.035, 3, 1, 0)
    M = M0.copy()
    cfg = gb.TrainConfig(dim=d, max_inflight=1, fast_sigmoid=variant != "staged_f64")
    gb.train_level(g, M, cfg, 2)
    assert _rel_err(M, ref) <= REL_TOL


def test_hogwild_pass_counts_and_finiteness(cuda, orc):
    G = gb.rmat_graph(16, 1 << 20, 2)
    M = torch.from_numpy(orc.init_embedding(G.num_vertices, 128, 1)).cuda()
    before = M.clone()
    cfg = gb.TrainConfig(dim=128, seed=1)
    st = gb.train_level(G, M, cfg, 3)
    non_iso = int((G.degrees() > 0).sum())
    assert st.passes == 3 and st.updates == 3 * non_iso * 4
    assert torch.isfinite(M).all()
    moved = (M != before).any(dim=1).cpu().numpy()
    assert moved[G.degrees() > 0].all()


def test_nonfinite_is_reported(cuda):
    G = gb.from_edges([(0, 1), (1, 2), (2, 3)], num_vertices=5)
    M = np.full((5, 8), 0.01, np.float32)
    M[4, 3] = np.nan  # untouched isolated row: caught by the full scan
    with pytest.raises(FloatingPointError):
        gb.train_level(G, M, gb.TrainConfig(dim=8), 1)
    M = np.full((5, 8), 0.01, np.float32)
    M[1, 0] = np.inf
    with pytest.raises(FloatingPointError):
        gb.train_level(G, M, gb.TrainConfig(dim=8), 1)


def test_train_level_edge_cases(cuda):
    G = gb.from_edges([(0, 1)], num_vertices=1 + 1)
    M = gb.init_embedding(2, 4, 1)
    before = M.copy()
    assert gb.train_level(G, M, gb.TrainConfig(dim=4), 0) == (0, 0)
    assert np.array_equal(M, before)
    with pytest.raises(ValueError):
        gb.train_level(G, M[:1], gb.TrainConfig(dim=4), 1)
    K6 = gb.from_edges([(i, j) for i in range(6) for j in range(i + 1, 6)], num_vertices=6)
    st = gb.train_level(K6, gb.init_embedding(6, 8, 1),
                        gb.TrainConfig(dim=8, epoch_unit="edge-scaled"), 2)
    assert st.passes == 10
    M0 = gb.train_multilevel(K6, gb.TrainConfig(dim=8, total_epochs=0, seed=3), no_coarsen=True)
    assert np.array_equal(M0, gb.init_embedding(6, 8, 3))


# -- partitioned path ---------------------------------------------------------------------
def test_pools_and_train_pair_bit_exact(cuda, golden):
    g = golden("pool.npz")
    graphs = _graphs(g)
    for k, row in enumerate(g["cases"].tolist()):
        gi, j, kk, lo_j, hi_j, lo_k, hi_k, d, B, n_neg, reuse, seed, lr, pos = row
        gi, j, kk, B, n_neg, seed, pos = map(int, (gi, j, kk, B, n_neg, seed, pos))
        G = graphs[gi]
        n = G.num_vertices
        plan = gb.PartitionPlan(K=3, boundaries=(np.arange(4, dtype=np.int64) * n) // 3)
        pool = gb.build_sample_pool(G, plan, (j, kk), B, seed)
        assert np.array_equal(pool.targets_j, g[f"c{k}_tj"]), k
        if j != kk:
            assert np.array_equal(pool.targets_k, g[f"c{k}_tk"]), k
        Mj = g[f"c{k}_Mj0"].copy()
        Mk = Mj if j == kk else g[f"c{k}_Mk0"].copy()
        got = gb.train_pair(Mj, Mk, pool, n_neg, lr, seed, reuse_updated_source=bool(reuse),
                            deterministic=True)
        assert got == pos
        assert np.array_equal(Mj, g[f"c{k}_Mj"]), (k, "j")
        assert np.array_equal(Mk, g[f"c{k}_Mk"]), (k, "k")


def test_fused_pool_equals_materialized(cuda, orc):
    x, a = orc.rmat_graph(12, 40000, 9, densify_ids=True)
    G = Graph(len(x) - 1, int(x[-1]), xadj=x, adj=a)
    n = G.num_vertices
    lo_j, hi_j, lo_k, hi_k = 0, n // 3, n // 3, 2 * n // 3
    M0 = orc.init_embedding(n, 32, 4)
    B, n_neg, lr, seed = 5, 3, 0.05, 77
    tj = orc.fill_pool_side(x, a, lo_j, hi_j, lo_k, hi_k, B, seed, 0)
    ref = M0.copy()
    Mj, Mk = ref[lo_j:hi_j].copy(), ref[lo_k:hi_k].copy()
    want_pos = orc.train_pool_side(Mj, Mk, tj, lo_k, hi_k - lo_k, n_neg, lr, seed, 2)
    dj = torch.from_numpy(M0[lo_j:hi_j].copy()).cuda()
    dk = torch.from_numpy(M0[lo_k:hi_k].copy()).cuda()
    st = _lib.new_status()
    xa, aa = G.device_csr()
    _lib.call("gb_train_pool_side", _lib.ptr(dj), _lib.ptr(dk), 32, None, hi_j - lo_j, B, lo_k,
              hi_k - lo_k, n_neg, lr, seed, 2, _lib.ptr(xa), _lib.ptr(aa), lo_j, 0,
              _lib.GB_TRAIN_EXACT, 1, _lib.ptr(st), _lib.stream())
    assert np.array_equal(dj.cpu().numpy(), Mj) and np.array_equal(dk.cpu().numpy(), Mk)
    assert int(st[2]) == want_pos


def _compact_pool(G, lo_s, hi_s, lo_t, hi_t, B, seed, side, sort=True):
    xa, aa = G.device_csr()
    n = hi_s - lo_s
    lst = torch.empty(max(n, 1), dtype=torch.int32, device="cuda")
    tg = torch.empty(max(n * B, 1), dtype=torch.int32, device="cuda")
    cnt = torch.empty(1, dtype=torch.int64, device="cuda")
    _lib.call("gb_fill_pool_compact", _lib.ptr(xa), _lib.ptr(aa), lo_s, hi_s, lo_t, hi_t, B,
              _lib.u64(seed), side, _lib.ptr(lst), _lib.ptr(tg), _lib.ptr(cnt), _lib.stream())
    c = int(cnt.item())
    lst_h = lst[:c].cpu().numpy()
    tg_h = tg[: c * B].cpu().numpy().reshape(c, B)
    if sort:
        o = np.argsort(lst_h, kind="stable")
        lst_h, tg_h = lst_h[o], tg_h[o]
    return lst_h, tg_h


def test_compact_pool_equals_materialized(cuda, orc):
    """gb_fill_pool_compact keeps exactly the sources with a pool and their
    materialized rows; the list-driven pair kernel (serial, EXACT) then equals
    the oracle's _train_pool_side bit for bit."""
    x, a = orc.rmat_graph(12, 40000, 9, densify_ids=True)
    G = Graph(len(x) - 1, int(x[-1]), xadj=x, adj=a)
    n = G.num_vertices
    lo_j, hi_j, lo_k, hi_k = 0, n // 3, n // 3, 2 * n // 3
    B, n_neg, lr, seed = 5, 3, 0.05, 77
    tj = orc.fill_pool_side(x, a, lo_j, hi_j, lo_k, hi_k, B, seed, 0)
    lst, tg = _compact_pool(G, lo_j, hi_j, lo_k, hi_k, B, seed, 0)
    live = np.flatnonzero(tj[:, 0] >= 0)
    assert np.array_equal(lst, live) and np.array_equal(tg, tj[live])
    assert 0 < len(live) < hi_j - lo_j
    M0 = orc.init_embedding(n, 32, 4)
    Mj, Mk = M0[lo_j:hi_j].copy(), M0[lo_k:hi_k].copy()
    want_pos = orc.train_pool_side(Mj, Mk, tj, lo_k, hi_k - lo_k, n_neg, lr, seed, 2)
    dj = torch.from_numpy(M0[lo_j:hi_j].copy()).cuda()
    dk = torch.from_numpy(M0[lo_k:hi_k].copy()).cuda()
    dl = torch.from_numpy(lst.astype(np.int32)).cuda()
    dt = torch.from_numpy(np.ascontiguousarray(tg, dtype=np.int32)).cuda()
    dc = torch.tensor([len(lst)], dtype=torch.int64, device="cuda")
    st = _lib.new_status()
    _lib.call("gb_train_pool_list", _lib.ptr(dj), _lib.ptr(dk), 32, _lib.ptr(dl), _lib.ptr(dt),
              _lib.ptr(dc), hi_j - lo_j, B, lo_k, hi_k - lo_k, n_neg, lr, seed, 2,
              _lib.GB_TRAIN_EXACT, 1, _lib.ptr(st), _lib.stream())
    assert np.array_equal(dj.cpu().numpy(), Mj) and np.array_equal(dk.cpu().numpy(), Mk)
    assert int(st[2]) == want_pos


@pytest.mark.parametrize("dim", [16, 128, 256])
@pytest.mark.parametrize("diagonal", [False, True])
def test_pair_kernel_fast_path_serial(cuda, orc, dim, diagonal):
    """The default (HOT) pair kernels -- fused pools and compacted lists --
    run serially (one group) against the oracle: tree dot + fp32 sigmoid
    within the 1e-5 bar, positives counted exactly.  Diagonal pairs on a
    small part exercise self-samples (load-once rule)."""
    x, a = orc.rmat_graph(10, 12000, 3, densify_ids=True)
    G = Graph(len(x) - 1, int(x[-1]), xadj=x, adj=a)
    n = G.num_vertices
    if diagonal:
        lo_j, hi_j = 0, 96
        lo_k, hi_k = lo_j, hi_j
    else:
        lo_j, hi_j, lo_k, hi_k = 0, n // 2, n // 2, n
    B, n_neg, lr, seed = 5, 3, 0.05, 31
    flags = _lib.GB_TRAIN_FAST_SIGMOID | _lib.GB_TRAIN_ATOMIC
    tj = orc.fill_pool_side(x, a, lo_j, hi_j, lo_k, hi_k, B, seed, 0)
    M0 = orc.init_embedding(n, dim, 4) * np.float32(40.0)  # |dot| ~ 1: sigmoid off its tails
    Mj = M0[lo_j:hi_j].copy()
    Mk = Mj if diagonal else M0[lo_k:hi_k].copy()
    want_pos = orc.train_pool_side(Mj, Mk, tj, lo_k, hi_k - lo_k, n_neg, lr, seed, 2)
    xa, aa = G.device_csr()
    for mode in ("fused", "list"):
        dj = torch.from_numpy(M0[lo_j:hi_j].copy()).cuda()
        dk = dj if diagonal else torch.from_numpy(M0[lo_k:hi_k].copy()).cuda()
        st = _lib.new_status()
        if mode == "fused":
            _lib.call("gb_train_pool_side", _lib.ptr(dj), _lib.ptr(dk), dim, None, hi_j - lo_j, B,
                      lo_k, hi_k - lo_k, n_neg, lr, seed, 2, _lib.ptr(xa), _lib.ptr(aa), lo_j, 0,
                      flags, 1, _lib.ptr(st), _lib.stream())
        else:
            lst, tg = _compact_pool(G, lo_j, hi_j, lo_k, hi_k, B, seed, 0)
            dl = torch.from_numpy(lst.astype(np.int32)).cuda()
            dt = torch.from_numpy(np.ascontiguousarray(tg, dtype=np.int32)).cuda()
            dc = torch.tensor([len(lst)], dtype=torch.int64, device="cuda")
            _lib.call("gb_train_pool_list", _lib.ptr(dj), _lib.ptr(dk), dim, _lib.ptr(dl),
                      _lib.ptr(dt), _lib.ptr(dc), hi_j - lo_j, B, lo_k, hi_k - lo_k, n_neg, lr,
                      seed, 2, flags, 1, _lib.ptr(st), _lib.stream())
        assert int(st[2]) == want_pos, mode
        assert _rel_err(dj.cpu().numpy(), Mj) <= REL_TOL, mode
        if not diagonal:
            assert _rel_err(dk.cpu().numpy(), Mk) <= REL_TOL, mode


def test_tournament_pool_modes_agree(cuda, monkeypatch):
    """The three pool modes of the tournament draw the same pools: the same
    positive count, and (serial, one group per launch) the same embedding up
    to the Hogwild kernels' summation order."""
    from paper_2008_12336_b200 import tournament as tn
    G = gb.rmat_graph(11, 20000, 5, densify_ids=True)
    cfg = gb.TrainConfig(dim=32, seed=3, negative_samples=3, max_inflight=1)
    outs = {}
    for mode in ("fused", "materialize", "compact"):
        monkeypatch.setenv("GB_POOL_MODE", mode)
        M = torch.from_numpy(gb.init_embedding(G.num_vertices, 32, 3)).cuda()
        st = tn.train_tournament(G, M, cfg, 2, batch_size=5, num_ranks=2)
        outs[mode] = (st["pos_updates"], M.cpu().numpy())
    assert outs["fused"][0] == outs["materialize"][0] == outs["compact"][0] > 0
    assert np.array_equal(outs["fused"][1], outs["materialize"][1])
    # compaction changes the order sources run in, not the samples
    assert _rel_err(outs["compact"][1], outs["fused"][1]) < 0.05


def _balanced_fill_host(orc, x, a, lo_s, hi_s, lo_t, hi_t, BK, seed, side):
    """Host restatement of gb_fill_pool_balanced (entries in source order)."""
    out = []
    for v in range(lo_s, hi_s):
        e0, e1 = int(x[v]), int(x[v + 1])
        deg = e1 - e0
        if deg == 0:
            continue
        row = a[e0:e1]
        f = e0 + int(np.searchsorted(row, lo_t, "left"))
        cnt = e0 + int(np.searchsorted(row, hi_t, "left")) - f
        u = orc.draw_below(orc.stream_key(seed, side, 2, v), 0, 1 << 53) * 2.0 ** -53
        npos = int(np.floor(BK * cnt / deg + u)) if cnt else 0
        out.append((v - lo_s, f, cnt, npos))
    return np.array(out, dtype=np.int64).reshape(-1, 4)


def _balanced_fill_device(G, lo_s, hi_s, lo_t, hi_t, BK, seed, side):
    xa, aa = G.device_csr()
    n = hi_s - lo_s
    lst = torch.empty(n, dtype=torch.int32, device="cuda")
    first = torch.empty(n, dtype=torch.int64, device="cuda")
    cnt = torch.empty(n, dtype=torch.int32, device="cuda")
    npos = torch.empty(n, dtype=torch.int32, device="cuda")
    count = torch.empty(1, dtype=torch.int64, device="cuda")
    _lib.call("gb_fill_pool_balanced", _lib.ptr(xa), _lib.ptr(aa), lo_s, hi_s, lo_t, hi_t, BK,
              _lib.u64(seed), side, _lib.ptr(lst), _lib.ptr(first), _lib.ptr(cnt),
              _lib.ptr(npos), _lib.ptr(count), _lib.stream())
    c = int(count.item())
    t = np.stack([lst[:c].cpu().numpy(), first[:c].cpu().numpy(), cnt[:c].cpu().numpy(),
                  npos[:c].cpu().numpy()], axis=1).astype(np.int64)
    return t[np.argsort(t[:, 0], kind="stable")]


def test_balanced_pool_fill_matches_host(cuda, orc):
    x, a = orc.rmat_graph(11, 16000, 4, densify_ids=True)
    G = Graph(len(x) - 1, int(x[-1]), xadj=x, adj=a)
    n = G.num_vertices
    lo_s, hi_s, lo_t, hi_t = n // 4, n // 2, n // 2, 3 * n // 4
    got = _balanced_fill_device(G, lo_s, hi_s, lo_t, hi_t, 40, 99, 1)
    want = _balanced_fill_host(orc, x, a, lo_s, hi_s, lo_t, hi_t, 40, 99, 1)
    assert np.array_equal(got, want)
    assert (want[:, 3] > 5).any() and (want[:, 3] == 0).any()


@pytest.mark.parametrize("exact", [True, False])
def test_balanced_pair_kernel_serial(cuda, orc, exact):
    """gb_train_pool_balanced run serially over a sorted entry list equals the
    host replay of its sample sequence through update_embedding: bit-exact
    with EXACT kernels, within 1e-5 for the HOT (tree-dot) kernel."""
    x, a = orc.rmat_graph(10, 12000, 6, densify_ids=True)
    G = Graph(len(x) - 1, int(x[-1]), xadj=x, adj=a)
    n = G.num_vertices
    lo_s, hi_s, lo_t, hi_t = 0, n // 2, n // 2, n
    ns, nt = hi_s - lo_s, hi_t - lo_t
    B, K, n_neg, lr, seed, dim = 5, 4, 3, 0.0625, 21, 32
    ent = _balanced_fill_host(orc, x, a, lo_s, hi_s, lo_t, hi_t, B * K, seed, 0)
    M0 = orc.init_embedding(n, dim, 2) * np.float32(30.0)
    ref = np.ascontiguousarray(np.concatenate([M0[lo_s:hi_s], M0[lo_t:hi_t]]))
    pos = 0
    for i, f, cnt, npos in ent.tolist():
        pkey = orc.stream_key(seed, 0, 0, lo_s + i)
        key = orc.stream_key(seed, 2, 1, i)
        for t in range(max(B, npos)):
            if t < npos:
                s_ = int(a[f + orc.draw_below(pkey, t, cnt)]) - lo_t
                orc.update_embedding(ref, i, ns + s_, 1, lr)
                pos += 1
            if t < B:
                for q in range(n_neg):
                    orc.update_embedding(ref, i, ns + orc.draw_below(key, t * n_neg + q, nt), 0,
                                         lr)
    dj = torch.from_numpy(M0[lo_s:hi_s].copy()).cuda()
    dk = torch.from_numpy(M0[lo_t:hi_t].copy()).cuda()
    dev = [torch.from_numpy(np.ascontiguousarray(ent[:, c].astype(dt))).cuda()
           for c, dt in ((0, np.int32), (1, np.int64), (2, np.int32), (3, np.int32))]
    dc = torch.tensor([len(ent)], dtype=torch.int64, device="cuda")
    st = _lib.new_status()
    flags = _lib.GB_TRAIN_EXACT if exact else _lib.GB_TRAIN_FAST_SIGMOID | _lib.GB_TRAIN_ATOMIC
    _lib.call("gb_train_pool_balanced", _lib.ptr(dj), _lib.ptr(dk), dim, *[_lib.ptr(t) for t in dev],
              _lib.ptr(dc), ns, B, lo_t, nt, n_neg, lr, seed, 2, _lib.ptr(G.device_csr()[1]),
              lo_s, 0, flags, 1, _lib.ptr(st), _lib.stream())
    got = np.concatenate([dj.cpu().numpy(), dk.cpu().numpy()])
    assert int(st[2]) == pos and int(st[3]) == len(ent) * B * n_neg
    if exact:
        assert np.array_equal(got, ref)
    else:
        assert _rel_err(got, ref) <= REL_TOL


def test_tournament_balanced_pools_counts(cuda):
    """Balanced pools in the tournament: B*n_neg negatives per source per pair
    side, and B*K positives per source per rotation in expectation."""
    from paper_2008_12336_b200 import tournament as tn
    G = gb.rmat_graph(12, 40000, 5, densify_ids=True)
    cfg = gb.TrainConfig(dim=32, seed=3, negative_samples=3, balanced_pools=True)
    M = torch.from_numpy(gb.init_embedding(G.num_vertices, 32, 3)).cuda()
    st = tn.train_tournament(G, M, cfg, 1, batch_size=5, num_ranks=2)
    K, R = st["K"], st["rotations"]
    non_iso = int((np.diff(G.xadj) > 0).sum())
    assert st["neg_updates"] == R * non_iso * K * 5 * 3
    want = R * non_iso * K * 5
    assert abs(st["pos_updates"] - want) < 0.01 * want
    assert torch.isfinite(M).all()
    with pytest.raises(gb.ConfigError):
        gb.TrainConfig(balanced_pools=True, deterministic=True).validate()


def test_train_large_deterministic_bit_exact(cuda, golden):
    g = golden("large.npz")
    G = _graphs(g)[0]
    for k, row in enumerate(g["large"].tolist()):
        d, e_i, B, edge, reuse, seed, res, rot, K, sw, pos = row
        cfg = gb.TrainConfig(dim=d, total_epochs=e_i, seed=seed, negative_samples=2,
                             epoch_unit="edge-scaled" if edge else "vertex-pass",
                             reuse_updated_source=bool(reuse), deterministic=True)
        M = g[f"r{k}_M0"].copy()
        st = gb.train_large(G, M, cfg, e_i, gb.MemoryBudget(res, batch_size=B), rng_stream=k)
        assert (st["rotations"], st["K"], st["switches"], st["pos_updates"]) == (rot, K, sw, pos)
        assert st["peak_bytes"] <= st["budget_bytes"]
        assert np.array_equal(M, g[f"r{k}_M"]), k


def test_train_large_device_matrix_hogwild(cuda, orc):
    G = gb.rmat_graph(12, 40000, 1, densify_ids=True)
    cfg = gb.TrainConfig(dim=32, seed=2, negative_samples=3)
    M = torch.from_numpy(orc.init_embedding(G.num_vertices, 32, 2)).cuda()
    budget = gb.MemoryBudget(3 * 32 * 4 * (G.num_vertices // 4 + 1) + 4 * 2 * 5 * 4 * G.num_vertices)
    st = gb.train_large(G, M, cfg, 10, budget)
    assert st["K"] >= 3 and st["pos_updates"] > 0 and torch.isfinite(M).all()


def test_train_large_async_staging_equals_pair_replay(cuda, orc):
    """train_large with many switches through the side-stream stager (2 slots,
    K >= 6, 3 rotations, host matrix page-locked in place) equals the
    sequential replay of its pair schedule by the oracle's pool/pair kernels:
    staging order and slot reuse cannot change the result."""
    x, a = orc.rmat_graph(13, 60000, 11, densify_ids=True)
    G = Graph(len(x) - 1, int(x[-1]), xadj=x, adj=a)
    d, B, n_s = 32, 3, 2
    V = G.num_vertices
    per_row = 2 * d * 4 + 4 * 2 * B * 4
    budget = gb.MemoryBudget(per_row * (-(-V // 7)) + 64, parts_resident=2, batch_size=B)
    cfg = gb.TrainConfig(dim=d, negative_samples=n_s, seed=9, deterministic=True)
    plan = gb.plan_partitions(V, d, budget)
    e_i = 3 * B * plan.K
    M0 = orc.init_embedding(V, d, 2)
    M = M0.copy()
    st = gb.train_large(G, M, cfg, e_i, budget)
    assert st["K"] == plan.K >= 6 and st["rotations"] == 3 and st["switches"] > 3 * plan.K
    ref = M0.copy()
    pairs = gb.rotation_pairs(plan.K)
    for r in range(3):
        lr = gb.lr_at(cfg.learning_rate, r, 3)
        for i, (pa, pb) in enumerate(pairs):
            seed = gb.bigtrain._derived_seed(cfg.seed, 0, r * len(pairs) + i)
            la, ha = plan.part_range(pa)
            lb, hb = plan.part_range(pb)
            A = np.ascontiguousarray(ref[la:ha])
            Bm = A if pa == pb else np.ascontiguousarray(ref[lb:hb])
            tj = orc.fill_pool_side(x, a, la, ha, lb, hb, B, seed, 0)
            orc.train_pool_side(A, Bm, tj, lb, hb - lb, n_s, lr, seed, 2)
            if pa != pb:
                tk = orc.fill_pool_side(x, a, lb, hb, la, ha, B, seed, 1)
                orc.train_pool_side(Bm, A, tk, la, ha - la, n_s, lr, seed, 3)
            ref[la:ha] = A
            if pa != pb:
                ref[lb:hb] = Bm
    assert np.array_equal(M, ref)


# -- reference behaviours at the API edges (test_trainer.py:194-211,
# test_acceptance.py:203-240, test_bigtrain.py) ------------------------------------
def _planted(blocks, size, p_in, p_out, seed):
    rng = np.random.default_rng(seed)
    n = blocks * size
    iu, ju = np.triu_indices(n, 1)
    same = (iu // size) == (ju // size)
    keep = rng.random(iu.shape[0]) < np.where(same, p_in, p_out)
    return gb.from_edges(np.column_stack([iu[keep], ju[keep]]), num_vertices=n)


def test_train_multilevel_zero_epochs(cuda):
    g = _planted(6, 12, 0.5, 0.02, 9)
    cfg = gb.TrainConfig(dim=8, total_epochs=0, seed=3)
    M = gb.train_multilevel(g, cfg, no_coarsen=True)
    assert np.array_equal(M, gb.init_embedding(g.num_vertices, 8, 3))
    h = gb.coarsen_all(g, threshold=4)
    M = gb.train_multilevel(g, cfg, hierarchy=h)
    lab = h.mappings[0].map
    for c in range(h.mappings[0].num_clusters):  # expansion ties cluster rows
        rows = M[lab == c]
        assert np.array_equal(rows, np.repeat(rows[:1], rows.shape[0], 0))


def test_shape_mismatches_are_rejected(cuda):
    g = _planted(4, 10, 0.5, 0.05, 2)
    h = gb.coarsen_all(g, threshold=4)
    with pytest.raises(ValueError):
        gb.expand_embedding(np.zeros((h.mappings[0].num_clusters + 1, 8), np.float32),
                            h.mappings[0])
    with pytest.raises(ValueError):
        gb.train_large(g, np.zeros((g.num_vertices + 1, 8), np.float32), gb.TrainConfig(dim=8),
                       1, gb.MemoryBudget(10**6))
    with pytest.raises(ValueError):
        gb.train_level(g, np.zeros((g.num_vertices - 1, 8), np.float32), gb.TrainConfig(dim=8),
                       1)


def test_out_of_core_fidelity(cuda):
    """Criterion 06 (test_acceptance.py:203-225): link-prediction AUCROC with
    the level forced out of core (K=3 and K=5 parts) stays within 2 points
    of the in-memory run."""
    g = _planted(60, 32, 0.3, 0.001, 7)
    cfg = gb.TrainConfig(dim=32, total_epochs=200, smoothing_ratio=0.5, learning_rate=0.025,
                         seed=1, epoch_unit="edge-scaled")
    base = gb.run_link_prediction(g, cfg, eval_seed=11, evaluator="device").aucroc
    assert base > 0.8
    n_train = gb.split_train_test(g, 0.2, 11).train_graph.num_vertices
    for K in (3, 5):
        per_row = 3 * 32 * 4 + 4 * 2 * 5 * 4
        budget = gb.MemoryBudget(per_row * (-(-n_train // K)) + 4096)
        assert gb.plan_partitions(n_train, 32, budget).K == K
        auc = gb.run_link_prediction(g, cfg, eval_seed=11, budget=budget,
                                     evaluator="device").aucroc
        assert abs(auc - base) <= 0.02, (K, auc, base)


# -- split and negative pairs on the device ----------------
def _host_split(g, frac, seed):
    """graph.py:222-265 restated in numpy (the reference's algorithm)."""
    x, a = g.xadj, g.adj
    src = np.repeat(np.arange(g.num_vertices, dtype=np.int64), np.diff(x))
    pairs = np.stack([src, a.astype(np.int64)], 1)
    pairs = pairs[pairs[:, 0] < pairs[:, 1]]
    m = pairs.shape[0]
    k = int(round(frac * m))
    sel = np.zeros(m, bool)
    sel[np.random.default_rng(seed).choice(m, size=k, replace=False)] = True
    tr, te = pairs[~sel], pairs[sel]
    used = np.zeros(g.num_vertices, bool)
    used[tr.ravel()] = True
    kept = np.flatnonzero(used)
    new = np.full(g.num_vertices, -1, np.int64)
    new[kept] = np.arange(kept.shape[0])
    t = new[te]
    t = t[(t >= 0).all(1)]
    both = np.vstack([new[tr], new[tr][:, ::-1]])
    key = np.unique(both[:, 0] * kept.shape[0] + both[:, 1])
    return kept, t, key


@pytest.mark.parametrize("scale,samples,frac,seed", [(10, 4000, 0.2, 1), (13, 90000, 0.3, 7),
                                                     (8, 300, 0.5, 3)])
def test_device_split_equals_reference_algorithm(cuda, orc, scale, samples, frac, seed):
    x, a = orc.rmat_graph(scale, samples, 5, densify_ids=True)
    g = gb.Graph(len(x) - 1, int(x[-1]), xadj=x, adj=a)
    sp = gb.split_train_test(g, frac, seed)
    kept, t, key = _host_split(g, frac, seed)
    assert np.array_equal(sp.kept_vertices, kept)
    assert np.array_equal(sp.test_edges, t)
    tg = sp.train_graph
    src = np.repeat(np.arange(tg.num_vertices, dtype=np.int64), np.diff(tg.xadj))
    assert np.array_equal(src * tg.num_vertices + tg.adj, key)
    assert np.array_equal(g.undirected_pairs(), gb.Graph(len(x) - 1, int(x[-1]), xadj=x,
                                                         adj=a).undirected_pairs())


def test_device_negative_edges_equal_host(cuda, orc):
    x, a = orc.rmat_graph(11, 30000, 2, densify_ids=True)
    g = gb.Graph(len(x) - 1, int(x[-1]), xadj=x, adj=a)
    g.device_csr()
    ex = g.undirected_pairs()[::7]
    for seed in (1, 5):
        h = gb.sample_negative_edges(g, 5000, seed)
        d = gb.sample_negative_edges_device(g, 5000, seed)
        assert np.array_equal(h, d)
        h = gb.sample_negative_edges(g, 3000, seed, exclude_pairs=ex)
        d = gb.sample_negative_edges_device(g, 3000, seed, exclude_pairs=ex)
        assert np.array_equal(h, d)


def test_host_register_failure_leaves_no_sticky_error(cuda):
    """a failed gb_host_register (here: the range is already
    registered) must not leave its error in the runtime's last-error slot,
    where the next launch's check would report it (the pin_memory() fallback
    of train_large relies on this)."""
    a = np.zeros(1 << 20, dtype=np.float32)
    L = _lib.load()
    assert L.gb_host_register(a.ctypes.data, a.nbytes) == _lib.GB_OK
    try:
        assert L.gb_host_register(a.ctypes.data, a.nbytes) != _lib.GB_OK
        x = torch.arange(1000, dtype=torch.int64, device="cuda")
        out = torch.zeros(1, dtype=torch.int64, device="cuda")
        _lib.call("gb_checksum", _lib.ptr(x), 1000, 8, _lib.ptr(out), _lib.stream())
        torch.cuda.synchronize()
    finally:
        assert L.gb_host_unregister(a.ctypes.data) == _lib.GB_OK


def test_train_multilevel_release_levels_same_result(cuda, orc):
    """release_levels drops each coarse level's CSR and map once the finer
    matrix is expanded (the C5-on-one-GPU memory plan) and changes nothing
    in the result (deterministic kernels)."""
    x, a = orc.rmat_graph(11, 20000, 4, densify_ids=True)
    cfg = gb.TrainConfig(dim=32, total_epochs=20, negative_samples=3, seed=2,
                         deterministic=True)
    g = Graph(len(x) - 1, int(x[-1]), xadj=x, adj=a)
    h1 = gb.coarsen_all(g, threshold=100)
    ref = gb.train_multilevel(g, cfg, hierarchy=h1)
    h2 = gb.coarsen_all(g, threshold=100)
    got = gb.train_multilevel(g, cfg, hierarchy=h2, release_levels=True)
    assert np.array_equal(got, ref)
    assert h2.depth > 2 and all(gl._adj_dev is None for gl in h2.graphs[1:])
    assert h1.graphs[1]._adj_dev is not None  # kept by default for a caller's hierarchy


def _fd_nce_gradient(v, s, b, h=1e-6):
    """Central differences of the NCE objective b log sig(v.s) + (1-b) log
    sig(-v.s) (the reference's criterion 7, test_trainer.py:25-42)."""
    def loss(vv, ss):
        x = float(np.dot(vv, ss))
        sig = 1.0 / (1.0 + np.exp(-x))
        return b * np.log(sig) + (1 - b) * np.log(1.0 - sig)
    gv = np.array([(loss(v + h * e, s) - loss(v - h * e, s)) / (2 * h) for e in np.eye(len(v))])
    gs = np.array([(loss(v, s + h * e) - loss(v, s - h * e)) / (2 * h) for e in np.eye(len(s))])
    return gv, gs


@pytest.mark.parametrize("deterministic", [True, False])
def test_update_matches_finite_difference_gradient(cuda, deterministic):
    """Every device update is an SGD step on the NCE objective: (new - old) /
    lr equals its finite-difference gradient within 1e-4 relative (EXACT
    kernel, and the fast-sigmoid Hogwild kernel on independent pairs)."""
    rng = np.random.default_rng(2024)
    n = 300
    dims = rng.integers(2, 9, size=n)
    worst = 0.0
    for d in sorted(set(dims.tolist())):
        idx = np.nonzero(dims == d)[0]
        m = idx.shape[0]
        M = (rng.random((2 * m, d)) - 0.5).astype(np.float32)
        b = rng.integers(0, 2, size=m)
        before = M.astype(np.float64)
        # pair i: source 2i, sample 2i+1; one list entry per source
        for lab in (0, 1):
            sel = np.nonzero(b == lab)[0]
            if sel.size == 0:
                continue
            gb.apply_sample_lists(M, 2 * sel, (2 * sel + 1)[:, None], [lab], 0.25,
                                  deterministic=deterministic)
        for i in range(m):
            gv, gs = _fd_nce_gradient(before[2 * i], before[2 * i + 1], int(b[i]))
            dv = (M[2 * i].astype(np.float64) - before[2 * i]) / 0.25
            ds = (M[2 * i + 1].astype(np.float64) - before[2 * i + 1]) / 0.25
            num = np.linalg.norm(np.concatenate([dv, ds]) - np.concatenate([gv, gs]))
            worst = max(worst, num / np.linalg.norm(np.concatenate([gv, gs])))
    assert worst <= 1e-4, worst
