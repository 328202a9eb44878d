"""Sharded part-pair training (paper_2008_12336_b200/tournament.py).

CPU: the circle-method schedule covers rotation_pairs(K) once per rotation
with disjoint pairs per round and neighbour-only moves; the schedule +
exchange run over gloo with world_size 2 and 3 (the pair step replaced by
the oracle's C restatement of bigtrain.py's pool/pair kernels) equals the
sequential execution of the same pair order.  GPU: the device pair kernel
(deterministic) under virtual ranks equals that sequential oracle replay
bit for bit.
"""
from __future__ import annotations

import os
import tempfile

import numpy as np
import pytest
import torch

import paper_2008_12336_b200 as gb
from paper_2008_12336_b200 import tournament as tn
from paper_2008_12336_b200.graph import Graph


# -- schedule ----------------------------------------------------------------------
@pytest.mark.parametrize("G", [1, 2, 3, 4, 8])
def test_rounds_cover_every_pair_once_disjointly(G):
    K = 2 * G
    rounds = tn.tournament_rounds(K)
    assert len(rounds) == K
    seen = [pr for rnd in rounds for pr in rnd]
    assert sorted(seen) == sorted(gb.rotation_pairs(K))
    for rnd in rounds:
        parts = [p for pr in rnd for p in set(pr)]
        assert len(parts) == len(set(parts)) == K


@pytest.mark.parametrize("G", [2, 3, 4, 8])
def test_shift_moves_are_neighbour_only_and_a_permutation(G):
    K = 2 * G
    moves = tn.shift_moves(K)
    for sr, ss, dr, ds in moves:
        assert abs(sr - dr) <= 1
    per_rank_send = [sum(1 for m in moves if m[0] == r and m[2] != r) for r in range(G)]
    assert max(per_rank_send) <= 2
    # applying the moves to holdings equals shifting the arrangement
    arr = tn.initial_arrangement(K)
    hold = [list(h) for h in tn.holdings(arr)]
    new = [list(h) for h in hold]
    for sr, ss, dr, ds in moves:
        new[dr][ds] = hold[sr][ss]
    assert [tuple(h) for h in new] == tn.holdings(tn.shift(arr))
    for _ in range(K - 1):
        arr = tn.shift(arr)
    assert arr == tn.initial_arrangement(K)


def test_rejects_odd_part_count():
    with pytest.raises(gb.ConfigError):
        tn.tournament_rounds(3)


# -- CPU pair step (the oracle, as the checker) -----------------------------------
def _graph(orc, scale=9, samples=3000, seed=5):
    x, a = orc.rmat_graph(scale, samples, seed, densify_ids=True)
    return Graph(len(x) - 1, int(x[-1]), xadj=x, adj=a), x, a


def _oracle_pair_fn(orc, x, a, B, n_s):
    def fn(Ma, Mb, s):
        A = Ma.numpy()
        Bm = A if s.a == s.b else Mb.numpy()
        tj = orc.fill_pool_side(x, a, s.lo_a, s.hi_a, s.lo_b, s.hi_b, B, s.seed, 0)
        orc.train_pool_side(A, Bm, tj, s.lo_b, s.hi_b - s.lo_b, n_s, s.lr, s.seed, 2)
        if s.a != s.b:
            tk = orc.fill_pool_side(x, a, s.lo_b, s.hi_b, s.lo_a, s.hi_a, B, s.seed, 1)
            orc.train_pool_side(Bm, A, tk, s.lo_a, s.hi_a - s.lo_a, n_s, s.lr, s.seed, 3)
    return fn


def _sequential_replay(orc, g, x, a, M, cfg, e_i, G, B=5, stream=0):
    """The same pair order on one full matrix, no parts, no exchange."""
    K = 2 * G
    V = M.shape[0]
    bnd = (np.arange(K + 1, dtype=np.int64) * V) // K
    rot = tn.tournament_rotations(g, cfg, e_i, K, B)
    idx = tn.pair_index(K)
    P = len(idx)
    rnd_of = tn.pair_rounds(K)
    for r, (pa, pb) in tn.sequential_order(K, rot):
        lr = tn.round_lr(cfg.learning_rate, r, rnd_of[(pa, pb)], rot, K, e_i)
        seed = gb.bigtrain._derived_seed(cfg.seed, stream, r * P + idx[(pa, pb)])
        la, ha, lb, hb = int(bnd[pa]), int(bnd[pa + 1]), int(bnd[pb]), int(bnd[pb + 1])
        A = M[la:ha]
        Bm = A if pa == pb else M[lb:hb]
        tj = orc.fill_pool_side(x, a, la, ha, lb, hb, B, seed, 0)
        A2 = np.ascontiguousarray(A)
        B2 = A2 if pa == pb else np.ascontiguousarray(Bm)
        orc.train_pool_side(A2, B2, tj, lb, hb - lb, cfg.negative_samples, lr, seed, 2)
        if pa != pb:
            tk = orc.fill_pool_side(x, a, lb, hb, la, ha, B, seed, 1)
            orc.train_pool_side(B2, A2, tk, la, ha - la, cfg.negative_samples, lr, seed, 3)
        M[la:ha] = A2
        if pa != pb:
            M[lb:hb] = B2
    return rot


@pytest.mark.parametrize("G", [1, 2, 3, 4])
def test_virtual_ranks_equal_sequential_replay(orc, G):
    g, x, a = _graph(orc)
    cfg = gb.TrainConfig(dim=16, negative_samples=3, seed=3, deterministic=True)
    M0 = orc.init_embedding(g.num_vertices, 16, 1)
    ref = M0.copy()
    rot = _sequential_replay(orc, g, x, a, ref, cfg, 30, G)
    M = torch.from_numpy(M0.copy())
    st = tn.train_tournament(g, M, cfg, 30, num_ranks=G,
                             pair_fn=_oracle_pair_fn(orc, x, a, 5, 3))
    assert st["rotations"] == rot and st["K"] == 2 * G
    assert st["pairs"] == rot * (2 * G) * (2 * G + 1) // 2
    assert np.array_equal(M.numpy(), ref)
    assert not np.array_equal(ref, M0)


def _gloo_worker(rank, world, port, out_path, per_process=1):
    import torch.distributed as dist
    from oracle import oracle as orc
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        g, x, a = _graph(orc)
        cfg = gb.TrainConfig(dim=16, negative_samples=3, seed=3, deterministic=True)
        M = torch.from_numpy(orc.init_embedding(g.num_vertices, 16, 1))
        st = tn.train_tournament(g, M, cfg, 30, pair_fn=_oracle_pair_fn(orc, x, a, 5, 3),
                                 per_process=per_process)
        np.save(f"{out_path}.{rank}.npy", M.numpy())
        np.save(f"{out_path}.{rank}.stats.npy",
                np.array([st["pairs"], st["exchange_bytes"], st["ranks"]]))
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("world,per_process", [(2, 1), (3, 1), (4, 1), (2, 2)])
def test_gloo_tournament_equals_sequential_replay(orc, world, per_process):
    """K = 2 * world * per_process parts over `world` gloo processes: the
    schedule, the P2P shift (per_process=2 mixes in-process relabels with
    cross-process sends) and the all_gather equal the sequential replay."""
    import socket

    import torch.multiprocessing as mp
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        port = s.getsockname()[1]
    with tempfile.TemporaryDirectory() as td:
        out = os.path.join(td, "m")
        mp.spawn(_gloo_worker, args=(world, port, out, per_process), nprocs=world, join=True)
        g, x, a = _graph(orc)
        cfg = gb.TrainConfig(dim=16, negative_samples=3, seed=3, deterministic=True)
        ref = orc.init_embedding(g.num_vertices, 16, 1)
        G = world * per_process
        rot = _sequential_replay(orc, g, x, a, ref, cfg, 30, G)
        K = 2 * G
        for r in range(world):
            M = np.load(f"{out}.{r}.npy")
            assert np.array_equal(M, ref), f"rank {r}"
            pairs, sent, ranks = np.load(f"{out}.{r}.stats.npy").tolist()
            assert ranks == G and pairs == rot * K * (K + 1) // 2
            # every process sends <= 2 parts per shift; K-1 shifts per rotation
            max_rows = -(-g.num_vertices // K)
            assert 0 < sent <= rot * (K - 1) * world * 2 * max_rows * 16 * 4


def test_init_embedding_rows_equals_slice_of_full_draw():
    for V, d, seed in [(1000, 16, 1), (77, 33, 9), (5, 128, 2)]:
        full = gb.init_embedding(V, d, seed)
        for lo, hi in [(0, V), (0, 1), (V // 3, V // 2), (V - 1, V)]:
            assert np.array_equal(tn.init_embedding_rows(V, d, seed, lo, hi), full[lo:hi])


# -- GPU: device pair kernel under the tournament ----------------------------------
@pytest.mark.gpu
@pytest.mark.parametrize("G", [1, 2, 4])
def test_device_tournament_deterministic_bit_exact(cuda, orc, G):
    g, x, a = _graph(orc, scale=10, samples=6000)
    cfg = gb.TrainConfig(dim=32, negative_samples=3, seed=4, deterministic=True)
    M0 = orc.init_embedding(g.num_vertices, 32, 2)
    ref = M0.copy()
    _sequential_replay(orc, g, x, a, ref, cfg, 20, G)
    M = torch.from_numpy(M0.copy()).cuda()
    tn.train_tournament(g, M, cfg, 20, num_ranks=G)
    assert np.array_equal(M.cpu().numpy(), ref)


@pytest.mark.gpu
@pytest.mark.parametrize("G", [1, 2, 4])
def test_rotation_graph_deterministic_bit_exact(cuda, orc, G, monkeypatch):
    """Rotations 1.. replayed from one captured CUDA graph (seeds and lr from
    the device table, *_dp kernels) equal the sequential replay bit for bit,
    with the virtual ranks on their own streams (G > 1) and serialised."""
    g, x, a = _graph(orc, scale=10, samples=6000)
    cfg = gb.TrainConfig(dim=32, negative_samples=3, seed=4, deterministic=True)
    M0 = orc.init_embedding(g.num_vertices, 32, 2)
    ref = M0.copy()
    rot = _sequential_replay(orc, g, x, a, ref, cfg, 60, G)
    assert rot >= 2
    ref2 = ref.copy()
    _sequential_replay(orc, g, x, a, ref2, cfg, 60, G)  # a second call's worth
    monkeypatch.setenv("GB_ROTATION_GRAPH", "1")  # from 2 rotations (auto: 16)
    for vs in ("1", "0"):
        monkeypatch.setenv("GB_VIRTUAL_STREAMS", vs)
        tn.clear_rotation_graphs()
        M = torch.from_numpy(M0.copy()).cuda()
        st = tn.train_tournament(g, M, cfg, 60, num_ranks=G)
        assert st["rotations"] == rot and st["pairs"] == rot * (2 * G) * (2 * G + 1) // 2
        assert np.array_equal(M.cpu().numpy(), ref), vs
        # the second call replays the cached graph for every rotation
        assert len(tn._ROTATION_GRAPHS) == 1
        st2 = tn.train_tournament(g, M, cfg, 60, num_ranks=G)
        assert st2["pairs"] == st["pairs"] and st2["kernel_launches"] == st["kernel_launches"]
        assert np.array_equal(M.cpu().numpy(), ref2), vs


@pytest.mark.gpu
def test_rotation_graph_cache_keyed_on_kernel_flags(cuda, orc, monkeypatch):
    """The captured launches bake in the kernel flags, so a call whose flags
    differ (here the sigmoid flavour) must capture afresh instead of
    replaying the cached graph."""
    g, x, a = _graph(orc, scale=10, samples=6000)
    monkeypatch.setenv("GB_ROTATION_GRAPH", "1")
    tn.clear_rotation_graphs()
    M0 = orc.init_embedding(g.num_vertices, 32, 2)
    keys = []
    for fast in (True, False):
        cfg = gb.TrainConfig(dim=32, negative_samples=3, seed=4, fast_sigmoid=fast)
        M = torch.from_numpy(M0.copy()).cuda()
        tn.train_tournament(g, M, cfg, 60, num_ranks=2)
        assert len(tn._ROTATION_GRAPHS) == 1
        keys.append(next(iter(tn._ROTATION_GRAPHS)))
    assert keys[0] != keys[1]
    tn.clear_rotation_graphs()


@pytest.mark.gpu
@pytest.mark.parametrize("balanced", [False, True])
def test_rotation_graph_hogwild_matches_eager(cuda, orc, monkeypatch, balanced):
    """Default (Hogwild) pools: the graph-replayed rotations draw exactly the
    eager path's samples (equal positive/negative counts) and train to the
    same matrix up to Hogwild interleaving."""
    g, x, a = _graph(orc, scale=12, samples=40000)
    cfg = gb.TrainConfig(dim=64, negative_samples=3, seed=4, balanced_pools=balanced)
    M0 = torch.from_numpy(orc.init_embedding(g.num_vertices, 64, 2)).cuda()
    out = {}
    for mode in ("1", "0"):
        monkeypatch.setenv("GB_ROTATION_GRAPH", mode)
        M = M0.clone()
        st = tn.train_tournament(g, M, cfg, 200, num_ranks=4)
        assert st["rotations"] >= 3
        out[mode] = (M, st["pos_updates"], st["neg_updates"])
    (Mg, pg, ng), (Me, pe, ne) = out["1"], out["0"]
    assert (pg, ng) == (pe, ne) and pg > 0
    rel = float((Mg - Me).norm() / (Me - M0).norm())
    assert rel < 0.1, rel


@pytest.mark.gpu
@pytest.mark.parametrize("G", [2, 3])
def test_host_staged_parts_deterministic_bit_exact(cuda, orc, G):
    """Parts in pinned host memory staged through four device slots (the
    budget mode for levels whose parts exceed HBM) equal the sequential
    replay bit for bit, and only the slots occupy HBM."""
    g, x, a = _graph(orc, scale=10, samples=6000)
    cfg = gb.TrainConfig(dim=32, negative_samples=3, seed=4, deterministic=True)
    M0 = orc.init_embedding(g.num_vertices, 32, 2)
    ref = M0.copy()
    _sequential_replay(orc, g, x, a, ref, cfg, 20, G)
    M = M0.copy()
    st = tn.train_tournament(g, M, cfg, 20, num_ranks=G, host_parts=True)
    assert np.array_equal(M, ref)
    max_rows = -(-g.num_vertices // (2 * G))
    assert st["part_device_bytes"] == 4 * max_rows * 32 * 4


@pytest.mark.gpu
def test_sharded_multilevel_holds_only_parts(cuda, orc):
    """train_multilevel_sharded expands the coarse matrix straight into each
    rank's parts: with return_parts the finest level never exists whole on
    the device; gathering the parts gives the full-matrix path's result
    (deterministic kernels, virtual ranks)."""
    g, x, a = _graph(orc, scale=11, samples=20000)
    cfg = gb.TrainConfig(dim=32, total_epochs=20, negative_samples=3, seed=4,
                         deterministic=True)
    ref, _ = gb.train_multilevel_sharded(g, cfg, num_ranks=4)
    store, stats = gb.train_multilevel_sharded(g, cfg, num_ranks=4, return_parts=True)
    assert isinstance(store, tn.PartStore) and stats[-1]["sharded"]
    assert np.array_equal(store.to_full().cpu().numpy(), ref)
    store_h, _ = gb.train_multilevel_sharded(g, cfg, num_ranks=4, return_parts=True,
                                             host_parts=True)
    assert np.array_equal(store_h.to_full().cpu().numpy(), ref)
    assert store_h.device_bytes < g.num_vertices * 32 * 4


@pytest.mark.gpu
def test_device_tournament_hogwild_counts(cuda, orc):
    g, x, a = _graph(orc, scale=12, samples=40000)
    cfg = gb.TrainConfig(dim=128, negative_samples=3, seed=4, epoch_unit="edge-scaled")
    M = torch.from_numpy(orc.init_embedding(g.num_vertices, 128, 2)).cuda()
    st = tn.train_tournament(g, M, cfg, 2, num_ranks=4)
    assert st["pos_updates"] > 0 and st["neg_updates"] == 3 * st["pos_updates"]
    assert bool(torch.isfinite(M).all())


def test_ragged_parts_and_tiny_levels(orc):
    """Parts of unequal size (V not a multiple of K) and a level barely
    larger than K still equal the sequential replay; fewer rows than parts
    is rejected."""
    x, a = orc.rmat_graph(5, 120, 9, densify_ids=True)
    g = Graph(len(x) - 1, int(x[-1]), xadj=x, adj=a)
    cfg = gb.TrainConfig(dim=8, negative_samples=2, seed=5, deterministic=True)
    for G in (5, 7):  # V = 24: parts of 2 and 3 rows (K=10), 1 and 2 rows (K=14)
        assert g.num_vertices % (2 * G) != 0
        M0 = orc.init_embedding(g.num_vertices, 8, 4)
        ref = M0.copy()
        _sequential_replay(orc, g, x, a, ref, cfg, 7, G)
        M = torch.from_numpy(M0.copy())
        tn.train_tournament(g, M, cfg, 7, num_ranks=G, pair_fn=_oracle_pair_fn(orc, x, a, 5, 2))
        assert np.array_equal(M.numpy(), ref)
    tiny = Graph(3, 4, xadj=np.array([0, 1, 3, 4]), adj=np.array([1, 0, 2, 1], np.int32))
    with pytest.raises(gb.ConfigError):
        tn.train_tournament(tiny, torch.zeros(3, 8), cfg, 1, num_ranks=2,
                            pair_fn=lambda *args: None)


def test_virtual_streams_knob_validated(monkeypatch):
    """GB_VIRTUAL_STREAMS accepts auto / 0 / 1 only (tournament.py)."""
    g = Graph(4, 4, xadj=np.array([0, 1, 2, 3, 4]), adj=np.array([1, 0, 3, 2], np.int32))
    cfg = gb.TrainConfig(dim=8, negative_samples=2, seed=5, deterministic=True)
    monkeypatch.setenv("GB_VIRTUAL_STREAMS", "yes")
    with pytest.raises(gb.ConfigError):
        tn.train_tournament(g, torch.zeros(4, 8), cfg, 1, num_ranks=2,
                            pair_fn=lambda *args: None)
    monkeypatch.setenv("GB_VIRTUAL_STREAMS", "0")
    tn.train_tournament(g, torch.zeros(4, 8), cfg, 1, num_ranks=2, pair_fn=lambda *args: None)


def _nccl_worker(rank, world, port, out_path):
    import torch.distributed as dist
    from oracle import oracle as orc
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    torch.cuda.set_device(rank)
    dist.init_process_group("nccl", rank=rank, world_size=world,
                            device_id=torch.device("cuda", rank))
    try:
        g, x, a = _graph(orc, scale=10, samples=6000)
        cfg = gb.TrainConfig(dim=32, total_epochs=30, negative_samples=3, seed=4,
                             deterministic=True)
        M, stats = gb.train_multilevel_sharded(g, cfg)
        np.save(f"{out_path}.{rank}.npy", M)
    finally:
        dist.destroy_process_group()


def _nccl_tournament_worker(rank, world, port, out_path):
    import torch.distributed as dist
    from oracle import oracle as orc
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    torch.cuda.set_device(rank)
    dist.init_process_group("nccl", rank=rank, world_size=world,
                            device_id=torch.device("cuda", rank))
    try:
        g, x, a = _graph(orc, scale=10, samples=6000)
        cfg = gb.TrainConfig(dim=32, negative_samples=3, seed=4, deterministic=True)
        M = torch.from_numpy(orc.init_embedding(g.num_vertices, 32, 2)).cuda()
        st = tn.train_tournament(g, M, cfg, 20)
        np.save(f"{out_path}.{rank}.npy", M.cpu().numpy())
        np.save(f"{out_path}.{rank}.sent.npy", np.array([st["exchange_bytes"]]))
    finally:
        dist.destroy_process_group()


@pytest.mark.gpu
def test_nccl_two_ranks_exchange_equals_sequential_replay(cuda, orc):
    """Two real ranks (one GPU each): K = 4 parts, so every off-diagonal round
    ends with an NCCL P2P part exchange over NVLink (_the_ multi-GPU data
    path); the result equals the sequential replay bit for bit."""
    import socket

    import torch.multiprocessing as mp
    if torch.cuda.device_count() < 2:
        pytest.skip("needs two GPUs (gloo world 2-4 covers the exchange on CPU)")
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        port = s.getsockname()[1]
    with tempfile.TemporaryDirectory() as td:
        out = os.path.join(td, "m")
        mp.spawn(_nccl_tournament_worker, args=(2, port, out), nprocs=2, join=True)
        g, x, a = _graph(orc, scale=10, samples=6000)
        cfg = gb.TrainConfig(dim=32, negative_samples=3, seed=4, deterministic=True)
        ref = orc.init_embedding(g.num_vertices, 32, 2)
        _sequential_replay(orc, g, x, a, ref, cfg, 20, 2)
        for r in range(2):
            assert np.array_equal(np.load(f"{out}.{r}.npy"), ref)
            assert int(np.load(f"{out}.{r}.sent.npy")[0]) > 0


@pytest.mark.gpu
def test_nccl_process_group_path_equals_virtual_ranks(cuda, orc):
    """The torch.distributed (NCCL) code path of the sharded multilevel
    driver -- broadcast, tournament, all_reduce, all_gather -- on the GPUs
    this box has equals the in-process virtual-rank run bit for bit."""
    import socket

    import torch.multiprocessing as mp
    world = torch.cuda.device_count()
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        port = s.getsockname()[1]
    with tempfile.TemporaryDirectory() as td:
        out = os.path.join(td, "m")
        mp.spawn(_nccl_worker, args=(world, port, out), nprocs=world, join=True)
        g, x, a = _graph(orc, scale=10, samples=6000)
        cfg = gb.TrainConfig(dim=32, total_epochs=30, negative_samples=3, seed=4,
                             deterministic=True)
        ref, _ = gb.train_multilevel_sharded(g, cfg, num_ranks=world)
        for r in range(world):
            assert np.array_equal(np.load(f"{out}.{r}.npy"), ref)


def _gloo_gpu_worker(rank, world, port, out_path, what):
    """Processes sharing cuda:0 over gloo: the distributed device code path
    (device pair kernels, P2P shifts staged through the host, all_gather,
    all_reduce, broadcast) when only one GPU is present."""
    import torch.distributed as dist
    from oracle import oracle as orc
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    torch.cuda.set_device(0)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        g, x, a = _graph(orc, scale=10, samples=6000)
        if what == "tournament":
            cfg = gb.TrainConfig(dim=32, negative_samples=3, seed=4, deterministic=True)
            M = torch.from_numpy(orc.init_embedding(g.num_vertices, 32, 2)).cuda()
            st = tn.train_tournament(g, M, cfg, 20)
            np.save(f"{out_path}.{rank}.npy", M.cpu().numpy())
            np.save(f"{out_path}.{rank}.sent.npy", np.array([st["exchange_bytes"]]))
        else:
            cfg = gb.TrainConfig(dim=32, total_epochs=30, negative_samples=3, seed=4,
                                 deterministic=True)
            M, _ = gb.train_multilevel_sharded(g, cfg, shard_levels=2)
            np.save(f"{out_path}.{rank}.npy", M)
    finally:
        dist.destroy_process_group()


@pytest.mark.gpu
@pytest.mark.parametrize("world", [2, 3])
def test_gloo_processes_on_one_gpu_tournament(cuda, orc, world):
    """world processes x one rank each on the one GPU (K = 2 world parts):
    every off-diagonal round ends with a real cross-process part shift; the
    result equals the sequential replay bit for bit on every rank."""
    import socket

    import torch.multiprocessing as mp
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        port = s.getsockname()[1]
    with tempfile.TemporaryDirectory() as td:
        out = os.path.join(td, "m")
        mp.spawn(_gloo_gpu_worker, args=(world, port, out, "tournament"), nprocs=world,
                 join=True)
        g, x, a = _graph(orc, scale=10, samples=6000)
        cfg = gb.TrainConfig(dim=32, negative_samples=3, seed=4, deterministic=True)
        ref = orc.init_embedding(g.num_vertices, 32, 2)
        _sequential_replay(orc, g, x, a, ref, cfg, 20, world)
        for r in range(world):
            assert np.array_equal(np.load(f"{out}.{r}.npy"), ref), r
            assert int(np.load(f"{out}.{r}.sent.npy")[0]) > 0


@pytest.mark.gpu
def test_gloo_processes_on_one_gpu_sharded_multilevel(cuda, orc):
    """train_multilevel_sharded over two processes (broadcast of the coarse
    matrix, expand into parts, two sharded levels, all_gather) equals the
    in-process virtual-rank run bit for bit."""
    import socket

    import torch.multiprocessing as mp
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        port = s.getsockname()[1]
    with tempfile.TemporaryDirectory() as td:
        out = os.path.join(td, "m")
        mp.spawn(_gloo_gpu_worker, args=(2, port, out, "multilevel"), nprocs=2, join=True)
        g, x, a = _graph(orc, scale=10, samples=6000)
        cfg = gb.TrainConfig(dim=32, total_epochs=30, negative_samples=3, seed=4,
                             deterministic=True)
        ref, _ = gb.train_multilevel_sharded(g, cfg, num_ranks=2, shard_levels=2)
        for r in range(2):
            assert np.array_equal(np.load(f"{out}.{r}.npy"), ref), r


def test_round_lr_follows_the_in_memory_epochs():
    """round_lr gives each round the in-memory rate of the epoch its share of
    the level's work falls in: a one-epoch level (edge-scaled: ceil(E/V)
    passes at one rate) trains every round at lr0; a level with one epoch
    per round decays per round; the rate never increases."""
    lr0, K = 0.035, 8
    for rotations in (1, 3):
        R = rotations * K
        one = [tn.round_lr(lr0, r // K, r % K, rotations, K, 1) for r in range(R)]
        assert all(x == lr0 for x in one)
        per_round = [tn.round_lr(lr0, r // K, r % K, rotations, K, R) for r in range(R)]
        assert per_round == [gb.lr_at(lr0, r, R) for r in range(R)]
        for e in (2, 5, 83, 1000):
            seq = [tn.round_lr(lr0, r // K, r % K, rotations, K, e) for r in range(R)]
            assert all(a >= b for a, b in zip(seq, seq[1:])) and seq[0] == lr0
