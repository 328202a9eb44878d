"""Part-pair training sharded over GPUs: a round-robin tournament of parts.

The reference trains a level that does not fit in memory part pair by part
pair, one pair at a time, in the inside-out order of rotation_pairs
(bigtrain.py:133-161, 343-493).  During a pair only the rows of its two parts
are touched (bigtrain.py:215-260), so pairs with disjoint parts commute: G
GPUs can train G disjoint pairs at once with no reduction at all.  This
module schedules that:

  * K = 2G contiguous parts (PartitionPlan boundaries, bigtrain.py:58-75);
  * the circle method: positions 0..K-1, rank r holds the parts at positions
    r ("top") and K-1-r ("bottom"); after each round position 0 stays and
    every other part moves one position (p -> p+1, K-1 -> 1), so K-1 rounds
    pair every two parts exactly once.  Each move is to the same rank or a
    neighbouring one, so one round's exchange is <= 2 sends + 2 receives of
    one part per rank (NCCL send/recv over NVLink on the GPU box, gloo in
    the CPU tests);
  * every rotation starts with a diagonal round (each rank trains (t,t) and
    (b,b) on its own parts), then the K-1 off-diagonal rounds; after them
    the arrangement is back at the start;
  * a pair (a,b), a>=b as in rotation_pairs, trains side 2 (sources of a
    against b) then side 3 exactly like train_large's pair step, with the
    positive pools drawn on the GPU from the replicated device CSR
    (bigtrain.PairSides: compacted pools + list pair kernel) and seed _derived_seed(seed, stream,
    rot*P + index of (a,b) in rotation_pairs(K)) -- the pair's seed does
    not depend on the number of GPUs;
  * lr decays per rotation (bigtrain.py:432) and the rotation count is
    train_large's max(1, round(eff/(B*K))).

Because concurrent pairs are disjoint, the result on G ranks equals the
sequential execution of the same pair order (diagonal rounds, then rounds,
pairs within a round in any order): bit-exact in deterministic mode, which
tests/test_tournament.py checks for G=1..4 on CPU (gloo, virtual ranks) and
on the GPU.
"""
from __future__ import annotations

import dataclasses
import os
import time
from dataclasses import dataclass
from typing import Callable

import numpy as np
import torch

from . import _lib
from .bigtrain import PairSides, PartitionPlan, _derived_seed, rotation_pairs
from .errors import ConfigError
from .graph import Graph
from .trainer import TrainConfig, lr_at

TOP, BOT = 0, 1


# ---------------------------------------------------------------------------
# schedule (host, pure)
# ---------------------------------------------------------------------------
def position_owner(p: int, K: int) -> tuple[int, int]:
    """(rank, slot) that holds circle position p."""
    G = K // 2
    return (p, TOP) if p < G else (K - 1 - p, BOT)


def initial_arrangement(K: int) -> list[int]:
    """Part at each circle position at the start of a rotation."""
    return list(range(K))


def shift(arr: list[int]) -> list[int]:
    """One circle-method step: position 0 fixed, p -> p+1, K-1 -> 1."""
    if len(arr) <= 2:
        return list(arr)
    return [arr[0], arr[-1]] + arr[1:-1]


def holdings(arr: list[int]) -> list[tuple[int, int]]:
    """(top part, bottom part) per rank for an arrangement."""
    K = len(arr)
    return [(arr[r], arr[K - 1 - r]) for r in range(K // 2)]


def shift_moves(K: int) -> list[tuple[int, int, int, int]]:
    """(src_rank, src_slot, dst_rank, dst_slot) for one shift; moves that
    stay in place are omitted."""
    moves = []
    for p in range(1, K):
        q = p + 1 if p < K - 1 else 1
        if q == p:
            continue
        s, d = position_owner(p, K), position_owner(q, K)
        if s != d:
            moves.append((s[0], s[1], d[0], d[1]))
    return moves


def pair_key(a: int, b: int) -> tuple[int, int]:
    return (a, b) if a >= b else (b, a)


def tournament_rounds(K: int) -> list[list[tuple[int, int]]]:
    """One rotation: the diagonal round (2 pairs per rank, top first) then
    K-1 off-diagonal rounds (one pair per rank).  Round entries are per rank;
    the diagonal round is flattened as [r0 top, r0 bottom, r1 top, ...]."""
    if K < 2 or K % 2:
        raise ConfigError("the tournament needs an even number of parts >= 2")
    arr = initial_arrangement(K)
    rounds = [[(p, p) for t, b in holdings(arr) for p in (t, b)]]
    for _ in range(K - 1):
        rounds.append([pair_key(t, b) for t, b in holdings(arr)])
        arr = shift(arr)
    return rounds


def pair_index(K: int) -> dict[tuple[int, int], int]:
    return {pr: i for i, pr in enumerate(rotation_pairs(K))}


def tournament_rotations(g: Graph, cfg: TrainConfig, e_i: int, K: int, B: int) -> int:
    """train_large's rotation count (bigtrain.py:389-395)."""
    eff = e_i
    if cfg.epoch_unit == "edge-scaled" and g.num_edges > 0:
        eff = e_i * (-(-g.num_edges // g.num_vertices))
    return max(1, round(eff / (B * K)))


# ---------------------------------------------------------------------------
# pair step
# ---------------------------------------------------------------------------
@dataclass
class PairStep:
    """Everything one pair launch needs besides the two part buffers."""

    a: int
    b: int
    lo_a: int
    hi_a: int
    lo_b: int
    hi_b: int
    seed: int
    lr: float


PairFn = Callable[[torch.Tensor, torch.Tensor, PairStep], None]


def device_pair_fn(g: Graph, cfg: TrainConfig, B: int,
                   K: int = 1, status: torch.Tensor | None = None
                   ) -> tuple[PairFn, torch.Tensor]:
    """Pair step on the GPU: side 2 then side 3 (bigtrain.py:241-260) through
    bigtrain.PairSides (compacted pools + list pair kernel by default);
    returns (fn, status block).  Each fn owns its pool scratch, so fns made
    with a shared status may run on different streams at once."""
    _lib.require_cuda()
    csr = g.device_csr()
    flags = (_lib.GB_TRAIN_REUSE if cfg.reuse_updated_source else 0) | (
        _lib.GB_TRAIN_EXACT if cfg.deterministic else _lib.GB_TRAIN_FAST_SIGMOID) | (
        _lib.GB_TRAIN_ATOMIC if cfg.atomic_rows and not cfg.deterministic else 0)
    if status is None:
        status = _lib.new_status()
    n_s = cfg.negative_samples
    side_step = PairSides(csr, cfg, flags, B, status, K=K)

    def fn(Ma: torch.Tensor, Mb: torch.Tensor, s: PairStep) -> None:
        if s.hi_a - s.lo_a <= 0 or s.hi_b - s.lo_b <= 0:
            return
        side_step(Ma, Mb, s.lo_a, s.hi_a, s.lo_b, s.hi_b, s.seed, s.lr, 0, 2)
        if s.a != s.b:
            side_step(Mb, Ma, s.lo_b, s.hi_b, s.lo_a, s.hi_a, s.seed, s.lr, 1, 3)

    return fn, status


# ---------------------------------------------------------------------------
# communication: real ranks (torch.distributed) or virtual ranks (one process)
# ---------------------------------------------------------------------------
class _RankParts:
    """The two part buffers of one rank plus their receive twins."""

    def __init__(self, max_rows: int, dim: int, device, dtype=torch.float32):
        self.cur = [torch.zeros((max_rows, dim), dtype=dtype, device=device) for _ in range(2)]
        self.nxt = [torch.zeros((max_rows, dim), dtype=dtype, device=device) for _ in range(2)]


def _exchange_dist(parts: _RankParts, rank: int, moves, group) -> int:
    """Apply one shift on this rank with P2P send/recv; returns bytes sent.
    A slot takes the part of a local move, else what it received, else it
    keeps its part (position 0 never moves)."""
    import torch.distributed as dist
    ops, sent = [], 0
    new = list(parts.cur)
    received = set()
    for sr, ss, dr, ds in moves:
        if sr == rank and dr == rank:
            new[ds] = parts.cur[ss]
        elif sr == rank:
            ops.append(dist.P2POp(dist.isend, parts.cur[ss], dr, group))
            sent += parts.cur[ss].numel() * parts.cur[ss].element_size()
        elif dr == rank:
            ops.append(dist.P2POp(dist.irecv, parts.nxt[ds], sr, group))
            received.add(ds)
    if ops:
        for w in dist.batch_isend_irecv(ops):
            w.wait()
    for ds in received:
        new[ds] = parts.nxt[ds]
    used = {id(t) for t in new}
    parts.nxt = [t for t in parts.cur + parts.nxt if id(t) not in used]
    parts.cur = new
    return sent


def _exchange_virtual(all_parts: list[_RankParts], moves) -> None:
    """Apply one shift to every virtual rank by swapping buffer references."""
    new = [list(p.cur) for p in all_parts]
    for sr, ss, dr, ds in moves:
        new[dr][ds] = all_parts[sr].cur[ss]
    for r, p in enumerate(all_parts):
        p.cur = new[r]


# ---------------------------------------------------------------------------
# driver
# ---------------------------------------------------------------------------
def _steps_for_round(rnd: list[tuple[int, int]], G: int, diagonal: bool):
    if diagonal:
        return [rnd[2 * r: 2 * r + 2] for r in range(G)]
    return [[rnd[r]] for r in range(G)]


def train_tournament(g: Graph, M, cfg: TrainConfig, e_i: int, batch_size: int = 5,
                     rng_stream: int = 0, group=None, num_ranks: int | None = None,
                     pair_fn: PairFn | None = None, gather: bool = True) -> dict:
    """Part-pair training of the level (g, M) for an e_i-epoch budget,
    sharded over the ranks of `group` (torch.distributed; NCCL on GPUs), or
    over `num_ranks` virtual ranks in this process when no process group is
    initialised.  M is the full matrix, identical on every rank (CUDA
    tensor, or numpy/CPU tensor staged to the rank's device); with gather
    the trained matrix is written back into M on every rank.

    pair_fn overrides the pair step (tests substitute a CPU checker to run
    the schedule and exchange over gloo); the default is the device kernel.
    Returns a stats dict in train_large's shape plus the exchange volume."""
    cfg.validate()
    if M.shape[0] != g.num_vertices:
        raise ValueError("matrix rows must match vertex count")
    import torch.distributed as dist
    distributed = dist.is_available() and dist.is_initialized()
    if distributed:
        G, rank = dist.get_world_size(group), dist.get_rank(group)
    else:
        G, rank = (num_ranks or 1), -1
    if G < 1:
        raise ConfigError("num_ranks must be >= 1")
    K, B, V, d = 2 * G, batch_size, M.shape[0], M.shape[1]
    if V < K:
        raise ConfigError(f"{V} rows cannot be split into {K} parts")
    plan = PartitionPlan(K=K, boundaries=(np.arange(K + 1, dtype=np.int64) * V) // K)
    rotations = tournament_rotations(g, cfg, e_i, K, B)
    rounds = tournament_rounds(K)
    index = pair_index(K)
    P = len(index)
    moves = shift_moves(K)
    status = None
    # virtual ranks on one GPU: each rank's pairs go to their own stream (the
    # pairs of a round touch disjoint parts, as on G GPUs), joined once per
    # round before the exchange.  Only small parts gain (C2, d=128: 32 MiB
    # parts 3.14 -> 5.80 G upd/s; 64 MiB parts equal at d=128, -20% at
    # d=256; 128 MiB parts -10%): GB_VIRTUAL_STREAMS auto (parts under
    # 48 MiB) / 1 / 0
    streams = None
    vs = os.environ.get("GB_VIRTUAL_STREAMS", "auto")
    if vs not in ("auto", "0", "1"):
        raise ConfigError(f"GB_VIRTUAL_STREAMS={vs!r}: expected auto, 0 or 1")
    if pair_fn is None:
        pair_fn, status = device_pair_fn(g, cfg, B, K)
        device = torch.device("cuda", torch.cuda.current_device())
        if not distributed and G > 1 and (
                vs == "1" or (vs == "auto" and plan.max_rows * d * 4 < 48 << 20)):
            streams = [torch.cuda.Stream(device) for _ in range(G)]
            rank_fns = [pair_fn] + [device_pair_fn(g, cfg, B, K, status)[0]
                                    for _ in range(G - 1)]
    else:
        device = M.device if isinstance(M, torch.Tensor) else torch.device("cpu")
    Mt = M if isinstance(M, torch.Tensor) else torch.from_numpy(M)
    if Mt.dtype != torch.float32:
        raise TypeError("embedding matrix must be float32")

    my_ranks = [rank] if distributed else list(range(G))
    parts = {r: _RankParts(plan.max_rows, d, device) for r in my_ranks}
    arr0 = initial_arrangement(K)
    for r in my_ranks:
        for slot, part in enumerate(holdings(arr0)[r]):
            lo, hi = plan.part_range(part)
            parts[r].cur[slot][: hi - lo].copy_(Mt[lo:hi], non_blocking=True)

    sent_bytes, n_pairs = 0, 0
    t0 = time.perf_counter()
    main = torch.cuda.current_stream(device) if streams else None
    for rot in range(rotations):
        lr = lr_at(cfg.learning_rate, rot, rotations)
        arr = initial_arrangement(K)
        for ri, rnd in enumerate(rounds):
            diagonal = ri == 0
            hold = holdings(arr)
            per_rank = _steps_for_round(rnd, G, diagonal)
            for r in my_ranks:
                if streams:
                    streams[r].wait_stream(main)
                    pair_fn = rank_fns[r]
                for a, b in per_rank[r]:
                    slot_of = {hold[r][TOP]: TOP, hold[r][BOT]: BOT}
                    Ma = parts[r].cur[slot_of[a]]
                    Mb = Ma if a == b else parts[r].cur[slot_of[b]]
                    lo_a, hi_a = plan.part_range(a)
                    lo_b, hi_b = plan.part_range(b)
                    seed = _derived_seed(cfg.seed, rng_stream, rot * P + index[(a, b)])
                    step = PairStep(a, b, lo_a, hi_a, lo_b, hi_b, seed, lr)
                    if streams:
                        with torch.cuda.stream(streams[r]):
                            pair_fn(Ma[: hi_a - lo_a], Mb[: hi_b - lo_b], step)
                    else:
                        pair_fn(Ma[: hi_a - lo_a], Mb[: hi_b - lo_b], step)
                    n_pairs += 1
            if streams:
                for st_r in streams:
                    main.wait_stream(st_r)
            if not diagonal and K > 2:
                if distributed:
                    sent_bytes += _exchange_dist(parts[rank], rank, moves, group)
                else:
                    _exchange_virtual([parts[r] for r in my_ranks], moves)
                    sent_bytes += sum(plan.max_rows * d * 4 for sr, _, dr, _ in moves
                                      if sr != dr)
                arr = shift(arr)
    if device.type == "cuda":
        torch.cuda.current_stream(device).synchronize()
    train_s = time.perf_counter() - t0

    pos_local = neg_local = 0
    if status is not None:
        st = status.cpu().tolist()
        if st[0]:
            raise FloatingPointError("non-finite embedding after tournament training")
        pos_local, neg_local = int(st[2]), int(st[3])
    else:  # checker pair_fn: the reference's pools, n_neg negatives per positive
        neg_local = pos_local * cfg.negative_samples
    pos, neg = pos_local, neg_local
    if distributed:
        t = torch.tensor([pos_local, neg_local, n_pairs, sent_bytes], dtype=torch.int64,
                         device=device if dist.get_backend(group) == "nccl" else "cpu")
        dist.all_reduce(t, group=group)
        pos, neg, n_pairs, sent_bytes = (int(x) for x in t.tolist())

    if gather:
        _gather(Mt, parts, plan, G, rank, distributed, group, device)
        if not isinstance(M, torch.Tensor):
            M[...] = Mt.numpy()
        if not bool(torch.isfinite(Mt).all()):
            raise FloatingPointError("non-finite embedding after tournament training")
    return {
        "rotations": rotations,
        "K": K,
        "ranks": G,
        "rounds_per_rotation": len(rounds),
        "pairs": n_pairs,
        "pos_updates": pos,
        "neg_updates": neg,
        "exchange_bytes": sent_bytes,
        "train_s": train_s,
    }


def _gather(Mt: torch.Tensor, parts, plan: PartitionPlan, G: int, rank: int, distributed: bool,
            group, device) -> None:
    """Write every part back into the full matrix on every rank (the
    arrangement is the initial one again after a whole rotation)."""
    hold = holdings(initial_arrangement(plan.K))
    if distributed:
        import torch.distributed as dist
        mine = torch.stack(parts[rank].cur)
        if dist.get_backend(group) != "nccl" and mine.is_cuda:
            mine = mine.cpu()
        bufs = [torch.empty_like(mine) for _ in range(G)]
        dist.all_gather(bufs, mine, group=group)
        src = {r: bufs[r] for r in range(G)}
    else:
        src = {r: parts[r].cur for r in range(G)}
    for r in range(G):
        for slot, part in enumerate(hold[r]):
            lo, hi = plan.part_range(part)
            Mt[lo:hi].copy_(src[r][slot][: hi - lo])


def sequential_order(K: int, rotations: int):
    """The pair sequence a single device would run for the same schedule:
    (rotation, pair) in tournament order.  Used by the tests as the
    equivalence target."""
    out = []
    for rot in range(rotations):
        for rnd in tournament_rounds(K):
            for pr in rnd:
                out.append((rot, pr))
    return out


def train_multilevel_sharded(g0: Graph, cfg: TrainConfig, threshold: int = 100,
                             shard_levels: int = 1, batch_size: int = 5, group=None,
                             num_ranks: int | None = None, hierarchy=None,
                             return_device: bool = False, balanced_pools: bool = True):
    """train_multilevel (trainer.py:252-288) with the finest `shard_levels`
    levels trained by the tournament across ranks.  Every rank coarsens
    (the device collapse is deterministic, so the hierarchies are identical
    with no communication); the coarse levels train on rank 0 and the matrix
    is broadcast before the first sharded level.  Returns
    (matrix, per-level stats).

    balanced_pools (default; Hogwild runs only): the sharded levels draw
    balanced pools (TrainConfig.balanced_pools), which keeps this path's
    AUCROC at the in-memory pass's (C3: 0.823-0.829 vs 0.826) where the
    reference's fixed-B pools of train_large lose 0.04;
    False keeps the reference's pools."""
    from .coarsen import coarsen_all
    from .trainer import epoch_plan, expand_embedding, init_embedding, train_level
    import torch.distributed as dist
    cfg.validate()
    if balanced_pools and not cfg.deterministic and not cfg.balanced_pools:
        cfg = dataclasses.replace(cfg, balanced_pools=True)
    distributed = dist.is_available() and dist.is_initialized()
    rank = dist.get_rank(group) if distributed else 0
    if hierarchy is None:
        hierarchy = coarsen_all(g0, threshold=threshold)
    depth = hierarchy.depth
    # total_epochs == 0: the random-projection baseline, like train_multilevel
    plan = (np.zeros(depth, dtype=np.int64) if cfg.total_epochs == 0
            else epoch_plan(cfg.total_epochs, cfg.smoothing_ratio, depth).per_level)
    _lib.require_cuda()
    M = torch.from_numpy(init_embedding(hierarchy.graphs[-1].num_vertices, cfg.dim,
                                        cfg.seed)).cuda()
    stats = []
    broadcast_done = False
    for i in range(depth - 1, -1, -1):
        g_i = hierarchy.graphs[i]
        e_i = int(plan[i])
        sharded = i < shard_levels and g_i.num_vertices >= 2 * (
            dist.get_world_size(group) if distributed else (num_ranks or 1))
        t0 = time.perf_counter()
        if sharded and e_i > 0:
            if distributed and not broadcast_done:
                dist.broadcast(M, 0, group=group)
                broadcast_done = True
            st = train_tournament(g_i, M, cfg, e_i, batch_size=batch_size, rng_stream=i,
                                  group=group, num_ranks=num_ranks)
            entry = {"level": i, "sharded": True, **st}
        else:
            entry = {"level": i, "sharded": False, "passes": 0, "updates": 0}
            if rank == 0 and e_i > 0:
                ts = train_level(g_i, M, cfg, e_i, rng_stream=i)
                entry.update(passes=ts.passes, updates=ts.updates)
        torch.cuda.synchronize()
        entry["s"] = time.perf_counter() - t0
        stats.append(entry)
        if i > 0:
            M = expand_embedding(M, hierarchy.mappings[i - 1])
    if distributed and not broadcast_done:
        dist.broadcast(M, 0, group=group)
    return (M if return_device else M.cpu().numpy()), stats
