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
from .errors import ConfigError, PlanError
from .graph import Graph
from .trainer import TrainConfig, _train_flags, lr_at

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


def round_lr(lr0: float, rot: int, ri: int, rotations: int, K: int, epochs: int) -> float:
    """Learning rate of round ri of rotation rot of a level trained for
    `epochs` epochs: the in-memory rate of the epoch that round's share of
    the level's work falls in, lr_at(lr0, j, epochs) with
    j = floor((rot * K + ri) * epochs / (rotations * K)) (trainer.py:179-181,
    one rate per epoch, edge-scaled epochs being ceil(E/V) passes at one
    rate).  (train_large decays per rotation, bigtrain.py:432; with the one
    or two rotations that CLI-default budgets give a level, that keeps lr
    near lr0 for the whole level and the sharded AUCROC drifts well above the
    in-memory path's.  Decaying per round regardless of epochs instead halved
    the mean rate of a one-epoch edge-scaled level, whose in-memory passes
    all run at lr0.)"""
    j = ((rot * K + ri) * epochs) // max(rotations * K, 1)
    return lr_at(lr0, j, max(epochs, 1))


def pair_rounds(K: int) -> dict[tuple[int, int], int]:
    """Round index of each pair within a rotation."""
    return {pr: ri for ri, rnd in enumerate(tournament_rounds(K)) for pr in rnd}


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
    param: int | None = None  # device {seed, lr} (CUDA-graph rotations)


PairFn = Callable[[torch.Tensor, torch.Tensor, PairStep], None]


class DevicePair:
    """Pair step on the GPU: side 2 then side 3 (bigtrain.py:241-260) through
    bigtrain.PairSides, split into prepare (the pools: they depend only on the
    replicated CSR and the part ranges) and train (the pair kernels on the two
    part buffers), with named pool buffer sets so the next round's pools are
    drawn while the parts are still in flight between ranks."""

    def __init__(self, g: Graph, cfg: TrainConfig, B: int, K: int = 1,
                 status: torch.Tensor | None = None):
        _lib.require_cuda()
        flags = _train_flags(cfg, pair=True)
        self.status = status if status is not None else _lib.new_status()
        self.sides = PairSides(g.device_csr(), cfg, flags, B, self.status, K=K)

    def prepare(self, s: PairStep, tag: str = "0") -> None:
        if s.hi_a - s.lo_a <= 0 or s.hi_b - s.lo_b <= 0:
            return
        self.sides.prepare(s.lo_a, s.hi_a, s.lo_b, s.hi_b, s.seed, 0, tag + "a", s.param)
        if s.a != s.b:
            self.sides.prepare(s.lo_b, s.hi_b, s.lo_a, s.hi_a, s.seed, 1, tag + "b", s.param)

    def train(self, Ma: torch.Tensor, Mb: torch.Tensor, s: PairStep, tag: str = "0") -> None:
        if s.hi_a - s.lo_a <= 0 or s.hi_b - s.lo_b <= 0:
            return
        self.sides.train(Ma, Mb, s.lo_a, s.hi_a, s.lo_b, s.hi_b, s.seed, s.lr, 0, 2, tag + "a",
                         s.param)
        if s.a != s.b:
            self.sides.train(Mb, Ma, s.lo_b, s.hi_b, s.lo_a, s.hi_a, s.seed, s.lr, 1, 3,
                             tag + "b", s.param)

    def __call__(self, Ma: torch.Tensor, Mb: torch.Tensor, s: PairStep) -> None:
        self.prepare(s, "x")
        self.train(Ma, Mb, s, "x")


def device_pair_fn(g: Graph, cfg: TrainConfig, B: int, K: int = 1,
                   status: torch.Tensor | None = None) -> tuple[DevicePair, torch.Tensor]:
    """(pair step, status block); each step owns its pool scratch, so steps
    made with a shared status may run on different streams at once."""
    fn = DevicePair(g, cfg, B, K, status)
    return fn, fn.status


# ---------------------------------------------------------------------------
# part storage: a level's matrix as the parts this process holds
# ---------------------------------------------------------------------------
def init_embedding_rows(num_rows: int, dim: int, seed: int, lo: int, hi: int) -> np.ndarray:
    """Rows [lo, hi) of init_embedding(num_rows, dim, seed) (trainer.py:87-93)
    without drawing the others: numpy's uniform() consumes one PCG64 output
    per value in row-major order, so the generator is advanced by lo*dim
    outputs.  Bit-identical to the slice of the full draw."""
    from .errors import ConfigError as _CE
    if num_rows < 1 or dim < 1:
        raise _CE("embedding dimensions must be positive")
    bound = 0.5 / dim
    bg = np.random.PCG64(seed)
    bg.advance(lo * dim)
    return np.random.Generator(bg).uniform(-bound, bound, size=(hi - lo, dim)).astype(np.float32)


class PartStore:
    """One level's embedding matrix as the parts this process holds.

    parts[r][slot] is the part id held in slot TOP/BOT by local rank r (one
    rank per process under torch.distributed, every virtual rank otherwise)
    and data[part] its rows, a (max_rows, d) buffer.  A process therefore
    holds 2 parts per local rank (+ 2 receive twins with real ranks): 2|M|/G
    per GPU, never the whole matrix (C5's 256 GiB matrix over
    8 GPUs).

    Host mode (`host=True`): the buffers are pinned host memory and a pair's
    two parts are staged through device slots on a copy stream -- the
    per-rank form of train_large's residency (bigtrain.py:263-340) for parts
    that exceed the per-GPU budget.  The next local rank's parts load while
    the current pair trains; trained parts flush back behind it."""

    def __init__(self, V: int, d: int, G: int, local_ranks: list[int], device,
                 host: bool = False):
        self.V, self.d, self.G = V, d, G
        self.K = 2 * G
        self.plan = PartitionPlan(K=self.K,
                                  boundaries=(np.arange(self.K + 1, dtype=np.int64) * V) // self.K)
        self.local = list(local_ranks)
        self.device = torch.device(device)
        self.host = bool(host)
        hold = holdings(initial_arrangement(self.K))
        self.parts = {r: list(hold[r]) for r in self.local}
        self.data: dict[int, torch.Tensor] = {}
        for r in self.local:
            for p in self.parts[r]:
                self.data[p] = self._alloc()
        self.spare: list[torch.Tensor] = []  # receive twins (real ranks)
        self._stage = None

    def _alloc(self) -> torch.Tensor:
        if self.host:
            return torch.zeros((self.plan.max_rows, self.d), dtype=torch.float32).pin_memory()
        return torch.zeros((self.plan.max_rows, self.d), dtype=torch.float32, device=self.device)

    @property
    def device_bytes(self) -> int:
        """HBM held for parts (the C5 budget figure): part buffers, receive
        twins and staging slots."""
        row = self.plan.max_rows * self.d * 4
        n = 0 if self.host else len(self.data) + len(self.spare)
        if self._stage is not None:
            n += len(self._stage.slots)
        return n * row

    def rows(self, part: int) -> tuple[int, int]:
        return self.plan.part_range(part)

    def local_parts(self):
        """(part, lo, hi, buffer rows) of every part this process holds."""
        self.drain()
        for r in self.local:
            for p in self.parts[r]:
                lo, hi = self.rows(p)
                yield p, lo, hi, self.data[p][: hi - lo]

    # -- filling ---------------------------------------------------------------
    def load_full(self, Mt: torch.Tensor) -> None:
        from ._staging import copy_numpy_to_device
        for p, lo, hi, buf in self.local_parts():
            if Mt.device.type == "cpu" and buf.is_cuda and not Mt.is_pinned():
                copy_numpy_to_device(buf[: hi - lo], Mt[lo:hi].numpy())  # pinned chunks
            else:
                buf.copy_(Mt[lo:hi], non_blocking=True)

    def init_random(self, seed: int) -> None:
        """init_embedding(V, d, seed) restricted to the held rows."""
        for p, lo, hi, buf in self.local_parts():
            buf.copy_(torch.from_numpy(init_embedding_rows(self.V, self.d, seed, lo, hi)))

    def expand_from(self, coarse: torch.Tensor, mapping) -> None:
        """Row v of this level = row map[v] of the (replicated) coarser
        matrix (trainer.py:243-249), gathered straight into the held parts:
        the fine matrix is never materialised whole."""
        cmap = mapping.device_map()
        tmp = None
        for p, lo, hi, buf in self.local_parts():
            dst = buf
            if self.host:
                tmp = tmp if tmp is not None else torch.empty(
                    (self.plan.max_rows, self.d), dtype=torch.float32, device=coarse.device)
                dst = tmp[: hi - lo]
            _lib.call("gb_expand", _lib.ptr(coarse), coarse.shape[0], self.d,
                      cmap.data_ptr() + lo * cmap.element_size(), hi - lo, _lib.ptr(dst),
                      _lib.stream())
            if self.host:
                buf.copy_(dst)

    # -- output ------------------------------------------------------------------
    def to_full(self, out: torch.Tensor | None = None, group=None, distributed: bool = False,
                device=None) -> torch.Tensor:
        """The whole matrix on every rank (all_gather of the parts; only at the
        initial arrangement, i.e. between rotations)."""
        dev = device if device is not None else self.device
        self.drain()
        if out is None:
            out = torch.empty((self.V, self.d), dtype=torch.float32, device=dev)
        hold = holdings(initial_arrangement(self.K))
        if distributed:
            import torch.distributed as dist
            m = len(self.local)
            mine = torch.stack([self.data[p] for r in self.local for p in self.parts[r]])
            nccl = dist.get_backend(group) == "nccl"
            mine = mine.to(self.device if nccl else "cpu")
            bufs = [torch.empty_like(mine) for _ in range(self.G // m)]
            dist.all_gather(bufs, mine, group=group)
            for rr in range(self.G):
                for slot, p in enumerate(hold[rr]):
                    lo, hi = self.rows(p)
                    out[lo:hi].copy_(bufs[rr // m][2 * (rr % m) + slot][: hi - lo])
        else:
            from ._staging import copy_device_to_numpy
            for p, lo, hi, buf in self.local_parts():
                if out.device.type == "cpu" and buf.is_cuda and not out.is_pinned():
                    copy_device_to_numpy(out[lo:hi].numpy(), buf[: hi - lo])
                else:
                    out[lo:hi].copy_(buf)
        return out

    # -- pair views ----------------------------------------------------------------
    def begin_round(self, order: list[tuple[int, list[tuple[int, int]]]]) -> None:
        """Host mode: stage the first local rank's parts of a round."""
        if self.host:
            if self._stage is None:
                self._stage = _SlotStager(self)
            self._stage.begin(order)

    def pair_views(self, r: int, a: int, b: int) -> tuple[torch.Tensor, torch.Tensor]:
        if self.host:
            return self._stage.views(r, a, b)
        lo_a, hi_a = self.rows(a)
        lo_b, hi_b = self.rows(b)
        Ma = self.data[a][: hi_a - lo_a]
        return Ma, (Ma if a == b else self.data[b][: hi_b - lo_b])

    def end_pair(self, r: int) -> None:
        if self.host:
            self._stage.done(r)

    def end_round(self) -> None:
        """Nothing to wait for: the next round's loads queue behind this
        round's flushes on the copy stream."""

    # -- exchange --------------------------------------------------------------
    def shift(self, moves, arr: list[int], group=None, per_process: int = 0,
              before_wait: Callable[[], None] | None = None) -> int:
        """One circle shift (arrangement `arr` before it).  Moves between
        ranks of this process relabel parts; with torch.distributed
        (per_process = virtual ranks per process) a move to another process
        is an NCCL (gloo on CPU) send/recv of one part, received into a spare
        twin -- at most two sends and two receives per process, to its
        neighbours.  `before_wait` runs after the transfers are posted (the
        next round's pool draws overlap them).  Returns the bytes that left
        a GPU (virtual ranks: that would have)."""
        hold = holdings(arr)
        local = set(self.local)
        new = {r: list(self.parts[r]) for r in self.local}
        row_bytes = self.plan.max_rows * self.d * 4
        ops, sent, gone, arrived = [], 0, [], []
        m = per_process
        if m:
            import torch.distributed as dist
            self.drain()
        # gloo moves host tensors only: with device parts (one GPU shared by
        # test processes) the transfers are staged through host copies
        wire = (torch.device("cpu") if m and self.device.type == "cuda"
                and dist.get_backend(group) == "gloo" else self.device)
        for sr, ss, dr, ds in moves:
            part = hold[sr][ss]
            if sr in local and dr in local:
                new[dr][ds] = part
                if not m and sr != dr:
                    sent += row_bytes
            elif sr in local:
                buf = self.data[part]
                if buf.device != wire:  # host parts to HBM (NCCL); device parts to host (gloo)
                    buf = buf.to(wire)
                ops.append(dist.P2POp(dist.isend, buf, dr // m, group))
                sent += buf.numel() * buf.element_size()
                gone.append(part)
            elif dr in local:
                if not self.spare:
                    self.spare.append(self._alloc())
                buf = self.spare.pop()
                rbuf = buf if buf.device == wire else torch.empty(buf.shape, dtype=buf.dtype,
                                                                  device=wire)
                ops.append(dist.P2POp(dist.irecv, rbuf, sr // m, group))
                arrived.append((part, buf, rbuf))
                new[dr][ds] = part
        works = dist.batch_isend_irecv(ops) if ops else []
        if before_wait is not None:
            before_wait()
        for w in works:
            w.wait()
        for part in gone:
            self.spare.append(self.data.pop(part))
        for part, buf, rbuf in arrived:
            if rbuf is not buf:
                buf.copy_(rbuf)
            self.data[part] = buf
        self.parts = new
        return sent

    def drain(self) -> None:
        """Host mode: wait for outstanding flushes of trained parts."""
        if self._stage is not None:
            self._stage.drain()


class _SlotStager:
    """Host-mode residency of a PartStore: two pairs of device slots, one copy
    stream.  While local rank r trains in one slot pair, rank r+1's parts load
    into the other; a pair's parts flush back to their pinned host buffers
    behind its kernels (event-ordered), so PCIe copies overlap compute."""

    def __init__(self, store: PartStore):
        self.store = store
        shape = (store.plan.max_rows, store.d)
        self.slots = [torch.empty(shape, dtype=torch.float32, device=store.device)
                      for _ in range(4)]
        self.copy = torch.cuda.Stream(store.device)
        self.order: list = []
        self.loaded: dict[int, tuple[int, torch.cuda.Event, dict]] = {}
        self.prefetched: set[int] = set()

    def _load(self, idx: int) -> None:
        r, pairs = self.order[idx]
        base = 2 * (idx % 2)
        parts = list(dict.fromkeys(p for pr in pairs for p in pr))
        where = {}
        compute = torch.cuda.current_stream(self.store.device)
        fence = torch.cuda.Event()
        fence.record(compute)  # the slot pair's previous kernels are queued before this
        self.copy.wait_event(fence)
        with torch.cuda.stream(self.copy):
            for k, p in enumerate(parts):
                lo, hi = self.store.rows(p)
                self.slots[base + k][: hi - lo].copy_(self.store.data[p][: hi - lo],
                                                      non_blocking=True)
                where[p] = base + k
        ev = torch.cuda.Event()
        ev.record(self.copy)
        self.loaded[r] = (idx, ev, where)

    def begin(self, order) -> None:
        self.order = list(order)
        self.loaded = {}
        self.prefetched = set()
        if self.order:
            self._load(0)

    def views(self, r: int, a: int, b: int):
        idx, ev, where = self.loaded[r]
        torch.cuda.current_stream(self.store.device).wait_event(ev)
        if idx + 1 < len(self.order) and idx + 1 not in self.prefetched:
            self.prefetched.add(idx + 1)
            self._load(idx + 1)  # prefetch the next rank behind this one's kernels
        lo_a, hi_a = self.store.rows(a)
        lo_b, hi_b = self.store.rows(b)
        Ma = self.slots[where[a]][: hi_a - lo_a]
        return Ma, (Ma if a == b else self.slots[where[b]][: hi_b - lo_b])

    def done(self, r: int) -> None:
        idx, _, where = self.loaded.pop(r)
        compute = torch.cuda.current_stream(self.store.device)
        trained = torch.cuda.Event()
        trained.record(compute)
        self.copy.wait_event(trained)
        with torch.cuda.stream(self.copy):
            for p, sl in where.items():
                lo, hi = self.store.rows(p)
                self.store.data[p][: hi - lo].copy_(self.slots[sl][: hi - lo], non_blocking=True)
        # the slot pair is reused two ranks later: its next load waits on the
        # compute stream (fence in _load) and runs after this flush (same stream)

    def drain(self) -> None:
        self.copy.synchronize()


# ---------------------------------------------------------------------------
# driver
# ---------------------------------------------------------------------------
def _steps_for_round(rnd: list[tuple[int, int]], G: int, diagonal: bool):
    if diagonal:
        return [rnd[2 * r: 2 * r + 2] for r in range(G)]
    return [[rnd[r]] for r in range(G)]


# Captured rotations, keyed by everything a replay bakes in: the CSR and part
# buffer addresses, sizes, flags and layout.  A later call whose key matches
# (the next bench step, the next call on the same PartStore) replays without
# an eager rotation or a capture.  One entry: the cache keeps the pair steps'
# pool buffers alive.
_ROTATION_GRAPHS: dict = {}


def clear_rotation_graphs() -> None:
    """Drop the cached rotation graph (and the pool buffers it holds)."""
    _ROTATION_GRAPHS.clear()


def _graph_key(g: Graph, store: "PartStore", cfg: TrainConfig, B: int, streams: bool):
    x, a = g.device_csr()
    bufs = tuple((p, store.data[p].data_ptr()) for r in store.local for p in store.parts[r])
    return (str(store.device), g.num_vertices, g.num_edges, x.data_ptr(), a.data_ptr(),
            store.V, store.d, store.G, tuple(store.local), bufs, streams, B,
            cfg.dim, cfg.negative_samples, _train_flags(cfg, pair=True), cfg.balanced_pools,
            cfg.max_inflight,
            os.environ.get("GB_POOL_MODE", "compact"))


def _world(group, num_ranks, per_process: int = 1):
    """(distributed, G ranks of the schedule, this process's ranks).  Under
    torch.distributed each process runs `per_process` consecutive ranks of
    the schedule (K = 2 * world * per_process parts); otherwise all
    `num_ranks` are virtual ranks of this process."""
    import torch.distributed as dist
    if per_process < 1:
        raise ConfigError("per_process must be >= 1")
    distributed = dist.is_available() and dist.is_initialized()
    if distributed:
        world, rank = dist.get_world_size(group), dist.get_rank(group)
        G = world * per_process
        return True, G, list(range(rank * per_process, (rank + 1) * per_process))
    G = num_ranks or 1
    if G < 1:
        raise ConfigError("num_ranks must be >= 1")
    return False, G, list(range(G))


def train_tournament_parts(g: Graph, store: PartStore, cfg: TrainConfig, e_i: int,
                           batch_size: int = 5, rng_stream: int = 0, group=None,
                           pair_fn: PairFn | None = None,
                           exchange_events: list | None = None) -> dict:
    """Part-pair training of the level (g, parts in `store`) for an e_i-epoch
    budget.  Each rotation: a diagonal round, then K-1 off-diagonal rounds of
    one pair per rank with a circle shift between rounds.  Between real ranks
    the shift is posted as P2P transfers and the next round's pools are drawn
    while they are in flight; virtual ranks relabel parts and run their pairs
    on one stream each.  Returns train_large's stats plus exchange volume.
    exchange_events, if given, collects (start, end) CUDA events around each
    shift on the compute stream: the exposed (not overlapped) exchange time."""
    cfg.validate()
    if cfg.similarity != "adjacency":
        raise ConfigError("part-pair training draws adjacency positives from its pools "
                          f"(bigtrain.py:164-212); similarity={cfg.similarity!r} needs the "
                          "in-memory path")
    import torch.distributed as dist
    distributed = dist.is_available() and dist.is_initialized() and len(store.local) < store.G
    per_process = len(store.local) if distributed else 0
    G, K, B = store.G, store.K, batch_size
    plan = store.plan
    rotations = tournament_rotations(g, cfg, e_i, K, B)
    rounds = tournament_rounds(K)
    index = pair_index(K)
    P = len(index)
    moves = shift_moves(K)
    rnd_of = pair_rounds(K)
    pairs_by_index = [pr for pr, _ in sorted(index.items(), key=lambda kv: kv[1])]
    vs = os.environ.get("GB_VIRTUAL_STREAMS", "auto")
    if vs not in ("auto", "0", "1"):
        raise ConfigError(f"GB_VIRTUAL_STREAMS={vs!r}: expected auto, 0 or 1")
    status = None
    streams = None
    on_gpu = pair_fn is None
    if on_gpu:
        first, status = device_pair_fn(g, cfg, B, K)
        fns = {r: first for r in store.local}
        # virtual ranks: each rank's pairs on their own stream (the pairs of
        # a round touch disjoint parts, as on G GPUs), joined once per round.
        # Only small parts gain (C2, d=128: 32 MiB parts 3.14 -> 5.80 G upd/s;
        # 64 MiB equal; 128 MiB -10%): GB_VIRTUAL_STREAMS auto (< 48 MiB) / 1 / 0
        if not distributed and G > 1 and not store.host and (
                vs == "1" or (vs == "auto" and plan.max_rows * store.d * 4 < 48 << 20)):
            streams = {r: torch.cuda.Stream(store.device) for r in store.local}
            fns = {r: device_pair_fn(g, cfg, B, K, status)[0] for r in store.local}
    has_prepare = on_gpu
    cached = None
    rg0 = os.environ.get("GB_ROTATION_GRAPH", "auto")
    if (has_prepare and rg0 != "0" and not distributed and not store.host and
            exchange_events is None and first.sides.mode != "fused"):
        key = _graph_key(g, store, cfg, B, streams is not None)
        cached = _ROTATION_GRAPHS.get(key)
        if cached is not None and cached["P"] == len(pair_index(K)):
            fns, status = cached["fns"], cached["status"]
            status.copy_(_lib.new_status())
        else:
            cached = None

    # CUDA-graph rotations (one process holding every rank on the device):
    # a rotation is the same launch sequence each time -- the circle shifts
    # relabel parts and return to the initial arrangement after K-1 rounds --
    # except for the pairs' seeds and lr, which the *_dp kernels read from a
    # device table.  Rotation 0 runs eagerly (allocating every pool buffer),
    # the next is captured once, and each later rotation is one table upload
    # + one replay: the host's ~2 launches per pair side leave the path.
    # GB_ROTATION_GRAPH: auto (>= 16 rotations: capture + instantiate cost
    # ~2 eager rotations, a replay saves ~12% of one at K=16 on the C2 graph,
    # profiles/r02_rotation_graph_phases.jsonl), 1 (from 2 rotations), 0 (off)
    rg = os.environ.get("GB_ROTATION_GRAPH", "auto")
    if rg not in ("auto", "0", "1"):
        raise ConfigError(f"GB_ROTATION_GRAPH={rg!r}: expected auto, 0 or 1")
    use_graph = cached is not None or (
        has_prepare and not distributed and not store.host and
        exchange_events is None and first.sides.mode != "fused" and
        rotations >= (2 if rg == "1" else 16) and rg != "0")
    ptab = None
    if use_graph:
        if cached is not None:
            ptab, hbuf = cached["ptab"], cached["hbuf"]
        else:
            ptab = torch.zeros((P, 2), dtype=torch.int64, device=store.device)
            hbuf = [torch.zeros((P, 2), dtype=torch.int64).pin_memory() for _ in range(2)]
        hev: list = [None, None]

        def upload(rot):
            k = rot % 2
            if hev[k] is not None:
                hev[k].synchronize()  # the previous copy out of this buffer is done
            h = hbuf[k].numpy()
            seeds = np.array([_lib.u64(_derived_seed(cfg.seed, rng_stream, rot * P + q))
                              for q in range(P)], dtype=np.uint64)
            h[:, 0] = seeds.view(np.int64)
            h[:, 1] = np.array([round_lr(cfg.learning_rate, rot, rnd_of[pr], rotations, K, e_i)
                                for pr in pairs_by_index], dtype=np.float64).view(np.int64)
            ptab.copy_(hbuf[k], non_blocking=True)
            ev = torch.cuda.Event()
            ev.record()
            hev[k] = ev

    sent_bytes, n_pairs = 0, 0
    t0 = time.perf_counter()
    main0 = torch.cuda.current_stream(store.device) if store.device.type == "cuda" else None

    def round_steps(rot, ri, arr):
        diagonal = ri == 0
        per_rank = _steps_for_round(rounds[ri], G, diagonal)
        out = []
        for r in store.local:
            lst = []
            for k, (a, b) in enumerate(per_rank[r]):
                lo_a, hi_a = plan.part_range(a)
                lo_b, hi_b = plan.part_range(b)
                seed = _derived_seed(cfg.seed, rng_stream, rot * P + index[(a, b)])
                prm = ptab.data_ptr() + 16 * index[(a, b)] if ptab is not None else None
                lst.append((k, PairStep(a, b, lo_a, hi_a, lo_b, hi_b, seed,
                                        round_lr(cfg.learning_rate, rot, ri, rotations, K, e_i),
                                        prm)))
            out.append((r, lst))
        return out

    # Pools are drawn a round ahead (own buffer set per round parity and
    # rank) when something can overlap them: the P2P shift between real
    # ranks, or the other virtual ranks' streams.  Virtual ranks on one
    # stream draw each pair's pools right before it (one shared buffer set).
    ahead = has_prepare and (distributed or streams is not None)

    def tag(ri, r, k):
        return f"{ri % 2}.{r}.{k}." if ahead else f"x.{k}."

    def prepare(steps, ri):
        if not ahead:
            return
        for r, lst in steps:
            ctx = torch.cuda.stream(streams[r]) if streams else _null()
            with ctx:
                if streams:
                    streams[r].wait_stream(steps_fn_main)
                for k, s in lst:
                    fns[r].prepare(s, tag(ri, r, k))

    def run_rotation(rot, main):
        """All rounds of one rotation; returns (pairs, bytes shifted)."""
        nonlocal steps_fn_main
        steps_fn_main = main
        pairs, sent = 0, 0
        arr = initial_arrangement(K)
        steps = round_steps(rot, 0, arr)
        prepare(steps, 0)
        for ri in range(len(rounds)):
            diagonal = ri == 0
            store.begin_round([(r, [(s.a, s.b) for _, s in lst]) for r, lst in steps])
            for r, lst in steps:
                ctx = torch.cuda.stream(streams[r]) if streams else _null()
                with ctx:
                    if streams:
                        streams[r].wait_stream(main)
                    for k, s in lst:
                        Ma, Mb = store.pair_views(r, s.a, s.b)
                        if has_prepare:
                            if not ahead:
                                fns[r].prepare(s, tag(ri, r, k))
                            fns[r].train(Ma, Mb, s, tag(ri, r, k))
                        else:
                            pair_fn(Ma, Mb, s)
                        pairs += 1
                    store.end_pair(r)
            if streams:
                for st_r in streams.values():
                    main.wait_stream(st_r)
            store.end_round()
            nxt = None
            if ri + 1 < len(rounds):
                arr_next = shift(arr) if not diagonal and K > 2 else arr
                nxt = round_steps(rot, ri + 1, arr_next)
            if not diagonal and K > 2:
                after = (lambda: prepare(nxt, ri + 1)) if nxt else None
                if exchange_events is not None and main is not None:
                    e0 = torch.cuda.Event(enable_timing=True)
                    e0.record(main)
                sent += store.shift(moves, arr, group, per_process=per_process,
                                    before_wait=after if per_process else None)
                if exchange_events is not None and main is not None:
                    e1 = torch.cuda.Event(enable_timing=True)
                    e1.record(main)
                    exchange_events.append((e0, e1))
                if not per_process and after:
                    after()
                arr = shift(arr)
            elif nxt:
                prepare(nxt, ri + 1)
            steps = nxt
        return pairs, sent

    steps_fn_main = main0
    trace = os.environ.get("GB_TRACE_ROTATIONS") == "1"
    phases: dict[str, float] = {}

    def mark(name, t_prev):
        if trace:
            torch.cuda.synchronize()
            t = time.perf_counter()
            phases[name] = phases.get(name, 0.0) + t - t_prev
            return t
        return t_prev

    def launches():
        return sum(f.sides.launches for f in {id(f): f for f in fns.values()}.values()) \
            if has_prepare else 0

    launches0 = launches()
    if cached is not None:
        # a replay per rotation (rotation 0 included): nothing is issued eagerly
        tp = time.perf_counter()
        graph = cached["graph"]
        for rot in range(rotations):
            upload(rot)
            graph.replay()
        mark("replays", tp)
        n_pairs = cached["pairs"] * rotations
        sent_bytes = cached["sent"] * rotations
        n_launches = cached["launches"] * rotations
    elif use_graph:
        tp = time.perf_counter()
        upload(0)
        pr, sb = run_rotation(0, main0)
        per_rotation = launches() - launches0
        tp = mark("eager_rotation", tp)
        # capture on a side stream with the bare capture API: torch.cuda.graph()
        # would also gc.collect() and empty the caching allocator on entry,
        # which costs more than the launches the graph saves
        graph = torch.cuda.CUDAGraph()
        cap = torch.cuda.Stream(store.device)
        cap.wait_stream(main0)
        with torch.cuda.stream(cap):
            graph.capture_begin(capture_error_mode="relaxed")
            try:
                run_rotation(1, cap)
            finally:
                graph.capture_end()
        main0.wait_stream(cap)
        tp = mark("capture", tp)
        for rot in range(1, rotations):
            upload(rot)
            graph.replay()
        mark("replays", tp)
        n_pairs, sent_bytes = pr * rotations, sb * rotations
        n_launches = per_rotation * rotations
        _ROTATION_GRAPHS.clear()
        _ROTATION_GRAPHS[_graph_key(g, store, cfg, B, streams is not None)] = {
            "graph": graph, "fns": fns, "status": status, "ptab": ptab, "hbuf": hbuf,
            "P": P, "pairs": pr, "sent": sb, "launches": per_rotation}
    else:
        for rot in range(rotations):
            pr, sb = run_rotation(rot, main0)
            n_pairs += pr
            sent_bytes += sb
        n_launches = launches() - launches0
    store.drain()
    if store.device.type == "cuda":
        torch.cuda.current_stream(store.device).synchronize()
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
                         device=store.device if dist.get_backend(group) == "nccl" else "cpu")
        dist.all_reduce(t, group=group)
        pos, neg, n_pairs, sent_bytes = (int(x) for x in t.tolist())
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
        "kernel_launches": n_launches,  # this process's fill + pair kernels
        "part_device_bytes": store.device_bytes,
        **({"phases_s": phases} if phases else {}),
    }


class _null:
    def __enter__(self):
        return self

    def __exit__(self, *exc):
        return False


def train_tournament(g: Graph, M, cfg: TrainConfig, e_i: int, batch_size: int = 5,
                     rng_stream: int = 0, group=None, num_ranks: int | None = None,
                     pair_fn: PairFn | None = None, gather: bool = True,
                     host_parts: bool = False, per_process: int = 1) -> dict:
    """Part-pair training of the level (g, M) for an e_i-epoch budget,
    sharded over the ranks of `group` (torch.distributed; NCCL on GPUs), or
    over `num_ranks` virtual ranks in this process when no process group is
    initialised.  M is the full matrix, identical on every rank (CUDA
    tensor, or numpy/CPU tensor); each rank copies only its two parts in,
    trains them (PartStore), and with gather the trained matrix is written
    back into M on every rank.  host_parts keeps the parts in pinned host
    memory, staged through device slots (budget mode); per_process runs that
    many consecutive schedule ranks in each process (K = 2 * world *
    per_process).

    pair_fn overrides the pair step (tests substitute a CPU checker to run
    the schedule and exchange over gloo); the default is the device kernel.
    Returns a stats dict in train_large's shape plus the exchange volume."""
    cfg.validate()
    if M.shape[0] != g.num_vertices:
        raise ValueError("matrix rows must match vertex count")
    distributed, G, local = _world(group, num_ranks, per_process)
    K, V, d = 2 * G, M.shape[0], M.shape[1]
    if V < K:
        raise ConfigError(f"{V} rows cannot be split into {K} parts")
    vs = os.environ.get("GB_VIRTUAL_STREAMS", "auto")
    if vs not in ("auto", "0", "1"):
        raise ConfigError(f"GB_VIRTUAL_STREAMS={vs!r}: expected auto, 0 or 1")
    if pair_fn is None:
        _lib.require_cuda()
        device = torch.device("cuda", torch.cuda.current_device())
    else:
        device = M.device if isinstance(M, torch.Tensor) else torch.device("cpu")
    Mt = M if isinstance(M, torch.Tensor) else torch.from_numpy(M)
    if Mt.dtype != torch.float32:
        raise TypeError("embedding matrix must be float32")
    store = PartStore(V, d, G, local, device, host=host_parts)
    store.load_full(Mt)
    st = train_tournament_parts(g, store, cfg, e_i, batch_size=batch_size,
                                rng_stream=rng_stream, group=group, pair_fn=pair_fn)
    if gather:
        store.to_full(out=Mt, group=group, distributed=distributed, device=Mt.device)
        if not isinstance(M, torch.Tensor) and not np.shares_memory(M, Mt.numpy()):
            M[...] = Mt.numpy()
        if not bool(torch.isfinite(Mt).all()):
            raise FloatingPointError("non-finite embedding after tournament training")
    return st


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


def shard_plan(num_rows: int, dim: int, world: int, budget_bytes: int,
               distributed: bool) -> tuple[int, int, bool]:
    """Ranks of the schedule and part placement for a level under a per-GPU
    byte budget for parts (MemoryBudget.resident_bytes): returns (G schedule
    ranks, ranks per process, host_parts).

    Device parts are preferred: a process holds 2 parts per schedule rank it
    runs (+ 2 receive twins with real ranks).  When that exceeds the budget
    the parts go to pinned host memory and only 4 device slots (+ twins)
    stay, and K = 2G grows until those fit -- bigtrain.plan_partitions'
    rule (bigtrain.py:133-149) applied per GPU."""
    def part(G):
        return -(-num_rows // (2 * G)) * dim * 4
    twins = 2 if distributed else 0
    G = world
    if (2 * (1 if distributed else world) + twins) * part(world) <= budget_bytes:
        return world, 1, False
    m = 1
    while (4 + twins) * part(world * m) > budget_bytes:
        if 2 * world * m >= num_rows:
            raise PlanError(f"budget {budget_bytes} B cannot hold 4 part slots of a "
                            f"{num_rows}-row level")
        m *= 2
    G = world * m
    return G, (m if distributed else G), True


def _level_batch(g: Graph, cfg: TrainConfig, e_i: int, K: int, B: int) -> int:
    """Positives per pair side for a level whose budget is under one
    rotation (see train_multilevel_sharded's adapt_batch)."""
    eff = e_i
    if cfg.epoch_unit == "edge-scaled" and g.num_edges > 0:
        eff = e_i * (-(-g.num_edges // g.num_vertices))
    return B if eff >= B * K else max(1, min(B, round(eff / K)))


def _broadcast(M: torch.Tensor, group) -> None:
    """rank 0's M to every rank (gloo: staged through the host)."""
    import torch.distributed as dist
    if M.is_cuda and dist.get_backend(group) == "gloo":
        h = M.cpu()
        dist.broadcast(h, 0, group=group)
        M.copy_(h)
    else:
        dist.broadcast(M, 0, group=group)


def train_multilevel_sharded(g0: Graph, cfg: TrainConfig, threshold: int = 100,
                             shard_levels: int = 1, batch_size: int = 5, group=None,
                             num_ranks: int | None = None, hierarchy=None,
                             return_device: bool = False, balanced_pools: bool = True,
                             return_parts: bool = False, host_parts: bool = False,
                             per_process: int = 1, budget=None, no_coarsen: bool = False,
                             adapt_batch: bool = True):
    """train_multilevel (trainer.py:252-288) with the finest `shard_levels`
    levels trained by the tournament across ranks.

    shard_levels=1 (default): the finest level only.  With each round at the
    in-memory rate of its epoch (round_lr) it stays closest to the in-memory
    ladder's AUCROC across the measured schedules (8 ranks; C3 vertex-pass
    +0.007, C3 edge-scaled -0.001, friendster shape vertex-pass -0.009; C1
    over 30 paired seeds +0.001 / +0.003 at 2 / 4 ranks); 2 / 3 levels
    project 2.5x / 3.9x instead of 1.4x on 8 GPUs for C3 edge-scaled but
    drift further (profiles/r02_sharded_epoch_lr.jsonl,
    r02_c3_shard_levels_round_decay.jsonl).

    Every rank coarsens (the device collapse is deterministic, so the
    hierarchies are identical with no communication).  Levels above the
    sharded ones are small: they train on rank 0 and the matrix is broadcast
    once.  The first sharded level is expanded from that matrix straight into
    each rank's two parts; a further sharded level all-gathers the coarser
    level's parts (the coarse matrix is ~5x smaller) and expands into its
    own parts.  So no rank ever holds a whole sharded level: per GPU the
    finest level costs 2|M|/G plus two receive twins (C5: 64 GiB of parts,
    or pinned host parts with `host_parts`).

    Returns (matrix, per-level stats); with return_parts the finest level
    stays sharded and the first element is its PartStore (rows per rank).

    budget (MemoryBudget): per-GPU bytes for the parts of the sharded levels
    (shard_plan) -- beyond it parts go to pinned host memory and K grows;
    the schedule is then planned from the finest level.

    adapt_batch (default): a level whose budget is below one rotation at
    batch_size B (eff < B*K pass-equivalents, e.g. the CLI's 200 vertex-pass
    epochs on a large graph) trains one rotation at B = max(1, round(eff/K))
    instead of B -- train_large's max(1, round(eff/(B*K))) would otherwise
    train it up to B*K/eff times its budget (friendster shape, 8 ranks:
    AUCROC 0.935 against the in-memory ladder's 0.629 on the same budget).

    balanced_pools (default; Hogwild runs only): the sharded levels draw
    balanced pools (TrainConfig.balanced_pools), which keeps this path's
    AUCROC at the in-memory pass's (C3: 0.823-0.829 vs 0.826) where the
    reference's fixed-B pools of train_large lose 0.04;
    False keeps the reference's pools."""
    from .coarsen import Hierarchy, coarsen_all
    from .trainer import epoch_plan, expand_embedding, init_embedding, train_level
    import torch.distributed as dist
    cfg.validate()
    if balanced_pools and not cfg.deterministic and not cfg.balanced_pools:
        cfg = dataclasses.replace(cfg, balanced_pools=True)
    if budget is not None and shard_levels > 0:
        world = dist.get_world_size(group) if (dist.is_available() and dist.is_initialized()) \
            else (num_ranks or 1)
        Gb, per_process, host_parts = shard_plan(
            g0.num_vertices if hierarchy is None else hierarchy.graphs[0].num_vertices,
            cfg.dim, world, budget.resident_bytes,
            dist.is_available() and dist.is_initialized())
        if not (dist.is_available() and dist.is_initialized()):
            num_ranks = Gb
    distributed, G, local = _world(group, num_ranks, per_process)
    rank = dist.get_rank(group) if distributed else 0
    if hierarchy is None:
        hierarchy = (Hierarchy(graphs=[g0], mappings=[]) if no_coarsen
                     else coarsen_all(g0, threshold=threshold))
    depth = hierarchy.depth
    # total_epochs == 0: the random-projection baseline, like train_multilevel
    plan = (np.zeros(depth, dtype=np.int64) if cfg.total_epochs == 0
            else epoch_plan(cfg.total_epochs, cfg.smoothing_ratio, depth).per_level)
    _lib.require_cuda()
    device = torch.device("cuda", torch.cuda.current_device())

    def sharded(i):
        return i < shard_levels and hierarchy.graphs[i].num_vertices >= 2 * G

    stats = []
    M = None       # replicated full matrix of the current (unsharded) level
    store = None   # parts of the current sharded level
    top = depth - 1
    if sharded(top):
        store = PartStore(hierarchy.graphs[top].num_vertices, cfg.dim, G, local, device,
                          host=host_parts)
        store.init_random(cfg.seed)
    else:
        M = torch.from_numpy(init_embedding(hierarchy.graphs[top].num_vertices, cfg.dim,
                                            cfg.seed)).cuda()
    broadcast_done = False
    for i in range(depth - 1, -1, -1):
        g_i = hierarchy.graphs[i]
        e_i = int(plan[i])
        t0 = time.perf_counter()
        if store is not None:
            B_i = _level_batch(g_i, cfg, e_i, store.K, batch_size) if adapt_batch else batch_size
            st = train_tournament_parts(g_i, store, cfg, e_i, batch_size=B_i,
                                        rng_stream=i, group=group) if e_i > 0 else {}
            entry = {"level": i, "sharded": True, "batch_size": B_i, **st}
        else:
            entry = {"level": i, "sharded": False, "passes": 0, "updates": 0}
            if rank == 0 and e_i > 0:
                ts = train_level(g_i, M, cfg, e_i, rng_stream=i)
                entry.update(passes=ts.passes, updates=ts.updates)
        torch.cuda.synchronize()
        entry["s"] = time.perf_counter() - t0
        stats.append(entry)
        if i == 0:
            break
        mapping = hierarchy.mappings[i - 1]
        if sharded(i - 1):
            if store is None:  # first sharded level: from the replicated coarse matrix
                if distributed and not broadcast_done:
                    _broadcast(M, group)
                    broadcast_done = True
                coarse = M
            else:              # coarser level sharded too: gather it (it is ~5x smaller)
                coarse = store.to_full(group=group, distributed=distributed)
            store = PartStore(hierarchy.graphs[i - 1].num_vertices, cfg.dim, G, local, device,
                              host=host_parts)
            store.expand_from(coarse, mapping)
            del coarse
            M = None
        else:
            if store is not None:  # (not reached with the default finest-first sharding)
                M = store.to_full(group=group, distributed=distributed)
                store = None
            M = expand_embedding(M, mapping)
    clear_rotation_graphs()  # the cached rotation holds pool buffers and the CSR
    if store is not None:
        if return_parts:
            return store, stats
        M = store.to_full(group=group, distributed=distributed)
    elif distributed and not broadcast_done:
        _broadcast(M, group)
    if return_device:
        return M, stats
    from ._staging import device_to_numpy
    return device_to_numpy(M), stats
