"""VERSE/NCE embedding training on the GPU (reference: trainer.py).

Same API as the reference.  Embedding matrices may be numpy float32 arrays
(drop-in: uploaded, trained in HBM, copied back in place) or float32 CUDA
tensors (kept resident, trained in place).  The training pass is the
hand-written sm_100a kernel behind gb_train_passes: one group of lanes owns a
source row in registers for its 1 + n_neg chained updates, samples come from
the reference's counter-based RNG (identical choices), arithmetic is the
reference's (fp64 dot/sigmoid, fp32 score and row updates, no FMA).

Concurrency: like the reference with num_workers > 1, sources run
concurrently and sample rows race benignly (trainer.py:9-13).  Two device
knobs extend TrainConfig:
  deterministic  one source group in the reference's order with the serial
                 fp64 dot -- bit-equal to the reference at num_workers=1;
  max_inflight   cap on concurrently processed sources (0 = auto policy,
                 see `inflight_cap`), the knob that bounds Hogwild staleness
                 on small coarse levels (SURVEY.md finding 11);
  atomic_rows    write sample-row increments back with vector reductions
                 (red.global.add.v4.f32) instead of storing the updated row,
                 so concurrent updates of a hot row are never lost.
"""
from __future__ import annotations

import os
import struct
from dataclasses import dataclass
from typing import IO, NamedTuple

import numpy as np
import torch

from . import _lib
from ._staging import copy_device_to_numpy, device_to_numpy, numpy_to_device
from .coarsen import Hierarchy, Mapping, coarsen_all
from .errors import ConfigError, PlanError
from .graph import Graph

EMBED_MAGIC = b"GSHE"
EMBED_VERSION = 1
SIGMOID_CLAMP = 10.0
LR_FLOOR = 1e-4
EPOCH_UNITS = ("vertex-pass", "edge-scaled")
SIMILARITIES = ("adjacency", "ppr")
# GB_FAST_SIGMOID=0/1 overrides TrainConfig.fast_sigmoid's default (A/B runs)
FAST_SIGMOID_DEFAULT = {"0": False, "1": True}.get(os.environ.get("GB_FAST_SIGMOID", ""))
# auto in-flight policy max(FLOOR, V / DIVISOR).  Default: uncapped (the
# cap is >= V).  Round 1 needed max(256, V/16) to hold C1 AUCROC to the
# reference while source rows were written back with plain stores; with the
# source increments reduced (train_kernels.cuh writeback_source) the
# uncapped and capped policies land at the same paired difference over 60
# seeds (+0.0011 vs +0.0012, profiles/r02_c1_aucroc_60_seeds.jsonl) and
# uncapped embeds C1 2.4x faster.  The environment overrides exist for
# staleness/quality experiments (scripts/c1_auc_sweep.py).
INFLIGHT_FLOOR = int(os.environ.get("GB_INFLIGHT_FLOOR", "4096"))
INFLIGHT_DIVISOR = int(os.environ.get("GB_INFLIGHT_DIV", "1"))


@dataclass
class TrainConfig:
    """Run knobs (trainer.py:41-72) plus the two device knobs above."""

    dim: int = 128
    total_epochs: int = 100
    smoothing_ratio: float = 0.3
    learning_rate: float = 0.035
    negative_samples: int = 3
    seed: int = 1
    num_workers: int = 1
    epoch_unit: str = "vertex-pass"
    reuse_updated_source: bool = False
    deterministic: bool = False
    max_inflight: int = 0
    atomic_rows: bool = True
    # partitioned / sharded trainers only: balanced pools (bigtrain.PairSides)
    balanced_pools: bool = False
    # positive-sample similarity: "adjacency" (the reference, trainer.py:203)
    # or "ppr" -- VERSE's personalized PageRank with continue probability
    # ppr_alpha (not in the reference, SPEC.md:14;
    # in-memory levels only: the part-pair pools are adjacency by design)
    similarity: str = "adjacency"
    ppr_alpha: float = 0.85
    # parallel kernels' sigmoid: False = fp64 like the reference
    # (trainer.py:118), True = fp32 cancellation-free form (~1e-7 relative),
    # None (default) / False: the reference's fp64 sigmoid in vertex passes
    # and part-pair kernels (no cost on C2 or the K=16 tournament, 6% at the
    # power-capped K=2; profiles/r02_sigmoid_fp64_vs_fp32.jsonl,
    # r02_pair_sigmoid_default_fp64.jsonl); True: the fp32 form
    fast_sigmoid: bool | None = FAST_SIGMOID_DEFAULT

    def validate(self) -> None:
        if self.dim < 1:
            raise ConfigError("dim must be positive")
        if self.total_epochs < 0:
            raise ConfigError("total_epochs must be >= 0")
        if not 0.0 <= self.smoothing_ratio <= 1.0:
            raise ConfigError("smoothing_ratio must be in [0, 1]")
        if self.learning_rate <= 0.0:
            raise ConfigError("learning_rate must be positive")
        if self.negative_samples < 0:
            raise ConfigError("negative_samples must be >= 0")
        if self.num_workers < 1:
            raise ConfigError("num_workers must be >= 1")
        if self.epoch_unit not in EPOCH_UNITS:
            raise ConfigError(f"epoch_unit must be one of {EPOCH_UNITS}")
        if self.max_inflight < 0:
            raise ConfigError("max_inflight must be >= 0")
        if self.balanced_pools and self.deterministic:
            raise ConfigError("balanced_pools runs on the Hogwild kernels (deterministic=False)")
        if self.similarity not in SIMILARITIES:
            raise ConfigError(f"similarity must be one of {SIMILARITIES}")
        if self.similarity == "ppr" and not 0.0 < self.ppr_alpha < 1.0:
            raise ConfigError("ppr_alpha must be in (0, 1)")


@dataclass
class EpochPlan:
    """Epochs per level, index 0 = finest (trainer.py:75-79)."""

    per_level: np.ndarray


class TrainStats(NamedTuple):
    passes: int
    updates: int


def inflight_cap(cfg: TrainConfig, num_vertices: int) -> int:
    """Sources in flight for a level: 1 when deterministic, the explicit cap
    when set, else max(INFLIGHT_FLOOR, V / INFLIGHT_DIVISOR) -- uncapped by
    default (>= V); SURVEY.md finding 11's staleness bound survives as the
    max_inflight knob."""
    if cfg.deterministic:
        return 1
    if cfg.max_inflight > 0:
        return cfg.max_inflight
    return max(INFLIGHT_FLOOR, num_vertices // INFLIGHT_DIVISOR)


def init_embedding(num_rows: int, dim: int, seed: int) -> np.ndarray:
    """U[-0.5/d, 0.5/d] float32 rows from numpy's PCG64 (trainer.py:87-93);
    kept on the host so the draw is bit-identical to the reference."""
    if num_rows < 1 or dim < 1:
        raise ConfigError("embedding dimensions must be positive")
    bound = 0.5 / dim
    return np.random.default_rng(seed).uniform(-bound, bound, size=(num_rows, dim)).astype(
        np.float32)


def sigmoid(x):
    """1/(1+exp(-x)) with x clamped to [-10, 10] (trainer.py:96-99)."""
    z = np.clip(x, -SIGMOID_CLAMP, SIGMOID_CLAMP)
    return 1.0 / (1.0 + np.exp(-z))


# ---------------------------------------------------------------------------
# device helpers
# ---------------------------------------------------------------------------
class _DeviceMatrix:
    """A float32 matrix in HBM; writes back into a numpy original on close."""

    def __init__(self, M):
        _lib.require_cuda()
        self.host = None
        self.host_tensor = None
        if isinstance(M, torch.Tensor):
            if M.dtype != torch.float32 or not M.is_contiguous():
                raise TypeError("embedding tensor must be a contiguous float32 tensor")
            if M.is_cuda:
                self.dev = M
            else:  # host tensor (pinned for async copies): staged through HBM
                self.host_tensor = M
                self.dev = M.to("cuda", non_blocking=True)
        else:
            if not isinstance(M, np.ndarray) or M.dtype != np.float32:
                raise TypeError("embedding matrix must be float32")
            self.host = M
            self.dev = numpy_to_device(M)

    def close(self) -> None:
        if self.host is not None:
            if self.host.flags.c_contiguous:
                copy_device_to_numpy(self.host, self.dev)
            else:
                self.host[...] = device_to_numpy(self.dev)
        elif self.host_tensor is not None:
            self.host_tensor.copy_(self.dev, non_blocking=True)
            torch.cuda.current_stream().synchronize()


def _train_flags(cfg: TrainConfig, pair: bool = False) -> int:
    """EXACT kernels when deterministic; otherwise the parallel kernels with
    the reference's fp64 sigmoid or the fp32 cancellation-free one
    (TrainConfig.fast_sigmoid; None, the default: fp64 for vertex passes and
    pair kernels alike -- equal speed at K >= 4 parts, 6% slower at K = 2),
    fp64 dot either way.  `pair` names the caller; both kinds
    follow the same policy."""
    flags = _lib.GB_TRAIN_REUSE if cfg.reuse_updated_source else 0
    fast = bool(cfg.fast_sigmoid)
    if cfg.deterministic:
        flags |= _lib.GB_TRAIN_EXACT
    elif fast:
        flags |= _lib.GB_TRAIN_FAST_SIGMOID
    if cfg.atomic_rows and not cfg.deterministic:
        flags |= _lib.GB_TRAIN_ATOMIC
    return flags


def _raise_if_nonfinite(status: torch.Tensor, what: str) -> None:
    st = status.cpu().tolist()
    if st[0]:
        raise FloatingPointError(f"non-finite embedding after {what} {st[1]}")


def update_embedding(M, v: int, s: int, b: int, lr: float,
                     reuse_updated_source: bool = False) -> None:
    """One in-place positive (b=1) or negative (b=0) update of rows v and s
    (trainer.py:137-142), run by the device kernel in exact mode.  For a
    numpy matrix only the two touched rows travel."""
    if isinstance(M, np.ndarray) and M.dtype != np.float32:
        raise TypeError("embedding matrix must be float32")
    _lib.require_cuda()
    flags = _lib.GB_TRAIN_EXACT | (_lib.GB_TRAIN_REUSE if reuse_updated_source else 0)
    status = _lib.new_status()
    dm = None
    if isinstance(M, np.ndarray):
        rows = [v] if v == s else [v, s]
        buf = torch.from_numpy(np.ascontiguousarray(M[rows])).cuda()
        lv, ls = 0, (0 if v == s else 1)
    else:  # CUDA tensor: in place; host tensor: staged and written back by close()
        dm = _DeviceMatrix(M)
        buf, lv, ls = dm.dev, v, s
    src = torch.tensor([lv], dtype=torch.int64, device="cuda")
    smp = torch.tensor([ls], dtype=torch.int64, device="cuda")
    lab = torch.tensor([1 if b else 0], dtype=torch.int8, device="cuda")
    _lib.call("gb_apply_sample_lists", _lib.ptr(buf), buf.shape[1], 1, _lib.ptr(src), 1,
              _lib.ptr(smp), _lib.ptr(lab), float(lr), flags, 1, _lib.ptr(status),
              _lib.stream())
    if isinstance(M, np.ndarray):
        M[rows] = buf.cpu().numpy()
    else:
        dm.close()


def apply_sample_lists(M, sources, samples, labels, lr: float, deterministic: bool = False,
                       reuse_updated_source: bool = False, max_inflight: int = 0,
                       atomic_rows: bool = True) -> None:
    """Fixed sample lists: source sources[i] is updated against samples[i, j]
    (j ascending; -1 skips) with label labels[j].  Sources run concurrently
    unless deterministic.  The "single update epoch on fixed sample lists"
    parity unit of the north star."""
    dm = _DeviceMatrix(M)
    src = torch.as_tensor(np.asarray(sources, dtype=np.int64)).cuda()
    smp = torch.as_tensor(np.ascontiguousarray(samples, dtype=np.int64)).cuda()
    lab = torch.as_tensor(np.asarray(labels, dtype=np.int8)).cuda()
    k = int(smp.shape[1]) if smp.dim() == 2 else 0
    flags = (_lib.GB_TRAIN_EXACT if deterministic else 0) | (
        _lib.GB_TRAIN_REUSE if reuse_updated_source else 0) | (
        _lib.GB_TRAIN_ATOMIC if atomic_rows and not deterministic else 0)
    status = _lib.new_status()
    _lib.call("gb_apply_sample_lists", _lib.ptr(dm.dev), dm.dev.shape[1], int(src.numel()),
              _lib.ptr(src), k, _lib.ptr(smp), _lib.ptr(lab), float(lr), flags,
              1 if deterministic else max_inflight, _lib.ptr(status), _lib.stream())
    dm.close()


# ---------------------------------------------------------------------------
# epoch schedule (host)
# ---------------------------------------------------------------------------
def epoch_shares(e: int, p: float, depth: int) -> tuple[float, np.ndarray]:
    """Uniform share p*e/D and geometric shares (1-p)*e*2^i/(2^D-1)
    (trainer.py:145-151)."""
    geo = (1.0 - p) * e * np.power(2.0, np.arange(depth)) / (2.0 ** depth - 1.0)
    return p * e / depth, geo


def epoch_plan(e: int, p: float, depth: int) -> EpochPlan:
    """Round the shares half-up with a floor of 1; surplus goes to the
    coarsest level, deficits are taken from the largest entries, coarser
    first on ties (trainer.py:154-176)."""
    if depth < 1:
        raise PlanError("depth must be >= 1")
    if not 0.0 <= p <= 1.0:
        raise ConfigError("smoothing ratio must be in [0, 1]")
    if e < depth:
        raise PlanError(f"epoch budget {e} smaller than depth {depth}")
    uniform, geo = epoch_shares(e, p, depth)
    plan = np.maximum(np.floor(uniform + geo + 0.5).astype(np.int64), 1)
    diff = int(e - plan.sum())
    if diff > 0:
        plan[-1] += diff
    while diff < 0:
        i = depth - 1 - int(np.argmax(plan[::-1]))
        if plan[i] <= 1:
            raise PlanError("cannot repair rounding under the >=1 floor")
        plan[i] -= 1
        diff += 1
    return EpochPlan(per_level=plan)


def lr_at(lr0: float, j: int, e_i: int) -> float:
    """lr0 * max(1 - j/e_i, 1e-4) (trainer.py:179-181)."""
    return lr0 * max(1.0 - j / e_i, LR_FLOOR)


def passes_per_epoch(g: Graph, cfg: TrainConfig) -> int:
    """ceil(|E|/|V|) vertex passes per edge-scaled epoch, else 1
    (trainer.py:223-226)."""
    if cfg.epoch_unit == "edge-scaled" and g.num_edges > 0:
        return -(-g.num_edges // g.num_vertices)
    return 1


def _non_isolated(g: Graph) -> int:
    if g.on_device:
        x, _ = g.device_csr()
        return int((x[1:] > x[:-1]).sum().item())
    return int((g.degrees() > 0).sum())


# ---------------------------------------------------------------------------
# level training
# ---------------------------------------------------------------------------
def train_level(g: Graph, M, cfg: TrainConfig, e_i: int, lr0: float | None = None,
                rng_stream: int = 0) -> TrainStats:
    """Train M in place for e_i epochs on g (trainer.py:210-240).  One device
    launch per epoch (ppe passes, lr from the f32 schedule); the non-finite
    check is fused into the kernel (sticky flag) plus one full scan at the
    end, raising FloatingPointError like the reference."""
    cfg.validate()
    if M.shape[0] != g.num_vertices:
        raise ValueError("matrix rows must match vertex count")
    if lr0 is None:
        lr0 = cfg.learning_rate
    ppe = passes_per_epoch(g, cfg)
    if e_i <= 0:
        return TrainStats(passes=0, updates=0)
    dm = _DeviceMatrix(M)
    xadj, adj = g.device_csr()
    sources, n_src = g.active_sources()
    lrs = torch.tensor([float(np.float32(lr_at(lr0, j, e_i))) for j in range(e_i)],
                       dtype=torch.float32, device="cuda")
    status = _lib.new_status()
    cap = inflight_cap(cfg, g.num_vertices)
    flags = _train_flags(cfg)
    st = _lib.stream()
    ppr = cfg.similarity == "ppr"
    for j in range(e_i):
        args = (g.num_vertices, _lib.ptr(xadj), _lib.ptr(adj), _lib.ptr(sources), n_src,
                _lib.ptr(dm.dev), cfg.dim, cfg.negative_samples, _lib.u64(cfg.seed),
                _lib.u64(rng_stream), j * ppe, ppe, ppe, _lib.ptr(lrs), flags, cap,
                _lib.ptr(status))
        if ppr:
            _lib.call("gb_train_passes_ppr", *args, float(cfg.ppr_alpha), st)
        else:
            _lib.call("gb_train_passes", *args, st)
    _lib.call("gb_nonfinite_scan", _lib.ptr(dm.dev), dm.dev.numel(), e_i - 1, _lib.ptr(status),
              st)
    dm.close()
    _raise_if_nonfinite(status, "epoch")
    passes = e_i * ppe
    return TrainStats(passes=passes, updates=passes * n_src * (1 + cfg.negative_samples))


def expand_embedding(M_next, m: Mapping):
    """Row v of the result is row map[v] of M_next (trainer.py:243-249);
    coalesced device gather.  numpy in -> numpy out, tensor in -> tensor out."""
    if M_next.shape[0] != m.num_clusters:
        raise ValueError(f"matrix has {M_next.shape[0]} rows, mapping expects "
                         f"{m.num_clusters}")
    on_host = not isinstance(M_next, torch.Tensor)
    src = _DeviceMatrix(M_next).dev if on_host else M_next.contiguous()
    cmap = m.device_map()
    rows = int(cmap.numel())
    out = torch.empty((rows, src.shape[1]), dtype=torch.float32, device="cuda")
    _lib.call("gb_expand", _lib.ptr(src), m.num_clusters, src.shape[1], _lib.ptr(cmap), rows,
              _lib.ptr(out), _lib.stream())
    return out.cpu().numpy() if on_host else out


def level_bytes(g: Graph, dim: int) -> int:
    """Resident footprint of a level as the reference counts it
    (trainer.py:280): matrix + xadj + adj."""
    return g.num_vertices * dim * 4 + (g.num_vertices + 1) * 8 + g.num_edges * 4


def train_multilevel(g0: Graph, cfg: TrainConfig, budget=None, threshold: int = 100,
                     no_coarsen: bool = False, hierarchy: Hierarchy | None = None,
                     return_device: bool = False, release_levels: bool | None = None):
    """Coarsen, then train from the coarsest level down to g0
    (trainer.py:252-288).  The matrix lives in HBM throughout; levels whose
    footprint exceeds budget.resident_bytes take the partitioned path.
    Returns numpy float32 [V0, d] (or the CUDA tensor with return_device).

    release_levels (default: when the hierarchy is built here): a coarse
    level's device CSR and mapping are dropped as soon as the next finer
    matrix is expanded from it, so the finest level's matrix can take the
    HBM the coarse levels held (C5 at d=256 on one GPU: 116 GB matrix + 34 GB
    CSR)."""
    cfg.validate()
    if release_levels is None:
        release_levels = hierarchy is None
    if hierarchy is None:
        hierarchy = (Hierarchy(graphs=[g0], mappings=[]) if no_coarsen
                     else coarsen_all(g0, threshold=threshold, num_workers=cfg.num_workers))
    depth = hierarchy.depth
    plan = (np.zeros(depth, dtype=np.int64) if cfg.total_epochs == 0
            else epoch_plan(cfg.total_epochs, cfg.smoothing_ratio, depth).per_level)
    _lib.require_cuda()
    M = torch.from_numpy(init_embedding(hierarchy.graphs[-1].num_vertices, cfg.dim,
                                        cfg.seed)).cuda()
    for i in range(depth - 1, -1, -1):
        g_i = hierarchy.graphs[i]
        e_i = int(plan[i])
        if e_i > 0:
            if budget is None or level_bytes(g_i, cfg.dim) <= budget.resident_bytes:
                train_level(g_i, M, cfg, e_i, rng_stream=i)
            else:
                from .bigtrain import train_large
                train_large(g_i, M, cfg, e_i, budget, rng_stream=i)
        if i > 0:
            if release_levels:
                g_i._xadj_dev = g_i._adj_dev = None
                g_i.__dict__.pop("_active", None)
                M_next = expand_embedding(M, hierarchy.mappings[i - 1])
                del M
                hierarchy.mappings[i - 1]._map_dev = None
                M = M_next
            else:
                M = expand_embedding(M, hierarchy.mappings[i - 1])
    return M if return_device else device_to_numpy(M)


# ---------------------------------------------------------------------------
# embedding I/O (host)
# ---------------------------------------------------------------------------
def _host(M) -> np.ndarray:
    return M.detach().cpu().numpy() if isinstance(M, torch.Tensor) else np.asarray(M)


def save_embedding(M, path: str) -> None:
    """GSHE: magic, u32 version, u64 rows, u32 dim, f32 rows little-endian
    (trainer.py:291-298).  A CUDA matrix is streamed out of HBM through
    pinned chunks (no full host copy)."""
    if isinstance(M, torch.Tensor) and M.is_cuda:
        from ._staging import device_to_file
        if M.dim() != 2 or M.dtype != torch.float32:
            raise TypeError("embedding must be a 2-D float32 matrix")
        with open(path, "wb") as f:
            f.write(EMBED_MAGIC + struct.pack("<IQI", EMBED_VERSION, M.shape[0], M.shape[1]))
            device_to_file(f, M.contiguous().view(-1).view(torch.uint8))
        return
    A = np.ascontiguousarray(_host(M), dtype="<f4")
    with open(path, "wb") as f:
        f.write(EMBED_MAGIC + struct.pack("<IQI", EMBED_VERSION, A.shape[0], A.shape[1]))
        f.write(A.tobytes())


def load_embedding(path: str, device: bool = False):
    """Read a GSHE file (trainer.py:301-312) as a numpy float32 matrix; with
    device=True straight into a CUDA tensor through pinned chunks."""
    import os
    with open(path, "rb") as f:
        magic = f.read(4)
        if magic != EMBED_MAGIC:
            raise ValueError(f"bad magic {magic!r}, expected {EMBED_MAGIC!r}")
        (version,) = struct.unpack("<I", f.read(4))
        if version != EMBED_VERSION:
            raise ValueError(f"unsupported embedding version {version}")
        rows, dim = struct.unpack("<QI", f.read(12))
        if device and os.fstat(f.fileno()).st_size >= 20 + 4 * rows * dim:
            from ._staging import file_to_device
            _lib.require_cuda()
            out = torch.empty((rows, dim), dtype=torch.float32, device="cuda")
            file_to_device(f, out.view(-1).view(torch.uint8), 4 * rows * dim)
            return out
        data = np.fromfile(f, dtype="<f4", count=rows * dim)
    A = data.reshape(rows, dim).astype(np.float32)
    return torch.from_numpy(A).cuda() if device else A


def write_embedding_tsv(M, stream: IO[str], orig_ids: np.ndarray | None = None) -> None:
    """One "id<TAB>v0 v1 ..." line per row (trainer.py:315-321)."""
    A = _host(M)
    ids = orig_ids if orig_ids is not None else np.arange(A.shape[0])
    for i in range(A.shape[0]):
        stream.write(f"{ids[i]}\t" + " ".join(repr(float(x)) for x in A[i]) + "\n")


__all__ = ["TrainConfig", "EpochPlan", "TrainStats", "init_embedding", "sigmoid",
           "update_embedding", "apply_sample_lists", "epoch_shares", "epoch_plan", "lr_at",
           "train_level", "expand_embedding", "train_multilevel", "save_embedding",
           "load_embedding", "write_embedding_tsv", "inflight_cap", "passes_per_epoch",
           "level_bytes"]
