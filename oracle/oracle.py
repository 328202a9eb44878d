"""CPU oracle for the GOSH hot path -- TEST INFRASTRUCTURE ONLY.

numpy/ctypes front end of ``oracle/gosh_oracle.c``, a plain-C restatement of
the reference's numba kernels (``/root/reference/pkg/src/mlembed``; each
function cites the file:line it follows).  Only ``tests/``,
``__graft_entry__.smoke()``, ``bench.py``'s CPU-baseline legs and the
measurement scripts' CPU-baseline / reference legs (``scripts/``) import
this module, and only as the checker or the CPU reference -- never as the
GPU side measured or shipped.  The product package (``paper_2008_12336_b200``)
never imports it (``tests/test_host_cpu.py`` enforces that).

Pinning: ``tests/test_oracle_golden.py`` checks every function here against
golden vectors produced by the reference itself
(``tests/golden/make_golden.py``, run in the build container where the
reference is importable).
"""
from __future__ import annotations

import ctypes as C
import math
import os
import subprocess

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_LIB_PATH = os.path.join(_HERE, "liboracle.so")
_lib = None

_i64p = np.ctypeslib.ndpointer(np.int64, flags="C_CONTIGUOUS")
_i32p = np.ctypeslib.ndpointer(np.int32, flags="C_CONTIGUOUS")
_f32p = np.ctypeslib.ndpointer(np.float32, flags="C_CONTIGUOUS")
_u64, _i64, _int, _dbl, _flt = C.c_uint64, C.c_int64, C.c_int, C.c_double, C.c_float


def build() -> str:
    """Compile liboracle.so (gcc, no FMA contraction)."""
    subprocess.run(["make", "-s", "-C", _HERE], check=True)
    return _LIB_PATH


def lib():
    global _lib
    if _lib is None:
        if not os.path.exists(_LIB_PATH):
            build()
        L = C.CDLL(_LIB_PATH)
        sig = {
            "or_mix64": (_u64, [_u64]),
            "or_stream_key": (_u64, [_u64, _u64, _u64, _u64]),
            "or_draw_below": (_i64, [_u64, _u64, _i64]),
            "or_rng_draw_below": (None, [_u64, _u64, _u64, _u64, _u64, _i64, _i64, _i64p]),
            "or_update_embedding": (None, [_f32p, _int, _i64, _i64, _int, _dbl, _int]),
            "or_train_pass": (None, [_i64p, _i32p, _i64, _f32p, _int, _flt, _int, _u64, _u64,
                                     _u64, _int, _int]),
            "or_train_passes": (None, [_i64p, _i32p, _i64, _f32p, _int, _int, _u64, _u64, _i64,
                                       _i64, _i64, _f32p, _int, _int]),
            "or_train_passes_ppr": (None, [_i64p, _i32p, _i64, _f32p, _int, _int, _u64, _u64,
                                           _i64, _i64, _i64, _f32p, _int, _int, _dbl]),
            "or_ppr_positives": (None, [_i64p, _i32p, _i64, _dbl, _u64, _u64, _i64, _i64p]),
            "or_fill_pool_side": (None, [_i64p, _i32p, _i64, _i64, _i64, _i64, _int, _u64, _u64,
                                         _i32p]),
            "or_train_pool_side": (_i64, [_f32p, _f32p, _int, _i32p, _i64, _int, _i64, _i64,
                                          _int, _dbl, _u64, _u64, _int, _int]),
            "or_counting_order": (None, [_i64p, _i64, _i64p]),
            "or_collapse_seq": (_i64, [_i64p, _i32p, _i64p, _i64p, _i64, _dbl, _i32p]),
            "or_coarse_csr": (_i64, [_i64p, _i32p, _i64, _i32p, _i64, _i64p, _i32p]),
            "or_csr_from_arcs": (_i64, [_i64, _i64p, _i64p, _i64, C.c_uint, _i64p, _i32p]),
            "or_expand": (None, [_f32p, _int, _i32p, _i64, _f32p]),
            "or_rmat_permutation": (None, [_int, _u64, _i64p]),
            "or_rmat_edges": (None, [_int, _i64, _dbl, _dbl, _dbl, _u64, C.c_void_p, _i64p,
                                     _i64p]),
            "or_max_threads": (_int, []),
            "or_checksum": (_u64, [C.c_void_p, _i64, _int]),
        }
        for name, (res, args) in sig.items():
            f = getattr(L, name)
            f.restype = res
            f.argtypes = args
        _lib = L
    return _lib


def _u(x: int) -> int:
    return int(x) & 0xFFFFFFFFFFFFFFFF


def _c(a, dtype):
    return np.ascontiguousarray(a, dtype=dtype)


# -- _rng.py ------------------------------------------------------------------
def mix64(z: int) -> int:
    return int(lib().or_mix64(_u(z)))


def stream_key(seed, stream, step, vertex) -> int:
    return int(lib().or_stream_key(_u(seed), _u(stream), _u(step), _u(vertex)))


def draw_below(key: int, ctr: int, n: int) -> int:
    return int(lib().or_draw_below(_u(key), _u(ctr), int(n)))


def rng_draw_below(seed, stream, step, v0, ctr, n, count) -> np.ndarray:
    out = np.empty(count, dtype=np.int64)
    lib().or_rng_draw_below(_u(seed), _u(stream), _u(step), _u(v0), _u(ctr), int(n), count, out)
    return out


def max_threads() -> int:
    return int(lib().or_max_threads())


# -- trainer.py ------------------------------------------------------------------
def update_embedding(M: np.ndarray, v: int, s: int, b: int, lr: float, reuse=False) -> None:
    assert M.dtype == np.float32 and M.flags.c_contiguous
    lib().or_update_embedding(M, M.shape[1], v, s, int(b), float(lr), int(bool(reuse)))


def train_pass(xadj, adj, M, lr, n_neg, seed, stream, pass_idx, nthreads=1, reuse=False):
    assert M.dtype == np.float32 and M.flags.c_contiguous
    lib().or_train_pass(_c(xadj, np.int64), _c(adj, np.int32), len(xadj) - 1, M, M.shape[1],
                        np.float32(lr), int(n_neg), _u(seed), _u(stream), _u(pass_idx),
                        int(nthreads), int(bool(reuse)))


def lr_at(lr0: float, j: int, e_i: int) -> float:
    """trainer.py:179-181."""
    return lr0 * max(1.0 - j / e_i, 1e-4)


def passes_per_epoch(num_vertices: int, num_edges: int, epoch_unit: str) -> int:
    """trainer.py:223-226."""
    if epoch_unit == "edge-scaled" and num_edges > 0:
        return -(-num_edges // num_vertices)
    return 1


def train_level(xadj, adj, M, dim, e_i, lr0, n_neg, seed, stream, epoch_unit="vertex-pass",
                nthreads=1, reuse=False, ppr_alpha=0.0) -> tuple[int, int]:
    """train_level (trainer.py:210-240) over the C pass; returns (passes, updates)."""
    V = len(xadj) - 1
    E = int(xadj[-1])
    ppe = passes_per_epoch(V, E, epoch_unit)
    lrs = np.asarray([np.float32(lr_at(lr0, j, e_i)) for j in range(e_i)], dtype=np.float32)
    if e_i and ppr_alpha > 0:  # VERSE PPR positives (not in the reference)
        lib().or_train_passes_ppr(_c(xadj, np.int64), _c(adj, np.int32), V, M, dim, int(n_neg),
                                  _u(seed), _u(stream), 0, e_i * ppe, ppe, lrs, int(nthreads),
                                  int(bool(reuse)), float(np.float32(ppr_alpha)))
    elif e_i:
        lib().or_train_passes(_c(xadj, np.int64), _c(adj, np.int32), V, M, dim, int(n_neg),
                              _u(seed), _u(stream), 0, e_i * ppe, ppe, lrs, int(nthreads),
                              int(bool(reuse)))
    non_isolated = int((np.diff(xadj) > 0).sum())
    return e_i * ppe, e_i * ppe * non_isolated * (1 + n_neg)


# -- bigtrain.py -----------------------------------------------------------------
def ppr_positives(xadj, adj, v, alpha, seed, stream, n_draws) -> np.ndarray:
    """n_draws PPR positives of v, draw k keyed like pass k's source v."""
    out = np.empty(n_draws, dtype=np.int64)
    # alpha as the device holds it (float32, train_kernels.cuh PassArgs)
    lib().or_ppr_positives(_c(xadj, np.int64), _c(adj, np.int32), int(v),
                           float(np.float32(alpha)),
                           _u(seed), _u(stream), int(n_draws), out)
    return out


def fill_pool_side(xadj, adj, lo_s, hi_s, lo_t, hi_t, B, seed, side) -> np.ndarray:
    out = np.empty((hi_s - lo_s, B), dtype=np.int32)
    lib().or_fill_pool_side(_c(xadj, np.int64), _c(adj, np.int32), lo_s, hi_s, lo_t, hi_t, B,
                            _u(seed), _u(side), out)
    return out


def train_pool_side(Msrc, Mtgt, targets, lo_t, n_t, n_neg, lr, seed, side, nthreads=1,
                    reuse=False) -> int:
    """Msrc and Mtgt may be the same ndarray (diagonal pair)."""
    targets = _c(targets, np.int32)
    return int(lib().or_train_pool_side(Msrc, Mtgt, Msrc.shape[1], targets, targets.shape[0],
                                        targets.shape[1], lo_t, n_t, int(n_neg), float(lr),
                                        _u(seed), _u(side), int(nthreads), int(bool(reuse))))


def derived_seed(seed: int, stream: int, pos: int) -> int:
    """bigtrain.py:302-306."""
    h = mix64(_u(seed ^ (stream * 0x9E3779B97F4A7C15)))
    h = mix64(h ^ pos)
    return h & 0x7FFFFFFFFFFFFFFF


# -- coarsen.py ------------------------------------------------------------------
def counting_order(deg) -> np.ndarray:
    deg = _c(deg, np.int64)
    out = np.empty(deg.shape[0], dtype=np.int64)
    lib().or_counting_order(deg, deg.shape[0], out)
    return out


def collapse_seq(xadj, adj, order) -> tuple[np.ndarray, int]:
    xadj = _c(xadj, np.int64)
    V = len(xadj) - 1
    deg = np.diff(xadj).astype(np.int64)
    delta = float(xadj[-1]) / V if V else 0.0
    cmap = np.empty(V, dtype=np.int32)
    nc = lib().or_collapse_seq(xadj, _c(adj, np.int32), deg, _c(order, np.int64), V, delta,
                               cmap)
    return cmap, int(nc)


def coarse_csr(xadj, adj, cmap, nc) -> tuple[np.ndarray, np.ndarray]:
    xadj = _c(xadj, np.int64)
    adj = _c(adj, np.int32)
    xo = np.empty(nc + 1, dtype=np.int64)
    ao = np.empty(max(int(xadj[-1]), 1), dtype=np.int32)
    m = lib().or_coarse_csr(xadj, adj, len(xadj) - 1, _c(cmap, np.int32), nc, xo, ao)
    return xo, ao[:m].copy()


def coarsen_all(xadj, adj, threshold=100):
    """coarsen_all(num_workers=1) (coarsen.py:284-311): list of (xadj, adj),
    list of (cmap, nc), stalled."""
    graphs = [(_c(xadj, np.int64), _c(adj, np.int32))]
    maps = []
    stalled = False
    while len(graphs[-1][0]) - 1 > threshold:
        x, a = graphs[-1]
        V = len(x) - 1
        order = counting_order(np.diff(x))
        cmap, nc = collapse_seq(x, a, order)
        if nc > 0.99 * V:
            stalled = True
            break
        graphs.append(coarse_csr(x, a, cmap, nc))
        maps.append((cmap, nc))
    return graphs, maps, stalled


# -- graph.py ---------------------------------------------------------------------
def csr_from_arcs(V, src, dst, drop_self=True, symmetrize=True):
    src = _c(src, np.int64)
    dst = _c(dst, np.int64)
    n = src.shape[0]
    flags = (1 if drop_self else 0) | (2 if symmetrize else 0)
    xadj = np.empty(V + 1, dtype=np.int64)
    adj = np.empty(max(n * (2 if symmetrize else 1), 1), dtype=np.int32)
    m = lib().or_csr_from_arcs(V, src, dst, n, flags, xadj, adj)
    return xadj, adj[:m].copy()


def densify(xadj, adj):
    """Drop isolated vertices, ids re-densified ascending (graph.py:160-164)."""
    deg = np.diff(xadj)
    kept = np.flatnonzero(deg > 0).astype(np.int64)
    new_id = np.full(len(deg), -1, dtype=np.int64)
    new_id[kept] = np.arange(kept.shape[0])
    x2 = np.append(xadj[:-1][kept], xadj[-1]).astype(np.int64)
    a2 = new_id[adj].astype(np.int32)
    return x2, a2, kept


def expand(coarse, cmap) -> np.ndarray:
    coarse = _c(coarse, np.float32)
    cmap = _c(cmap, np.int32)
    out = np.empty((cmap.shape[0], coarse.shape[1]), dtype=np.float32)
    lib().or_expand(coarse, coarse.shape[1], cmap, cmap.shape[0], out)
    return out


# -- R-MAT -----------------------------------------------------------------------
RMAT_ABCD = (0.57, 0.19, 0.19, 0.05)


def rmat_thresholds(a=0.57, b=0.19, c=0.19):
    return a, a + b, a + b + c


def rmat_permutation(scale: int, seed: int) -> np.ndarray:
    out = np.empty(1 << scale, dtype=np.int64)
    lib().or_rmat_permutation(scale, _u(seed), out)
    return out


def rmat_edges(scale, n, seed, perm=None, thresholds=None):
    ta, tab, tabc = thresholds or rmat_thresholds()
    src = np.empty(n, dtype=np.int64)
    dst = np.empty(n, dtype=np.int64)
    pp = None if perm is None else _c(perm, np.int64)
    lib().or_rmat_edges(scale, n, ta, tab, tabc, _u(seed),
                        None if pp is None else pp.ctypes.data, src, dst)
    return src, dst


def rmat_graph(scale, n_samples, seed, densify_ids=False, permute=True):
    """The synthetic R-MAT input built on the CPU."""
    perm = rmat_permutation(scale, seed) if permute else None
    src, dst = rmat_edges(scale, n_samples, seed, perm)
    xadj, adj = csr_from_arcs(1 << scale, src, dst)
    if densify_ids:
        xadj, adj, _ = densify(xadj, adj)
    return xadj, adj


def init_embedding(num_rows: int, dim: int, seed: int) -> np.ndarray:
    """trainer.py:87-93 (numpy PCG64; identical in the product package)."""
    half = 0.5 / dim
    return np.random.default_rng(seed).uniform(-half, half, size=(num_rows, dim)).astype(
        np.float32)


def algorithmic_bytes_per_source(dim: int, n_neg: int) -> int:
    """8d(2+n_s) + 12 bytes per non-isolated source."""
    return 8 * dim * (2 + n_neg) + 12


__all__ = [n for n in dir() if not n.startswith("_") and n not in ("C", "math", "np", "os",
                                                                     "subprocess")]


def checksum(a: np.ndarray) -> int:
    """or_checksum of an int32/int64 array (twin of the device gb_checksum)."""
    a = np.ascontiguousarray(a)
    if a.dtype not in (np.int32, np.int64):
        raise TypeError("checksum takes int32 or int64 arrays")
    return int(lib().or_checksum(a.ctypes.data, a.size, a.dtype.itemsize))
