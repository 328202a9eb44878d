"""Synthetic R-MAT input on the GPU (the reference has no
generator).

Graph500 parameters (a, b, c, d) = (0.57, 0.19, 0.19, 0.05); every edge is a
pure function of (seed, edge index) through the reference's splitmix64
streams (key(seed, 'RMAT', e, 0), one draw per level), ids are relabelled by
a seeded permutation (stable sort of draw_u64(key(seed, 'PERM', 0, 0), i)),
then the arcs go through the same CSR build as from_edges (self-loops and
duplicates dropped, symmetrized).  Multilevel configs densify ids the way
load_edge_list does.  oracle/gosh_oracle.c restates the generator on the CPU
for the parity tests; the fixture tests pin it against the reference's
from_edges.
"""
from __future__ import annotations

import numpy as np
import torch

from . import _lib
from .graph import Graph, _csr_device, densify

RMAT_ABCD = (0.57, 0.19, 0.19, 0.05)


def rmat_edges(scale: int, num_samples: int, seed: int, permute: bool = True,
               abc=RMAT_ABCD[:3]) -> tuple[torch.Tensor, torch.Tensor]:
    """Raw sampled (src, dst) int64 device arrays over 2^scale ids."""
    _lib.require_cuda()
    a, b, c = abc
    st = _lib.stream()
    perm = None
    if permute:
        ws, wsb = _lib.workspace("gb_rmat_permutation_workspace", scale)
        perm = torch.empty(1 << scale, dtype=torch.int64, device="cuda")
        _lib.call("gb_rmat_permutation", scale, _lib.u64(seed), _lib.ptr(perm), _lib.ptr(ws),
                  wsb, st)
        del ws
    src = torch.empty(num_samples, dtype=torch.int64, device="cuda")
    dst = torch.empty(num_samples, dtype=torch.int64, device="cuda")
    _lib.call("gb_rmat_edges", scale, num_samples, a, a + b, a + b + c, _lib.u64(seed),
              _lib.ptr(perm), _lib.ptr(src), _lib.ptr(dst), st)
    return src, dst


def _samples_fit(scale: int, num_samples: int, max_block_keys: int) -> bool:
    """Whether the int64 sample arrays fit beside the row-block build: the
    samples (16 B each), the block's keys and workspace (~24 B per key), the
    CSR (<= 8 B per sample in adj, 8 B per id in xadj) and 4 GiB of slack."""
    free, _ = torch.cuda.mem_get_info()
    need = 16 * num_samples + 24 * max_block_keys + 8 * num_samples + 8 * (1 << scale) + (4 << 30)
    return need < free


def rmat_graph(scale: int, num_samples: int, seed: int = 7, densify_ids: bool = False,
               permute: bool = True, max_block_keys: int | None = None,
               batch_samples: int = 1 << 28, keep_samples: bool | None = None) -> Graph:
    """Undirected R-MAT CSR on the device.  With densify_ids, isolated ids
    are dropped (orig_ids holds the surviving raw ids).

    max_block_keys: build the CSR block by block (graph.csr_from_arc_batches)
    with samples regenerated in batches of batch_samples for every block
    (each sample is a pure function of its index), so neither the sample
    arrays nor the key scratch scale with the graph -- the path for graphs
    whose one-shot build exceeds one GPU (C5).  keep_samples (default: when
    they fit, _samples_fit) generates the samples once and keeps them for
    every block instead (C5: 69 GB; the nine block passes then read them
    instead of regenerating 4.3B samples each).  Same graph bit for bit."""
    flags = _lib.GB_CSR_DROP_SELF | _lib.GB_CSR_SYMMETRIZE
    if max_block_keys is not None:
        from .graph import csr_from_arc_batches
        _lib.require_cuda()
        a, b, c = RMAT_ABCD[:3]
        perm = None
        if permute:
            ws, wsb = _lib.workspace("gb_rmat_permutation_workspace", scale)
            perm = torch.empty(1 << scale, dtype=torch.int64, device="cuda")
            _lib.call("gb_rmat_permutation", scale, _lib.u64(seed), _lib.ptr(perm),
                      _lib.ptr(ws), wsb, _lib.stream())
            del ws
        bs = max(1, min(batch_samples, num_samples))
        if keep_samples is None:
            keep_samples = _samples_fit(scale, num_samples, max_block_keys)
        if keep_samples:  # generate once, every block reads them
            src = torch.empty(num_samples, dtype=torch.int64, device="cuda")
            dst = torch.empty(num_samples, dtype=torch.int64, device="cuda")
            for first in range(0, num_samples, bs):
                n = min(bs, num_samples - first)
                _lib.call("gb_rmat_edges_range", scale, first, n, a, a + b, a + b + c,
                          _lib.u64(seed), _lib.ptr(perm), src.data_ptr() + 8 * first,
                          dst.data_ptr() + 8 * first, _lib.stream())

            def batches():
                for first in range(0, num_samples, bs):
                    n = min(bs, num_samples - first)
                    yield src[first:first + n], dst[first:first + n]
        else:
            src = torch.empty(bs, dtype=torch.int64, device="cuda")
            dst = torch.empty(bs, dtype=torch.int64, device="cuda")

            def batches():
                for first in range(0, num_samples, bs):
                    n = min(bs, num_samples - first)
                    _lib.call("gb_rmat_edges_range", scale, first, n, a, a + b, a + b + c,
                              _lib.u64(seed), _lib.ptr(perm), _lib.ptr(src), _lib.ptr(dst),
                              _lib.stream())
                    yield src[:n], dst[:n]

        g = csr_from_arc_batches(1 << scale, batches, flags, max_block_keys)
        del src, dst, perm
    else:
        src, dst = rmat_edges(scale, num_samples, seed, permute)
        g = _csr_device(1 << scale, src, dst, flags, False)
        del src, dst
    if densify_ids:
        g2, kept = densify(g)
        g2.orig_ids = kept
        return g2
    return g


def samples_for_edges(target_undirected_edges: int, keep_ratio: float = 0.81) -> int:
    """Oversampling to reach a target count of unique undirected edges
    (dedup keeps ~81% at scale 14 and ~94% at scale 20)."""
    return int(np.ceil(target_undirected_edges / keep_ratio))
