"""MultiEdgeCollapse coarsening on the GPU (reference: coarsen.py).

The reference's deterministic path is the sequential greedy `_collapse_seq`
(coarsen.py:98-114); its parallel CAS collapse is run-dependent
(coarsen.py:117-156).  Here both entry points run the same deterministic
device algorithm: a vertex is a hub iff none of its
lower-rank "H-neighbours" is a hub, and a member joins its minimum-rank hub
H-neighbour -- decided in a few Gauss-Seidel rounds (gb_collapse), bit-equal
to `_collapse_seq`.  The coarse graph is rebuilt by sorting mapped arcs
(gb_coarse_csr).  Every level stays in HBM; host arrays materialize only on
access.
"""
from __future__ import annotations

import ctypes as C
import os
import time
from dataclasses import dataclass, field

import numpy as np
import torch

from . import _lib
from .errors import ConfigError
from .graph import Graph

STALL_RATIO = 0.99  # coarsen.py:33


class Mapping:
    """Cluster assignment of one step: map[v] = cluster of v in the next
    level, dense in [0, num_clusters) (coarsen.py:36-50).  Backed by a device
    tensor when produced on the GPU."""

    def __init__(self, map: np.ndarray | None = None, num_clusters: int = 0, *,
                 map_dev: torch.Tensor | None = None):
        if map is None and map_dev is None:
            raise ValueError("Mapping needs a host or device map")
        self._map = None if map is None else np.asarray(map)
        self._map_dev = map_dev
        self.num_clusters = int(num_clusters)

    @property
    def map(self) -> np.ndarray:
        if self._map is None:
            self._map = self._map_dev.cpu().numpy()
        return self._map

    @map.setter
    def map(self, value) -> None:
        self._map = np.asarray(value)
        self._map_dev = None

    def device_map(self) -> torch.Tensor:
        _lib.require_cuda()
        if self._map_dev is None:
            self._map_dev = torch.from_numpy(np.ascontiguousarray(self._map, np.int32)).cuda()
        return self._map_dev

    def validate(self) -> None:
        m = self.map
        if m.shape[0] == 0:
            raise ValueError("empty mapping")
        if m.min() < 0 or m.max() >= self.num_clusters:
            raise ValueError("cluster id out of range")
        if np.bincount(m, minlength=self.num_clusters).min() < 1:
            raise ValueError("mapping not surjective")

    def __repr__(self) -> str:
        return f"Mapping(num_clusters={self.num_clusters}, rows={self.rows})"

    @property
    def rows(self) -> int:
        return int(self._map_dev.numel() if self._map_dev is not None else self._map.shape[0])


@dataclass
class Hierarchy:
    """graphs[0] is the input, graphs[-1] the coarsest level; mappings[i]
    sends level i to level i+1 (coarsen.py:53-66)."""

    graphs: list[Graph]
    mappings: list[Mapping]
    stalled: bool = False
    level_ms: list[float] = field(default_factory=list)
    rounds: list[int] = field(default_factory=list)

    @property
    def depth(self) -> int:
        return len(self.graphs)


def _in_csr(g: Graph) -> tuple[torch.Tensor, torch.Tensor]:
    """In-arc CSR: the graph itself when undirected, its transpose otherwise."""
    xadj, adj = g.device_csr()
    if not g.directed:
        return xadj, adj
    cached = getattr(g, "_transpose", None)
    if cached is None:
        from .graph import _csr_device
        src = torch.repeat_interleave(torch.arange(g.num_vertices, device="cuda"),
                                      xadj[1:] - xadj[:-1])
        t = _csr_device(g.num_vertices, adj[: g.num_edges].long(), src, 0, True)
        cached = t.device_csr()
        g._transpose = cached
    return cached


def _degree_order_dev(g: Graph) -> torch.Tensor:
    xadj, _ = g.device_csr()
    V = g.num_vertices
    ws, wsb = _lib.workspace("gb_degree_order_workspace", V)
    order = torch.empty(V, dtype=torch.int64, device="cuda")
    _lib.call("gb_degree_order", V, _lib.ptr(xadj), _lib.ptr(order), _lib.ptr(ws), wsb,
              _lib.stream())
    return order


def degree_order(g: Graph) -> np.ndarray:
    """Vertex ids by nonincreasing degree, ties by ascending id
    (coarsen.py:69-95); stable device radix sort."""
    return _degree_order_dev(g).cpu().numpy()


def _collapse_dev(g: Graph, order) -> tuple[Mapping, int]:
    xadj, _ = g.device_csr()
    in_x, in_a = _in_csr(g)
    V = g.num_vertices
    if isinstance(order, torch.Tensor):
        order_t = order.to(device="cuda", dtype=torch.int64).contiguous()
    else:
        order_t = torch.from_numpy(np.ascontiguousarray(order, dtype=np.int64)).cuda()
    delta = g.num_edges / g.num_vertices  # coarsen.py:161
    ws, wsb = _lib.workspace("gb_collapse_workspace", V)
    cmap = torch.empty(V, dtype=torch.int32, device="cuda")
    nc = C.c_int64(0)
    rounds = C.c_int(0)
    _lib.call("gb_collapse", V, _lib.ptr(xadj), _lib.ptr(in_x), _lib.ptr(in_a),
              _lib.ptr(order_t), float(delta), _lib.ptr(cmap), C.byref(nc), C.byref(rounds),
              _lib.ptr(ws), wsb, _lib.stream())
    return Mapping(num_clusters=int(nc.value), map_dev=cmap), int(rounds.value)


def collapse_map(g: Graph, order) -> Mapping:
    """Greedy hub collapse, equal to the reference's sequential pass
    (coarsen.py:159-163) for the given order."""
    return _collapse_dev(g, order)[0]


def _collapse_cas_dev(g: Graph, order, num_workers: int) -> Mapping:
    xadj, adj = g.device_csr()
    V = g.num_vertices
    if isinstance(order, torch.Tensor):
        order_t = order.to(device="cuda", dtype=torch.int64).contiguous()
    else:
        order_t = torch.from_numpy(np.ascontiguousarray(order, dtype=np.int64)).cuda()
    ws, wsb = _lib.workspace("gb_collapse_cas_workspace", V)
    cmap = torch.empty(V, dtype=torch.int32, device="cuda")
    nc = C.c_int64(0)
    _lib.call("gb_collapse_cas", V, _lib.ptr(xadj), _lib.ptr(adj), _lib.ptr(order_t),
              g.num_edges / g.num_vertices, int(num_workers), _lib.ptr(cmap), C.byref(nc),
              _lib.ptr(ws), wsb, _lib.stream())
    return Mapping(num_clusters=int(nc.value), map_dev=cmap)


def collapse_map_parallel(g: Graph, order, num_workers: int,
                          run_dependent: bool = False) -> Mapping:
    """Reference signature of the parallel collapse (coarsen.py:166-179).

    Default: the device collapse, which is parallel AND deterministic, so
    every worker count returns the sequential result (the reference
    guarantees that only for num_workers=1).  run_dependent=True runs the
    reference's own try-lock algorithm (_collapse_par: CAS claims,
    skip-on-failure, hubs renumbered by order position) with num_workers
    concurrent warps (gb_collapse_cas): one worker equals collapse_map, more
    give a valid map that depends on the interleaving -- the reference's
    speed mode, outside its parity contract (coarsen.py:11-13)."""
    if num_workers < 1:
        raise ConfigError("num_workers must be >= 1")
    if run_dependent:
        return _collapse_cas_dev(g, order, num_workers)
    return collapse_map(g, order)


HEAVY_ARCS = 8192  # row-block builds split vertices above this over all warps


def build_coarse_graph(g: Graph, m: Mapping, num_workers: int = 1,
                       max_block_keys: int | None = None, scratch: dict | None = None) -> Graph:
    """Contract g along m: clusters become vertices, parallel arcs merged,
    self-loops dropped, rows sorted (coarsen.py:256-281).  max_block_keys
    builds the coarse rows block by block (gb_mapped_keys_range +
    gb_keys_to_rows) so the key scratch is bounded instead of 24 B per arc;
    the result is identical.  `scratch` (a dict) keeps the block key buffer and
    workspace for the next level's build."""
    xadj, adj = g.device_csr()
    cmap = m.device_map()
    V, E, nc = g.num_vertices, g.num_edges, m.num_clusters
    if max_block_keys is not None:
        from .graph import csr_from_blocks
        st = _lib.stream()
        hist = torch.zeros(nc, dtype=torch.int64, device="cuda")
        _lib.call("gb_mapped_histogram", _lib.ptr(xadj), _lib.ptr(adj), V, _lib.ptr(cmap),
                  _lib.ptr(hist), st)

        starts = torch.cumsum(hist, 0) - hist  # each row's first key (exclusive scan)
        # hubs (> HEAVY_ARCS arcs) are split over all warps; at most E / HEAVY_ARCS
        heavy_arcs = int(os.environ.get("GB_HEAVY_ARCS", str(HEAVY_ARCS)))
        heavy_cap = E // heavy_arcs + 1
        heavy = torch.empty(heavy_cap + 1, dtype=torch.int64, device="cuda")

        def fill(c0, c1, keys, cursor):
            # per-row cursors (gb_mapped_keys_rows): the block's rows start at
            # their scanned offsets, so the appends spread over the rows
            row_cursor = starts[c0:c1] - starts[c0]
            _lib.call("gb_mapped_keys_rows", _lib.ptr(xadj), _lib.ptr(adj), V, _lib.ptr(cmap),
                      nc, c0, c1, _lib.ptr(row_cursor), _lib.ptr(keys), _lib.ptr(heavy),
                      heavy_cap, heavy_arcs, st)
            cursor.copy_(hist[c0:c1].sum().reshape(1))

        return csr_from_blocks(nc, nc, hist, fill, max_block_keys, directed=g.directed,
                               scratch=scratch)
    n_ws = C.c_size_t(0)
    _lib.call("gb_coarse_csr_workspace", V, E, nc, C.byref(n_ws))
    wsb = int(n_ws.value)
    if scratch is not None:  # coarsen_all: the level-0 workspace serves every level
        from .graph import _scratch_buffer
        ws = _scratch_buffer(scratch, "coarse_ws", max(wsb, 1), torch.uint8)
    else:
        ws, wsb = _lib.workspace("gb_coarse_csr_workspace", V, E, nc)
    x2 = torch.empty(nc + 1, dtype=torch.int64, device="cuda")
    a2 = torch.empty(max(E, 1), dtype=torch.int32, device="cuda")
    ne = C.c_int64(0)
    _lib.call("gb_coarse_csr", V, E, _lib.ptr(xadj), _lib.ptr(adj), _lib.ptr(cmap), nc,
              _lib.ptr(x2), _lib.ptr(a2), C.byref(ne), _lib.ptr(ws), wsb, _lib.stream())
    del ws
    E2 = int(ne.value)
    a2 = a2[:max(E2, 1)].clone()
    return Graph(nc, E2, directed=g.directed, xadj_dev=x2, adj_dev=a2)


def coarsen_all(g: Graph, threshold: int = 100, num_workers: int = 1,
                max_block_keys: int | None = None, run_dependent: bool = False) -> Hierarchy:
    """order -> collapse -> contract until |V| <= threshold; a level keeping
    more than 99% of the vertices is discarded and flags a stall
    (coarsen.py:284-311).  num_workers is accepted for API parity;
    max_block_keys bounds the coarse-CSR key scratch (build_coarse_graph).
    run_dependent with num_workers > 1 collapses with the reference's
    try-lock mode (collapse_map_parallel, coarsen.py:299-302); the default is
    the deterministic device collapse for every worker count."""
    if threshold < 1:
        raise ConfigError("threshold must be >= 1")
    if num_workers < 1:
        raise ConfigError("num_workers must be >= 1")
    graphs, mappings, level_ms, rounds = [g], [], [], []
    scratch: dict = {}  # row-block key buffer + workspace, shared by the levels
    stalled = False
    while graphs[-1].num_vertices > threshold:
        cur = graphs[-1]
        t0 = time.perf_counter()
        order = _degree_order_dev(cur)
        if run_dependent and num_workers > 1:
            m, r = _collapse_cas_dev(cur, order, num_workers), 1
        else:
            m, r = _collapse_dev(cur, order)
        if m.num_clusters > STALL_RATIO * cur.num_vertices:
            stalled = True
            break
        nxt = build_coarse_graph(cur, m, max_block_keys=max_block_keys, scratch=scratch)
        torch.cuda.current_stream().synchronize()
        level_ms.append((time.perf_counter() - t0) * 1000.0)
        graphs.append(nxt)
        mappings.append(m)
        rounds.append(r)
    return Hierarchy(graphs=graphs, mappings=mappings, stalled=stalled, level_ms=level_ms,
                     rounds=rounds)
