"""CSR graph container and graph I/O (reference: graph.py).

`Graph` keeps the reference's fields and methods (graph.py:23-77) but can be
backed by device tensors: graphs built on the GPU (from_edges, the R-MAT
generator, every coarse level) stay in HBM and only materialize their numpy
`xadj`/`adj` when host code asks for them; host graphs upload once and cache
the device copy.  CSR construction runs on the GPU (gb_csr_build: 64-bit
key radix sort + unique + per-row binary search), producing exactly the
reference's rows (strictly ascending, no duplicates, self-loops dropped).

Text/binary I/O and the train/test split are host-side, as in the reference
(they feed the hot path; SURVEY.md 2.1 marks them out of scope for
acceleration).  The split keeps numpy's PCG64 stream so it selects the same
edges as the reference for the same seed.
"""
from __future__ import annotations

import ctypes as C
import json
import os
import struct
import time
from dataclasses import dataclass
from typing import IO, Iterable

import numpy as np
import torch

from . import _lib
from .errors import EdgeListParseError, EmptyGraphError, SplitError

GRAPH_MAGIC = b"GSHG"
GRAPH_VERSION = 1


class Graph:
    """Compressed-sparse-row adjacency; `num_edges` counts stored arcs (an
    undirected edge is two arcs).  Rows are strictly ascending."""

    def __init__(self, num_vertices: int, num_edges: int, xadj: np.ndarray | None = None,
                 adj: np.ndarray | None = None, directed: bool = False,
                 orig_ids: np.ndarray | None = None, *, xadj_dev: torch.Tensor | None = None,
                 adj_dev: torch.Tensor | None = None):
        if xadj is None and xadj_dev is None:
            raise ValueError("Graph needs host or device CSR arrays")
        self.num_vertices = int(num_vertices)
        self.num_edges = int(num_edges)
        self.directed = bool(directed)
        self.orig_ids = orig_ids
        self._xadj = None if xadj is None else np.asarray(xadj)
        self._adj = None if adj is None else np.asarray(adj)
        self._xadj_dev = xadj_dev
        self._adj_dev = adj_dev

    # -- host view (lazy download) ---------------------------------------------
    @property
    def xadj(self) -> np.ndarray:
        if self._xadj is None:
            from ._staging import device_to_numpy
            self._xadj = device_to_numpy(self._xadj_dev)
        return self._xadj

    @xadj.setter
    def xadj(self, value) -> None:
        self._xadj = np.asarray(value)
        self._xadj_dev = None

    @property
    def adj(self) -> np.ndarray:
        if self._adj is None:
            if self._adj_dev is None:
                self._adj = np.empty(0, dtype=np.int32)
            else:
                from ._staging import device_to_numpy
                self._adj = device_to_numpy(self._adj_dev[: self.num_edges])
        return self._adj

    @adj.setter
    def adj(self, value) -> None:
        self._adj = np.asarray(value)
        self._adj_dev = None

    # -- device view (lazy upload) -----------------------------------------------
    def device_csr(self) -> tuple[torch.Tensor, torch.Tensor]:
        """(xadj int64[V+1], adj int32[max(E,1)]) on the current CUDA device."""
        _lib.require_cuda()
        from ._staging import numpy_to_device
        if self._xadj_dev is None:
            self._xadj_dev = numpy_to_device(np.ascontiguousarray(self._xadj, dtype=np.int64))
        if self._adj_dev is None:
            a = np.ascontiguousarray(self.adj, dtype=np.int32)
            if a.size == 0:
                a = np.zeros(1, dtype=np.int32)
            self._adj_dev = numpy_to_device(a)
        return self._xadj_dev, self._adj_dev

    def active_sources(self) -> tuple[torch.Tensor, int]:
        """Non-isolated vertex ids (int32, ascending) -- the sources a
        training pass visits (trainer.py:198-200); computed once on the GPU."""
        cached = getattr(self, "_active", None)
        if cached is None:
            xadj, _ = self.device_csr()
            ws, wsb = _lib.workspace("gb_active_sources_workspace", self.num_vertices)
            out = torch.empty(self.num_vertices, dtype=torch.int32, device="cuda")
            n = C.c_int64(0)
            _lib.call("gb_active_sources", self.num_vertices, _lib.ptr(xadj), _lib.ptr(out),
                      C.byref(n), _lib.ptr(ws), wsb, _lib.stream())
            cached = (out[: max(int(n.value), 1)].clone(), int(n.value))
            self._active = cached
        return cached

    def drop_host(self) -> None:
        """Forget the host copies of a device-resident graph."""
        if self._xadj_dev is not None:
            self._xadj = None
            self._adj = None

    @property
    def on_device(self) -> bool:
        return self._xadj_dev is not None

    # -- reference methods (graph.py:37-77) --------------------------------------
    def degree(self, v: int) -> int:
        return int(self.xadj[v + 1] - self.xadj[v])

    def neighbors(self, v: int) -> np.ndarray:
        return self.adj[self.xadj[v]:self.xadj[v + 1]]

    def has_arc(self, u: int, v: int) -> bool:
        row = self.neighbors(u)
        i = int(np.searchsorted(row, v))
        return i < row.shape[0] and int(row[i]) == v

    def degrees(self) -> np.ndarray:
        return np.diff(self.xadj).astype(np.int64)

    def undirected_pairs(self) -> np.ndarray:
        """Arcs (u, v) with u < v as an (m, 2) array in CSR order; each
        undirected edge once (graph.py:52-59).  Enumerated on the GPU
        (gb_undirected_pairs) when the CSR lives there."""
        if self.on_device and self.num_edges > 0:
            pu, pv, m = _undirected_pairs_device(self)
            return np.stack([pu[:m].cpu().numpy(), pv[:m].cpu().numpy()], axis=1)
        src = np.repeat(np.arange(self.num_vertices, dtype=np.int64), np.diff(self.xadj))
        dst = self.adj.astype(np.int64)
        m = src < dst
        return np.stack([src[m], dst[m]], axis=1)

    def validate(self) -> None:
        x, a = self.xadj, self.adj
        if x.shape[0] != self.num_vertices + 1:
            raise ValueError("xadj length must be |V|+1")
        if x[0] != 0 or x[-1] != self.num_edges:
            raise ValueError("xadj endpoints inconsistent with |E|")
        steps = np.diff(x)
        if (steps < 0).any():
            raise ValueError("xadj must be nondecreasing")
        if self.num_edges:
            if a.shape[0] != self.num_edges:  # truncated file: numpy's broadcast ValueError
                raise ValueError(f"adj holds {a.shape[0]} entries, |E| = {self.num_edges}")
            if a.min() < 0 or a.max() >= self.num_vertices:
                raise ValueError("adj entry out of range")
            # strictly ascending inside each row: a rise must occur at every
            # position that is not a row start
            row_start = np.zeros(self.num_edges, dtype=bool)
            row_start[x[:-1][steps > 0]] = True
            if (np.diff(a.astype(np.int64)) <= 0)[~row_start[1:]].any():
                raise ValueError("adjacency rows must be strictly ascending")

    def __repr__(self) -> str:
        where = "device" if self.on_device else "host"
        return (f"Graph(num_vertices={self.num_vertices}, num_edges={self.num_edges}, "
                f"directed={self.directed}, {where})")


@dataclass
class SplitResult:
    """Train graph plus withheld test edges (train-graph ids); kept_vertices
    maps train id -> id in the split graph (graph.py:80-90)."""

    train_graph: Graph
    test_edges: np.ndarray
    kept_vertices: np.ndarray


def _csr_device(num_vertices: int, src: torch.Tensor, dst: torch.Tensor, flags: int,
                directed: bool, orig_ids=None) -> Graph:
    """gb_csr_build on device arc arrays (graph.py:93-109 semantics)."""
    _lib.require_cuda()
    src = src.to(device="cuda", dtype=torch.int64).contiguous()
    dst = dst.to(device="cuda", dtype=torch.int64).contiguous()
    n = int(src.numel())
    cap = n * (2 if flags & _lib.GB_CSR_SYMMETRIZE else 1)
    ws, wsb = _lib.workspace("gb_csr_build_workspace", num_vertices, n, flags)
    xadj = torch.empty(num_vertices + 1, dtype=torch.int64, device="cuda")
    adj = torch.empty(max(cap, 1), dtype=torch.int32, device="cuda")
    ne = C.c_int64(0)
    _lib.call("gb_csr_build", num_vertices, _lib.ptr(src) if n else None,
              _lib.ptr(dst) if n else None, n, flags, _lib.ptr(xadj), _lib.ptr(adj),
              C.byref(ne), _lib.ptr(ws), wsb, _lib.stream())
    del ws
    E = int(ne.value)
    adj = adj[:max(E, 1)].clone() if cap > 2 * max(E, 1) else adj
    return Graph(num_vertices, E, directed=directed, orig_ids=orig_ids, xadj_dev=xadj,
                 adj_dev=adj)


def plan_row_blocks(hist: np.ndarray, max_block_keys: int) -> list[tuple[int, int]]:
    """Consecutive row ranges whose arc counts (hist, an upper bound per row)
    sum to at most max_block_keys; a row above the cap gets a block of its
    own."""
    if max_block_keys < 1:
        raise ValueError("max_block_keys must be positive")
    csum = np.concatenate([[0], np.cumsum(hist, dtype=np.int64)])
    n = hist.shape[0]
    blocks, r0 = [], 0
    while r0 < n:
        r1 = int(np.searchsorted(csum, csum[r0] + max_block_keys, side="right")) - 1
        r1 = min(max(r1, r0 + 1), n)
        blocks.append((r0, r1))
        r0 = r1
    return blocks


def plan_row_blocks_tensor(hist: torch.Tensor, max_block_keys: int):
    """plan_row_blocks on a torch tensor where it lives (the device histogram
    of a C5-sized CSR has 2^28 rows: a 2 GB download plus host cumsum costs
    seconds): (blocks, total keys, largest block's keys).  Same blocks as
    plan_row_blocks."""
    if max_block_keys < 1:
        raise ValueError("max_block_keys must be positive")
    n = int(hist.shape[0])
    if n == 0:
        return [], 0, 0
    csum = torch.cumsum(hist.to(torch.int64), 0)  # csum[i] = keys of rows [0, i]
    upper = int(csum[-1])
    blocks, r0, before, largest = [], 0, 0, 0
    while r0 < n:
        target = torch.tensor([before + max_block_keys], dtype=torch.int64, device=csum.device)
        r1 = int(torch.searchsorted(csum, target, right=True))
        r1 = min(max(r1, r0 + 1), n)
        after = int(csum[r1 - 1])
        blocks.append((r0, r1))
        largest = max(largest, after - before)
        r0, before = r1, after
    return blocks, upper, largest


def _scratch_buffer(scratch: dict | None, name: str, numel: int, dtype) -> torch.Tensor:
    """A device buffer of at least numel elements, kept in `scratch` between
    row-block builds (a coarsening ladder asks for the same tens of GiB at
    every level; re-allocating them cost 0.2-1.1 s per level at C5)."""
    def alloc():
        try:
            return torch.empty(numel, dtype=dtype, device="cuda")
        except torch.OutOfMemoryError:
            # tens of GiB can fail on cached-but-fragmented blocks: hand them
            # back to the driver and retry once (as _lib.workspace does)
            torch.cuda.empty_cache()
            return torch.empty(numel, dtype=dtype, device="cuda")

    if scratch is None:
        return alloc()
    buf = scratch.get(name)
    if buf is None or buf.numel() < numel:
        scratch.pop(name, None)
        del buf
        buf = alloc()
        scratch[name] = buf
    return buf[:numel]


def csr_from_blocks(num_rows: int, num_cols: int, hist: torch.Tensor, fill_block,
                    max_block_keys: int, directed: bool = False, orig_ids=None,
                    scratch: dict | None = None) -> Graph:
    """Row-block CSR construction (gb_keys_to_rows): rows are keyed, sorted,
    deduplicated and emitted one block at a time, so scratch scales with
    max_block_keys instead of the arc count.  `fill_block(r0, r1, keys,
    cursor)` appends the keys of the block's arcs (gb_arc_keys_range /
    gb_mapped_keys_range over every batch).  Equal to the one-shot build bit
    for bit: blocks emit their rows in order."""
    trace = os.environ.get("GB_TRACE_BLOCKS")
    ts = [time.perf_counter()]
    if trace:
        torch.cuda.synchronize()  # the histogram pass
    ts.append(time.perf_counter())
    blocks, upper, block_keys = plan_row_blocks_tensor(hist, max_block_keys)
    ts.append(time.perf_counter())
    xadj = torch.empty(num_rows + 1, dtype=torch.int64, device="cuda")
    adj = torch.empty(max(upper, 1), dtype=torch.int32, device="cuda")
    keys = _scratch_buffer(scratch, "keys", max(block_keys, 1), torch.int64)
    cursor = torch.zeros(1, dtype=torch.int64, device="cuda")
    rows_max = max((b - a for a, b in blocks), default=1)
    if trace:
        torch.cuda.synchronize()
    ts.append(time.perf_counter())
    n_ws = C.c_size_t(0)
    _lib.call("gb_keys_to_rows_workspace", max(block_keys, 1), rows_max, num_cols,
              C.byref(n_ws))
    wsb = int(n_ws.value)
    ws = _scratch_buffer(scratch, "ws", max(wsb, 1), torch.uint8)
    base = 0
    if trace:
        torch.cuda.synchronize()
        ts.append(time.perf_counter())
        print(json.dumps({"blocks": len(blocks), "rows": num_rows, "upper_keys": upper,
                          "hist_ms": 1e3 * (ts[1] - ts[0]),
                          "plan_ms": 1e3 * (ts[2] - ts[1]),
                          "alloc_out_keys_ms": 1e3 * (ts[3] - ts[2]),
                          "alloc_workspace_ms": 1e3 * (ts[4] - ts[3]),
                          "alloc_gib": round((8 * num_rows + 4 * upper + 8 * block_keys + wsb)
                                             / 2**30, 1),
                          "reserved_gib": round(torch.cuda.memory_reserved() / 2**30, 1)}),
              flush=True)
    for r0, r1 in blocks:
        t0 = time.perf_counter() if trace else 0.0
        cursor.zero_()
        fill_block(r0, r1, keys, cursor)
        nk = int(cursor.item())
        t1 = time.perf_counter() if trace else 0.0
        nu = C.c_int64(0)
        _lib.call("gb_keys_to_rows", _lib.ptr(keys), nk, r1 - r0, num_cols, base,
                  xadj.data_ptr() + r0 * 8, adj.data_ptr() + base * 4, C.byref(nu),
                  _lib.ptr(ws), wsb, _lib.stream())
        base += int(nu.value)
        if trace:  # per-block phases (scripts/profile_coarsen.py)
            print(json.dumps({"block": [r0, r1], "keys": nk, "unique": int(nu.value),
                              "fill_ms": 1e3 * (t1 - t0),
                              "sort_ms": 1e3 * (time.perf_counter() - t1)}), flush=True)
    t_end = time.perf_counter()
    xadj[num_rows] = base
    del ws, keys
    adj = adj[: max(base, 1)].clone() if upper > 1.25 * max(base, 1) else adj
    if trace:
        torch.cuda.synchronize()
        print(json.dumps({"finish_ms": 1e3 * (time.perf_counter() - t_end)}), flush=True)
    return Graph(num_rows, base, directed=directed, orig_ids=orig_ids, xadj_dev=xadj,
                 adj_dev=adj)


def csr_from_arc_batches(num_vertices: int, batches, flags: int, max_block_keys: int,
                         directed: bool = False) -> Graph:
    """from_edges semantics (graph.py:93-131) over arcs that arrive in batches
    (`batches()` yields device (src, dst) int64 pairs and may be called once
    per block, e.g. regenerating R-MAT samples), built block by block."""
    _lib.require_cuda()
    st = _lib.stream()
    hist = torch.zeros(num_vertices, dtype=torch.int64, device="cuda")
    for src, dst in batches():
        _lib.call("gb_arc_histogram", _lib.ptr(src), _lib.ptr(dst), src.numel(), flags,
                  _lib.ptr(hist), st)

    def fill(r0, r1, keys, cursor):
        for src, dst in batches():
            _lib.call("gb_arc_keys_range", _lib.ptr(src), _lib.ptr(dst), src.numel(), flags,
                      num_vertices, r0, r1, _lib.ptr(keys), _lib.ptr(cursor), st)

    return csr_from_blocks(num_vertices, num_vertices, hist, fill, max_block_keys, directed)


def array_checksum(t) -> int:
    """Position-keyed checksum of an int32/int64 array on the device
    (gb_checksum): sum_i mix64((i * 0x9E3779B97F4A7C15) ^ int64(x[i])) mod
    2^64 -- the oracle's or_checksum of the same array.  Compares
    config-scale hierarchies against the reference without moving GBs."""
    if not isinstance(t, torch.Tensor):
        t = torch.from_numpy(np.ascontiguousarray(t))
    if t.dtype not in (torch.int32, torch.int64):
        raise TypeError("array_checksum takes int32 or int64 arrays")
    t = t.cuda().contiguous()
    out = torch.zeros(1, dtype=torch.int64, device=t.device)
    _lib.call("gb_checksum", _lib.ptr(t), t.numel(), t.element_size(), _lib.ptr(out),
              _lib.stream())
    return int(out.item()) & 0xFFFFFFFFFFFFFFFF


def from_edges(pairs: Iterable[tuple[int, int]] | np.ndarray, num_vertices: int | None = None,
               directed: bool = False) -> Graph:
    """CSR from (u, v) pairs over dense ids: self-loops and duplicate arcs
    dropped, symmetrized unless directed (graph.py:112-131); built on the GPU."""
    arr = np.asarray(pairs if isinstance(pairs, np.ndarray) else list(pairs), dtype=np.int64)
    arr = arr.reshape(-1, 2)
    if num_vertices is None:
        num_vertices = int(arr.max()) + 1 if arr.size else 0
    if num_vertices == 0:
        raise EmptyGraphError("graph has no vertices")
    flags = _lib.GB_CSR_DROP_SELF | (0 if directed else _lib.GB_CSR_SYMMETRIZE)
    t = torch.from_numpy(np.ascontiguousarray(arr))
    return _csr_device(int(num_vertices), t[:, 0], t[:, 1], flags, directed)


def densify(g: Graph) -> tuple[Graph, np.ndarray]:
    """Drop isolated vertices and re-number the rest in ascending order (the
    load_edge_list convention, graph.py:160-164), on the GPU.  Returns the new
    graph and kept (new id -> old id)."""
    xadj, adj = g.device_csr()
    V, E = g.num_vertices, g.num_edges
    ws, wsb = _lib.workspace("gb_csr_densify_workspace", V)
    x2 = torch.empty(V + 1, dtype=torch.int64, device="cuda")
    a2 = torch.empty(max(E, 1), dtype=torch.int32, device="cuda")
    new_id = torch.empty(V, dtype=torch.int64, device="cuda")
    kept = torch.empty(V, dtype=torch.int64, device="cuda")
    nk = C.c_int64(0)
    _lib.call("gb_csr_densify", V, E, _lib.ptr(xadj), _lib.ptr(adj), _lib.ptr(x2), _lib.ptr(a2),
              _lib.ptr(new_id), _lib.ptr(kept), C.byref(nk), _lib.ptr(ws), wsb, _lib.stream())
    k = int(nk.value)
    if k == 0:
        raise EmptyGraphError("graph has no non-isolated vertex")
    kept_h = kept[:k].cpu().numpy()
    return Graph(k, E, directed=g.directed, xadj_dev=x2[:k + 1].clone(), adj_dev=a2), kept_h


def _parse_edge_lines_host(lines, line_base: int = 0):
    """The reference's per-line loop (graph.py:143-157) over `lines`; returns
    (us, vs) lists or raises EdgeListParseError with the global line number."""
    us: list[int] = []
    vs: list[int] = []
    for lineno, raw in enumerate(lines, start=line_base + 1):
        line = raw.strip()
        if not line or line[0] == "#":
            continue
        fields = line.split()
        if len(fields) != 2:
            raise EdgeListParseError(lineno, f"expected two fields, got {len(fields)}")
        try:
            u, v = int(fields[0]), int(fields[1])
        except ValueError:
            raise EdgeListParseError(lineno, f"non-integer vertex id in {line!r}") from None
        us.append(u)
        vs.append(v)
    return us, vs


def _edges_to_graph(src: torch.Tensor, dst: torch.Tensor, directed: bool) -> Graph:
    """Densify ids in ascending order (graph.py:160-164) and build the CSR
    (self-loops dropped, symmetrized unless directed) -- on the GPU."""
    m = int(src.numel())
    ids = torch.cat([src, dst])
    uniq = torch.empty(2 * m, dtype=torch.int64, device="cuda")
    ws, wsb = _lib.workspace("gb_unique_ids_workspace", 2 * m)
    k = C.c_int64(0)
    _lib.call("gb_unique_ids", _lib.ptr(ids), 2 * m, _lib.ptr(uniq), C.byref(k), 1,
              _lib.ptr(ws), wsb, _lib.stream())
    del ws
    orig = uniq[: int(k.value)].cpu().numpy()
    flags = _lib.GB_CSR_DROP_SELF | (0 if directed else _lib.GB_CSR_SYMMETRIZE)
    return _csr_device(int(k.value), ids[:m], ids[m:], flags, directed, orig_ids=orig)


EDGE_TEXT_CHUNK = 256 << 20  # characters (bytes) per device parse


class _NeedsText(Exception):
    """The byte fast path met text Python splits differently (non-ASCII, a
    lone carriage return): restart on the text stream."""


class _EdgeTextParser:
    """Device parse of newline-terminated ASCII chunks (gb_parse_edge_text),
    accumulating the edge ids; malformed lines are re-read by the host loop
    for the reference's message."""

    def __init__(self):
        self.parts_u: list[torch.Tensor] = []
        self.parts_v: list[torch.Tensor] = []
        self.line_base = 0
        self.overflow = False
        self.ws, self.wsb = None, 0
        self.text = None

    def host_chunk(self, body: str) -> None:
        lines = body.split("\n")
        if body.endswith("\n"):
            lines.pop()
        us, vs = _parse_edge_lines_host(lines, self.line_base)
        if any(not -2**63 <= x < 2**63 for x in us + vs):
            self.overflow = True
        elif us:
            self.parts_u.append(torch.tensor(us, dtype=torch.int64))
            self.parts_v.append(torch.tensor(vs, dtype=torch.int64))
        self.line_base += len(lines)

    def device_chunk(self, pieces, body_text) -> bool:
        """pieces: numpy uint8 arrays whose concatenation is the chunk.
        Returns False (nothing consumed) when the chunk needs the host."""
        from ._staging import copy_numpy_to_device
        n = sum(int(p.shape[0]) for p in pieces)
        if self.text is None or self.text.numel() < n:
            self.text = torch.empty(max(n, 1), dtype=torch.uint8, device="cuda")
        off = 0
        for p in pieces:
            if p.shape[0]:
                copy_numpy_to_device(self.text[off:off + p.shape[0]], p)
                off += p.shape[0]
        need = C.c_size_t(0)
        _lib.call("gb_parse_edge_text_workspace", n, C.byref(need))
        if self.ws is None or self.wsb < need.value:
            self.ws = None
            self.ws, self.wsb = _lib.workspace("gb_parse_edge_text_workspace", n)
        cap = n // 2 + 1
        du = torch.empty(cap, dtype=torch.int64, device="cuda")
        dv = torch.empty(cap, dtype=torch.int64, device="cuda")
        res = (C.c_int64 * 5)()
        _lib.call("gb_parse_edge_text", _lib.ptr(self.text), n, _lib.ptr(du), _lib.ptr(dv), res,
                  _lib.ptr(self.ws), self.wsb, _lib.stream())
        m, L, bad, over, host = (int(x) for x in res)
        if host:
            return False
        if bad >= 0:
            body = body_text()
            lines = body.split("\n")
            _parse_edge_lines_host(lines[bad:bad + 1], self.line_base + bad)
            # the device flagged a line the host accepts: trust the host
            us, vs = _parse_edge_lines_host(lines[:-1] if body.endswith("\n") else lines,
                                            self.line_base)
            du = torch.tensor(us, dtype=torch.int64, device="cuda")
            dv = torch.tensor(vs, dtype=torch.int64, device="cuda")
            m = len(us)
        self.overflow = self.overflow or bool(over)
        self.parts_u.append(du[:m])
        self.parts_v.append(dv[:m])
        self.line_base += L
        return True

    def graph(self, directed: bool) -> Graph:
        self.ws = self.text = None
        if self.overflow:
            raise OverflowError("Python int too large to convert to C long")
        if sum(int(t.numel()) for t in self.parts_u) == 0:
            raise EmptyGraphError("edge list contains no edges")
        src = torch.cat([t.cuda() for t in self.parts_u])
        dst = torch.cat([t.cuda() for t in self.parts_v])
        return _edges_to_graph(src, dst, directed)


def _byte_source(text_stream):
    """The binary file under a fresh TextIOWrapper with an ASCII-compatible
    encoding, else None."""
    import codecs
    raw = getattr(text_stream, "buffer", None)
    enc = getattr(text_stream, "encoding", None)
    try:
        if raw is None or enc is None or not raw.seekable() or text_stream.tell() != 0:
            return None
        name = codecs.lookup(enc).name
    except (OSError, LookupError, ValueError):
        return None
    return raw if name in ("utf-8", "ascii", "latin-1", "iso8859-1", "cp1252") else None


def _parse_bytes(raw, parser: _EdgeTextParser) -> None:
    """Chunks of the binary file, cut after their last newline."""
    carry = b""
    while True:
        s = raw.read(EDGE_TEXT_CHUNK)
        eof = not s
        if not eof:
            cut = s.rfind(b"\n")
            if cut < 0:
                carry += s
                continue
            pieces = [np.frombuffer(carry, np.uint8), np.frombuffer(s, np.uint8, count=cut + 1)]
            tail = s[cut + 1:]
        else:
            pieces, tail = [np.frombuffer(carry, np.uint8)], b""
        if sum(p.shape[0] for p in pieces):
            body = (lambda c=carry, s_=s, k=(cut + 1 if not eof else 0):
                    (c + s_[:k]).decode("ascii"))
            if not parser.device_chunk(pieces, body):
                raise _NeedsText()
        carry = tail
        if eof:
            break


def load_edge_list(text_stream: IO[str], directed: bool = False) -> Graph:
    """Edge-list text, one "u v" per line, '#' comments and blank lines
    skipped; ids densified in ascending order with the originals kept in
    orig_ids (graph.py:134-171).

    On a GPU the text is parsed on the device (gb_parse_edge_text: one thread
    per line, Python int() syntax) chunk by chunk, and the ids are densified
    there (gb_unique_ids) before the CSR build; errors are the reference's
    (the first malformed line is re-read by the host loop for its message;
    a valid id outside int64 raises OverflowError after the whole input, as
    numpy's conversion does).  A text file opened with an ASCII-compatible
    encoding is read as bytes straight from its buffer (no decode/encode);
    text the host splits differently (non-ASCII, lone carriage returns)
    goes through the host loop -- for a file, from the start on the text
    stream, for other streams chunk by chunk.  Without a GPU the host loop
    parses everything (the CSR still needs one)."""
    if not torch.cuda.is_available():
        us, vs = _parse_edge_lines_host(text_stream)
        if not us:
            raise EmptyGraphError("edge list contains no edges")
        u_arr = np.asarray(us, dtype=np.int64)
        v_arr = np.asarray(vs, dtype=np.int64)
        return _edges_to_graph(torch.from_numpy(u_arr), torch.from_numpy(v_arr), directed)
    _lib.require_cuda()
    raw = _byte_source(text_stream)
    if raw is not None:
        parser = _EdgeTextParser()
        try:
            _parse_bytes(raw, parser)
            return parser.graph(directed)
        except _NeedsText:
            text_stream.seek(0)
    parser = _EdgeTextParser()
    carry = ""
    while True:
        s = text_stream.read(EDGE_TEXT_CHUNK)
        eof = not s
        buf = carry + s if carry else s
        if not eof:
            cut = buf.rfind("\n")
            if cut < 0:
                carry = buf
                continue
            body, carry = buf[:cut + 1], buf[cut + 1:]
        else:
            body, carry = buf, ""
        if body:
            enc = body.encode("utf-8")
            if not parser.device_chunk([np.frombuffer(enc, np.uint8)], lambda b=body: b):
                parser.host_chunk(body)
        if eof:
            break
    return parser.graph(directed)


def write_edge_list(g: Graph, text_stream: IO[str]) -> None:
    """Inverse of load_edge_list up to densification (graph.py:174-185)."""
    if g.directed:
        src = np.repeat(np.arange(g.num_vertices, dtype=np.int64), np.diff(g.xadj))
        pairs = np.stack([src, g.adj.astype(np.int64)], axis=1)
    else:
        pairs = g.undirected_pairs()
    names = g.orig_ids if g.orig_ids is not None else np.arange(g.num_vertices)
    text_stream.writelines(f"{names[a]} {names[b]}\n" for a, b in pairs)


def degree(g: Graph, v: int) -> int:
    """Number of arcs leaving v."""
    return g.degree(v)


def save_graph(g: Graph, path: str) -> None:
    """GSHG binary cache: magic, u32 version, u64 V, u64 E, u64 xadj[V+1],
    u32 adj[E], little-endian (graph.py:192-200).  A device-resident graph is
    streamed out through pinned chunks (no host copy of the CSR)."""
    header = GRAPH_MAGIC + struct.pack("<IQQ", GRAPH_VERSION, g.num_vertices, g.num_edges)
    with open(path, "wb") as f:
        f.write(header)
        if g._xadj is None and g._xadj_dev is not None and torch.cuda.is_available():
            from ._staging import device_to_file
            x, a = g.device_csr()
            device_to_file(f, x[: g.num_vertices + 1].contiguous().view(torch.uint8))
            device_to_file(f, a[: g.num_edges].contiguous().view(torch.uint8))
            return
        f.write(np.ascontiguousarray(g.xadj, dtype="<u8").tobytes())
        f.write(np.ascontiguousarray(g.adj, dtype="<u4").tobytes())


_VALIDATE_MESSAGES = ((1, "xadj endpoints inconsistent with |E|"),
                      (2, "xadj must be nondecreasing"),
                      (4, "adj entry out of range"),
                      (8, "adjacency rows must be strictly ascending"))


def validate_device(g: Graph) -> None:
    """Graph.validate (graph.py:61-77) on the device CSR: one coalesced pass
    over xadj and adj (gb_csr_validate); the reference's messages, first
    failing check first."""
    x, a = g.device_csr()
    if x.numel() != g.num_vertices + 1:
        raise ValueError("xadj length must be |V|+1")
    ws, wsb = _lib.workspace("gb_csr_validate_workspace", g.num_edges)
    flags = C.c_int(0)
    _lib.call("gb_csr_validate", g.num_vertices, g.num_edges, _lib.ptr(x),
              _lib.ptr(a) if g.num_edges else None, C.byref(flags), _lib.ptr(ws), wsb,
              _lib.stream())
    for bit, msg in _VALIDATE_MESSAGES:
        if flags.value & bit:
            raise ValueError(msg)


def load_graph(path: str, directed: bool = False) -> Graph:
    """Read a GSHG file written by save_graph (graph.py:203-219).  On a GPU
    the arrays are streamed straight into HBM through pinned chunks and
    validated there (validate_device): the result is a device-backed Graph
    whose host arrays materialise on first use.  Without a GPU, or for a
    truncated file (so the reference's error is raised), the host path."""
    import os
    with open(path, "rb") as f:
        magic = f.read(4)
        if magic != GRAPH_MAGIC:
            raise ValueError(f"bad magic {magic!r}, expected {GRAPH_MAGIC!r}")
        (version,) = struct.unpack("<I", f.read(4))
        if version != GRAPH_VERSION:
            raise ValueError(f"unsupported cache version {version}")
        nv, ne = struct.unpack("<QQ", f.read(16))
        full = os.fstat(f.fileno()).st_size >= 24 + 8 * (nv + 1) + 4 * ne
        if torch.cuda.is_available() and full and nv < 2**62:
            from ._staging import file_to_device
            _lib.require_cuda()
            x = torch.empty(nv + 1, dtype=torch.int64, device="cuda")
            a = torch.empty(max(ne, 1), dtype=torch.int32, device="cuda")
            file_to_device(f, x.view(torch.uint8), 8 * (nv + 1))
            file_to_device(f, a.view(torch.uint8), 4 * ne)
            g = Graph(int(nv), int(ne), directed=directed, xadj_dev=x, adj_dev=a)
            validate_device(g)
            return g
        xadj = np.fromfile(f, dtype="<u8", count=nv + 1).astype(np.int64)
        adj = np.fromfile(f, dtype="<u4", count=ne).astype(np.int32)
    g = Graph(int(nv), int(ne), xadj=xadj, adj=adj, directed=directed)
    g.validate()
    return g


def _undirected_pairs_device(g: Graph) -> tuple[torch.Tensor, torch.Tensor, int]:
    """(pu, pv, m): the u < v arcs of g's device CSR in CSR order."""
    xadj, adj = g.device_csr()
    ws, wsb = _lib.workspace("gb_undirected_pairs_workspace", g.num_vertices)
    m_c = C.c_int64(0)
    # a symmetric CSR without self-loops has exactly E/2 such arcs; anything
    # else is retried at the E upper bound
    for cap in (g.num_edges // 2 + 1, max(g.num_edges, 1)):
        pu = torch.empty(cap, dtype=torch.int64, device="cuda")
        pv = torch.empty(cap, dtype=torch.int64, device="cuda")
        rc = _lib.load().gb_undirected_pairs(_lib.ptr(xadj), _lib.ptr(adj), g.num_vertices,
                                             _lib.ptr(pu), _lib.ptr(pv), cap, C.byref(m_c),
                                             _lib.ptr(ws), wsb, _lib.stream())
        if rc == _lib.GB_OK:
            return pu, pv, int(m_c.value)
        del pu, pv
    _lib.check(rc, "gb_undirected_pairs")


def split_train_test(g: Graph, test_fraction: float, seed: int) -> SplitResult:
    """Withhold round(fraction * m) undirected edges chosen by numpy PCG64
    (the same draw as graph.py:242-244, on the host), drop vertices left
    isolated and re-densify; test edges losing an endpoint are dropped
    (graph.py:222-265).  The pair enumeration, partition, relabelling and
    the train CSR run on the GPU (csrc/split.cu, csrc/graph.cu)."""
    if g.directed:
        raise SplitError("split requires an undirected graph")
    if not 0.0 < test_fraction < 1.0:
        raise SplitError(f"test_fraction must be in (0, 1), got {test_fraction}")
    _lib.require_cuda()
    V = g.num_vertices
    st = _lib.stream()
    pu, pv, m = _undirected_pairs_device(g)
    k = int(round(test_fraction * m))
    if k < 1:
        raise SplitError(f"graph too small to withhold any edge "
                         f"({m} edges at fraction {test_fraction})")
    if k >= m:
        raise SplitError("withholding would leave no training edges")
    chosen = torch.from_numpy(np.random.default_rng(seed).choice(m, size=k, replace=False)
                              .astype(np.int64)).cuda()
    tu = torch.empty(m, dtype=torch.int64, device="cuda")
    tv = torch.empty(m, dtype=torch.int64, device="cuda")
    su = torch.empty(k, dtype=torch.int64, device="cuda")
    sv = torch.empty(k, dtype=torch.int64, device="cuda")
    relabel = torch.empty(V, dtype=torch.int64, device="cuda")
    kept = torch.empty(V, dtype=torch.int64, device="cuda")
    counts = (C.c_int64 * 3)()
    ws, wsb = _lib.workspace("gb_split_partition_workspace", m, V)
    _lib.call("gb_split_partition", _lib.ptr(pu[:m]), _lib.ptr(pv[:m]), m, _lib.ptr(chosen), k,
              V, _lib.ptr(tu), _lib.ptr(tv), _lib.ptr(su), _lib.ptr(sv), _lib.ptr(relabel),
              _lib.ptr(kept), counts, _lib.ptr(ws), wsb, st)
    del ws, pu, pv, chosen, relabel
    n_train, n_test, n_kept = int(counts[0]), int(counts[1]), int(counts[2])
    kept_h = kept[:n_kept].cpu().numpy()
    orig = g.orig_ids[kept_h] if g.orig_ids is not None else kept_h.copy()
    tg = _csr_device(n_kept, tu[:n_train], tv[:n_train],
                     _lib.GB_CSR_DROP_SELF | _lib.GB_CSR_SYMMETRIZE, False, orig_ids=orig)
    te = np.stack([su[:n_test].cpu().numpy(), sv[:n_test].cpu().numpy()], axis=1)
    return SplitResult(train_graph=tg, test_edges=te, kept_vertices=kept_h)
