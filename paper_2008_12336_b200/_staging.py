"""Pinned-host staging between files and device memory (graph / embedding
I/O).

Two pinned chunks and one side stream: while chunk k's host<->device copy
runs on the stream, the host reads (or writes) chunk k+1 of the file, so the
disk and PCIe transfers overlap and no full-size host copy (the reference's
`np.frombuffer(...).astype(...)`, graph.py:214-215) is ever made.
"""
from __future__ import annotations

import torch

CHUNK = 64 << 20
_pool: list[torch.Tensor] = []


def _buffers() -> list[torch.Tensor]:
    if not _pool:
        _pool.extend(torch.empty(CHUNK, dtype=torch.uint8).pin_memory() for _ in range(2))
    return _pool


def file_to_device(f, dst: torch.Tensor, nbytes: int) -> None:
    """Read nbytes from the binary file f into the start of dst (a CUDA uint8
    view).  Raises EOFError if the file ends early."""
    if nbytes == 0:
        return
    bufs = _buffers()
    main = torch.cuda.current_stream()
    side = torch.cuda.Stream()
    side.wait_stream(main)
    done: list[torch.cuda.Event | None] = [None, None]
    off, k = 0, 0
    while off < nbytes:
        n = min(CHUNK, nbytes - off)
        b = bufs[k % 2]
        if done[k % 2] is not None:
            done[k % 2].synchronize()  # the copy out of this buffer has finished
        got = f.readinto(memoryview(b.numpy())[:n])
        if got != n:
            side.synchronize()
            raise EOFError(f"file ended {nbytes - off - (got or 0)} bytes early")
        with torch.cuda.stream(side):
            dst[off:off + n].copy_(b[:n], non_blocking=True)
            ev = torch.cuda.Event()
            ev.record(side)
        done[k % 2] = ev
        off += n
        k += 1
    main.wait_stream(side)
    dst.record_stream(side)
    side.synchronize()


def device_to_file(f, src: torch.Tensor) -> None:
    """Write the bytes of src (a contiguous CUDA uint8 view) to f."""
    nbytes = src.numel()
    if nbytes == 0:
        return
    bufs = _buffers()
    main = torch.cuda.current_stream()
    side = torch.cuda.Stream()
    side.wait_stream(main)
    nchunks = -(-nbytes // CHUNK)
    ready: list[torch.cuda.Event | None] = [None, None]

    def issue(k):
        off = k * CHUNK
        n = min(CHUNK, nbytes - off)
        with torch.cuda.stream(side):
            bufs[k % 2][:n].copy_(src[off:off + n], non_blocking=True)
            ev = torch.cuda.Event()
            ev.record(side)
        ready[k % 2] = ev

    issue(0)
    for k in range(nchunks):
        if k + 1 < nchunks:
            issue(k + 1)  # its buffer was written to the file in iteration k-1
        ready[k % 2].synchronize()
        n = min(CHUNK, nbytes - k * CHUNK)
        f.write(memoryview(bufs[k % 2].numpy())[:n])
    src.record_stream(side)


# ---------------------------------------------------------------------------
# numpy <-> device arrays.  torch's .cuda() / .cpu() on pageable memory run at
# ~11 / ~2.2 GB/s here (the download into fresh pages is page-fault bound:
# 0.60 s for C3's 1.34 GB matrix, 64% of the end-to-end embed;
# profiles/r02_c3_e2e_phases.jsonl).  These stage through the two pinned
# chunks with the host-side copies split over a thread pool (numpy releases
# the GIL for plain copies), so the page faults and memcpy run in parallel
# while the next chunk's DMA is in flight.
# ---------------------------------------------------------------------------
_SMALL = 8 << 20  # below this, torch's own copy is as fast
_pool_threads = None


def _threads():
    global _pool_threads
    if _pool_threads is None:
        import os
        from concurrent.futures import ThreadPoolExecutor
        _pool_threads = ThreadPoolExecutor(max_workers=max(1, min(8, os.cpu_count() or 1)))
    return _pool_threads


def _par_copy(dst, src) -> None:
    """dst[...] = src for two equal-length 1-D uint8 numpy views, in pieces."""
    n = dst.shape[0]
    ex = _threads()
    k = ex._max_workers
    step = -(-n // k)
    futs = [ex.submit(dst.__setitem__, slice(i, min(i + step, n)), src[i:min(i + step, n)])
            for i in range(0, n, step)]
    for f in futs:
        f.result()


def copy_numpy_to_device(dst, a) -> None:
    """dst (contiguous CUDA tensor) <- numpy array a (same number of bytes)."""
    import warnings

    import numpy as np
    a = np.ascontiguousarray(a)
    with warnings.catch_warnings():  # read-only views (np.frombuffer): only read here
        warnings.simplefilter("ignore", UserWarning)
        t = torch.from_numpy(a)
    if a.nbytes < _SMALL or t.is_pinned():  # page-locked already: one direct DMA
        dst.view(-1).view(torch.uint8).copy_(t.reshape(-1).view(torch.uint8))
        return
    src = a.reshape(-1).view(np.uint8)
    dst = dst.view(-1).view(torch.uint8)
    bufs = _buffers()
    main = torch.cuda.current_stream()
    side = torch.cuda.Stream()
    side.wait_stream(main)
    done: list = [None, None]
    n = src.shape[0]
    off, k = 0, 0
    while off < n:
        m = min(CHUNK, n - off)
        b = bufs[k % 2]
        if done[k % 2] is not None:
            done[k % 2].synchronize()
        _par_copy(b.numpy()[:m], src[off:off + m])
        with torch.cuda.stream(side):
            dst[off:off + m].copy_(b[:m], non_blocking=True)
            ev = torch.cuda.Event()
            ev.record(side)
        done[k % 2] = ev
        off += m
        k += 1
    main.wait_stream(side)
    dst.record_stream(side)
    side.synchronize()


def numpy_to_device(a):
    """A CUDA tensor with the contents of numpy array `a` (same dtype/shape)."""
    import numpy as np
    a = np.ascontiguousarray(a)
    out = torch.empty(a.shape, dtype=torch.from_numpy(a[:0]).dtype, device="cuda")
    copy_numpy_to_device(out, a)
    return out


def copy_device_to_numpy(dst, t) -> None:
    """numpy array dst (C-contiguous) <- CUDA tensor t (same number of bytes)."""
    import numpy as np
    if not dst.flags.c_contiguous:
        raise ValueError("copy_device_to_numpy needs a C-contiguous destination")
    t = t.detach().contiguous()
    dst8 = dst.reshape(-1).view(np.uint8)
    if dst8.nbytes < _SMALL or torch.from_numpy(dst8).is_pinned():
        torch.from_numpy(dst8).copy_(t.view(-1).view(torch.uint8))
        return
    src = t.view(-1).view(torch.uint8)
    n = dst8.shape[0]
    bufs = _buffers()
    side = torch.cuda.Stream()
    side.wait_stream(torch.cuda.current_stream())
    pend = []
    off, k = 0, 0
    while off < n:
        m = min(CHUNK, n - off)
        b = bufs[k % 2]
        with torch.cuda.stream(side):
            b[:m].copy_(src[off:off + m], non_blocking=True)
            ev = torch.cuda.Event()
            ev.record(side)
        pend.append((ev, b, off, m))
        if len(pend) == 2:  # drain the older chunk while this one is in flight
            e, bb, o, mm = pend.pop(0)
            e.synchronize()
            _par_copy(dst8[o:o + mm], bb.numpy()[:mm])
        off += m
        k += 1
    for e, bb, o, mm in pend:
        e.synchronize()
        _par_copy(dst8[o:o + mm], bb.numpy()[:mm])
    t.record_stream(side)


def device_to_numpy(t):
    """A new numpy array with the contents of CUDA tensor `t`."""
    import numpy as np
    out = np.empty(tuple(t.shape), dtype=torch.empty(0, dtype=t.dtype).numpy().dtype)
    copy_device_to_numpy(out, t)
    return out
