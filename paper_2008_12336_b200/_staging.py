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
