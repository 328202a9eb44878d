"""Device memory for graphs that fill the GPU (C4/C5 shapes).

A C5 run allocates and frees tens of GiB per phase (the CSR's row-block key
buffers, every coarse level's arrays, the 116 GB matrix).  Each fresh
allocation of that size maps physical HBM into torch's allocator on the
spot: 0.2-3 s per allocation at the C5 shape, varying run to run
(profiles/r02_c5_coarsen_pool_reserve.jsonl).  `reserve_device_memory`
maps the memory once up front and keeps it mapped, after which those
allocations are served from the allocator's pool.  Measured at C5: build
7.0 -> 5.0 s and coarsening 2.7-3.0 -> 2.3 s, but the reservation itself
takes 2.7-6.5 s and the 116 GB matrix allocated later inside a fully mapped
pool cost the embed 1-9 s, so it pays for build/coarsen-only work and is
opt-in (RESERVE=1 in the scripts).
"""
from __future__ import annotations

import ctypes
import time

import torch

_CUDA_MEMPOOL_ATTR_RELEASE_THRESHOLD = 4  # cudaMemPoolAttrReleaseThreshold


def _keep_pool_mapped(device: int) -> None:
    """torch's cudaMallocAsync backend allocates from the device's default
    CUDA mempool, whose release threshold (0) hands freed memory back to the
    driver at every synchronisation; raise it so the pool keeps what it
    mapped."""
    lib = ctypes.CDLL("libcudart.so.12")
    pool = ctypes.c_void_p()
    if lib.cudaDeviceGetDefaultMemPool(ctypes.byref(pool), device) != 0:
        raise RuntimeError("cudaDeviceGetDefaultMemPool failed")
    v = ctypes.c_uint64(2**64 - 1)
    if lib.cudaMemPoolSetAttribute(pool, _CUDA_MEMPOOL_ATTR_RELEASE_THRESHOLD,
                                   ctypes.byref(v)) != 0:
        raise RuntimeError("cudaMemPoolSetAttribute failed")


def reserve_device_memory(nbytes: int | None = None, fraction: float = 0.9) -> dict:
    """Map `nbytes` (default: `fraction` of the free memory) of the current
    device into torch's allocator once and keep it there.  With the
    cudaMallocAsync backend the default mempool's release threshold is raised
    first; with the native caching allocator the freed block stays cached and
    later allocations are split from it.  Returns {"bytes", "seconds",
    "backend"}."""
    if not torch.cuda.is_available():
        raise RuntimeError("reserve_device_memory needs a CUDA device")
    torch.cuda.init()
    dev = torch.cuda.current_device()
    backend = torch.cuda.get_allocator_backend()
    if backend == "cudaMallocAsync":
        _keep_pool_mapped(dev)
    if nbytes is None:
        free, _ = torch.cuda.mem_get_info(dev)
        nbytes = int(free * fraction)
    t0 = time.perf_counter()
    if nbytes > 0:
        block = torch.empty(nbytes, dtype=torch.uint8, device="cuda")
        del block
    torch.cuda.synchronize()
    return {"bytes": int(nbytes), "seconds": time.perf_counter() - t0, "backend": backend}
