"""reserve_device_memory (memory.py): HBM mapped once into torch's allocator
and reused by later allocations (the C4/C5 scripts call it before building)."""
import pytest
import torch

import paper_2008_12336_b200 as gb


@pytest.mark.gpu
def test_reserve_device_memory_serves_later_allocations(cuda):
    torch.cuda.empty_cache()
    n = 1 << 30
    info = gb.reserve_device_memory(n)
    assert info["bytes"] == n and info["backend"] in ("native", "cudaMallocAsync")
    reserved = torch.cuda.memory_reserved()
    assert reserved >= n
    a = torch.empty(n // 2, dtype=torch.uint8, device="cuda")
    b = torch.empty(n // 4, dtype=torch.uint8, device="cuda")
    assert torch.cuda.memory_reserved() == reserved  # carved from the reserved block
    del a, b
