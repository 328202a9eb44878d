"""Host-side scalar splitmix64 (_rng.py:19-32) for seeds derived on the host
(bigtrain._derived_seed).  Per-sample draws happen only on the device."""
from __future__ import annotations

_M = 0xFFFFFFFFFFFFFFFF
GOLDEN = 0x9E3779B97F4A7C15
MIX1 = 0xBF58476D1CE4E5B9
MIX2 = 0x94D049BB133111EB


def mix64(z: int) -> int:
    z = (int(z) + GOLDEN) & _M
    z = ((z ^ (z >> 30)) * MIX1) & _M
    z = ((z ^ (z >> 27)) * MIX2) & _M
    return z ^ (z >> 31)


def stream_key(seed: int, stream: int, step: int, vertex: int) -> int:
    h = mix64((int(seed) ^ (int(stream) * GOLDEN)) & _M)
    h = mix64(h ^ (int(step) & _M))
    return mix64(h ^ (int(vertex) & _M))
