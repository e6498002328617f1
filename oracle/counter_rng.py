"""Host twin of ``tlb_fill_uniform`` (paper_1804_10120_b200/csrc/tlb_static.cu)
— test infrastructure: regenerates any slab of a counter-based synthetic
input so a full-size (2^28-point) GPU result can be checked slab by slab
against the oracle.

u01(seed, stream, i) = (mix64(key + (i + 1) * GAMMA) >> 11) * 2^-53,
key = mix64(seed ^ mix64(stream + GAMMA)), mix64 = splitmix64 finaliser.
"""

from __future__ import annotations

import numpy as np

GAMMA = np.uint64(0x9E3779B97F4A7C15)
M1 = np.uint64(0xBF58476D1CE4E5B9)
M2 = np.uint64(0x94D049BB133111EB)


def _mix(z):
    z = np.asarray(z, dtype=np.uint64)
    with np.errstate(over="ignore"):
        z = (z ^ (z >> np.uint64(30))) * M1
        z = (z ^ (z >> np.uint64(27))) * M2
    return z ^ (z >> np.uint64(31))


def key(seed: int, stream_id: int) -> np.uint64:
    with np.errstate(over="ignore"):
        inner = _mix(np.uint64(stream_id) + GAMMA)
    return _mix(np.uint64(seed) ^ inner)


def uniform(seed: int, stream_id: int, offset: int, n: int) -> np.ndarray:
    k = key(seed, stream_id)
    i = np.arange(offset + 1, offset + n + 1, dtype=np.uint64)
    with np.errstate(over="ignore"):
        h = _mix(k + i * GAMMA)
    return (h >> np.uint64(11)).astype(np.float64) * (2.0 ** -53)
