"""Seeded synthetic inputs (BASELINE.json configs). No dataset is involved.

Gaussian generator (written down exactly): the splitmix64
stream of reference core.hpp:44-63 started at `seed`, x_k = next_u64() of call
k (k = 0, 1, ...), u_k = (x_k >> 11) * 2^-53 in [0, 1); then Box-Muller on
consecutive pairs:  g_i = sqrt(-2 log(1 - u_{2i})) * cos(2 pi u_{2i+1}).
"""
from __future__ import annotations

import numpy as np

_GOLDEN = np.uint64(0x9E3779B97F4A7C15)


def splitmix64_u01(seed: int, n: int, offset: int = 0) -> np.ndarray:
    """u_k for k in [offset, offset + n) -- vectorised splitmix64."""
    k = np.arange(offset + 1, offset + n + 1, dtype=np.uint64)
    with np.errstate(over="ignore"):
        z = np.uint64(seed) + k * _GOLDEN
        z = (z ^ (z >> np.uint64(30))) * np.uint64(0xBF58476D1CE4E5B9)
        z = (z ^ (z >> np.uint64(27))) * np.uint64(0x94D049BB133111EB)
        z = z ^ (z >> np.uint64(31))
    return (z >> np.uint64(11)).astype(np.float64) * 2.0 ** -53


def gaussian(seed: int, n: int) -> np.ndarray:
    """n standard normals by Box-Muller on the splitmix64 stream."""
    u = splitmix64_u01(seed, 2 * n)
    return np.sqrt(-2.0 * np.log1p(-u[0::2])) * np.cos(2.0 * np.pi * u[1::2])


def uniform(seed: int, n: int, lo: float = -1.0, hi: float = 1.0) -> np.ndarray:
    """Rng(seed).uniform(lo, hi) x n (core.hpp:59)."""
    return lo + (hi - lo) * splitmix64_u01(seed, n)
