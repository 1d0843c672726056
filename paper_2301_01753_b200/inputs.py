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


def gaussian_ids(seed: int, ids: np.ndarray) -> np.ndarray:
    """Entries `ids` of gaussian(seed, n): a rank can draw its part of a global
    vector without generating the rest."""
    ids = np.asarray(ids, dtype=np.uint64)
    k = np.empty(2 * ids.size, dtype=np.uint64)
    k[0::2] = 2 * ids
    k[1::2] = 2 * ids + np.uint64(1)
    with np.errstate(over="ignore"):
        z = np.uint64(seed) + (k + np.uint64(1)) * _GOLDEN
        z = (z ^ (z >> np.uint64(30))) * np.uint64(0xBF58476D1CE4E5B9)
        z = (z ^ (z >> np.uint64(27))) * np.uint64(0x94D049BB133111EB)
        z = z ^ (z >> np.uint64(31))
    u = (z >> np.uint64(11)).astype(np.float64) * 2.0 ** -53
    return np.sqrt(-2.0 * np.log1p(-u[0::2])) * np.cos(2.0 * np.pi * u[1::2])


_GL3 = ((0.5 - 0.5 * np.sqrt(0.6), 5.0 / 18.0), (0.5, 8.0 / 18.0),
        (0.5 + 0.5 * np.sqrt(0.6), 5.0 / 18.0))


def pulse_params(seed: int, npulses: int = 1):
    """Seeded centres x0 in [0.3, 0.7]^3 and unit polarisations p of the
    Gaussian pulses (configs 3 and 5): u-stream entries 6k..6k+2 give x0,
    Box-Muller normals 3k..3k+2 of stream seed+1 give p (normalised)."""
    u = splitmix64_u01(seed, 6 * npulses)
    g = gaussian(seed + 1, 3 * npulses)
    out = []
    for k in range(npulses):
        x0 = 0.3 + 0.4 * u[6 * k:6 * k + 3]
        p = g[3 * k:3 * k + 3]
        out.append((x0, p / np.linalg.norm(p)))
    return out


def pulse_one_form(xyz, edge_vertices, seed: int, sigma: float = 0.1, npulses: int = 1):
    """Canonical projection of A = sum_k exp(-|x - x0_k|^2 / (2 sigma^2)) p_k
    onto edges: a_e = int_e A . dx, 3-point Gauss-Legendre along the edge
    (the integral DOF of the P1 rule, reference form_space.cpp:410-429)."""
    xa = xyz[edge_vertices[:, 0]]
    xb = xyz[edge_vertices[:, 1]]
    d = xb - xa
    a = np.zeros(len(edge_vertices))
    for x0, p in pulse_params(seed, npulses):
        tang = d @ p
        for s, w in _GL3:
            x = xa + s * d
            r2 = np.sum((x - x0) ** 2, axis=1)
            a += w * np.exp(-r2 / (2.0 * sigma * sigma)) * tang
    return a


def uniform(seed: int, n: int, lo: float = -1.0, hi: float = 1.0) -> np.ndarray:
    """Rng(seed).uniform(lo, hi) x n (core.hpp:59)."""
    return lo + (hi - lo) * splitmix64_u01(seed, n)
