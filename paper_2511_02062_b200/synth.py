"""Host-side generator of synthetic queries / query tokens: numpy restatement of
include/vx_synth.h (bit-identical to the device fill of the index and token store).
Used by the bench and the smoke run to build query batches on the host."""
from __future__ import annotations

import numpy as np


def _splitmix64(x: np.ndarray) -> np.ndarray:
    with np.errstate(over="ignore"):
        x = x + np.uint64(0x9E3779B97F4A7C15)
        x = (x ^ (x >> np.uint64(30))) * np.uint64(0xBF58476D1CE4E5B9)
        x = (x ^ (x >> np.uint64(27))) * np.uint64(0x94D049BB133111EB)
        return x ^ (x >> np.uint64(31))


def mult(dist: int, dim: int) -> np.ndarray:
    """vx_synth_mult: integer column multipliers of distribution dist (1: anisotropic)."""
    c = np.arange(dim, dtype=np.int64)
    if dist == 0:
        return np.ones(dim, np.int64)
    m = 1 + 32 // (1 + c // 4)
    return np.where(c % 97 == 13, 4 * m, m)


def rows(seed: int, row0: int, n: int, dim: int, dist: int = 0) -> np.ndarray:
    """Rows [row0, row0+n) of the unit-norm synthetic matrix, fp32 [n][dim]."""
    r = np.arange(row0, row0 + n, dtype=np.uint64)[:, None]
    c = np.arange(dim, dtype=np.uint64)[None, :]
    with np.errstate(over="ignore"):
        h = _splitmix64(np.uint64(seed) * np.uint64(0x9E3779B97F4A7C15) + r)
        h = _splitmix64(h ^ (c * np.uint64(0xD1B54A32D192ED03)))
    m = np.uint64(0xFFFF)
    v = ((h & m) + ((h >> np.uint64(16)) & m) + ((h >> np.uint64(32)) & m)
         + (h >> np.uint64(48))).astype(np.int64) - 131070
    v = v * mult(dist, dim)[None, :]
    nrm = np.sqrt((v * v).sum(axis=1).astype(np.float64))
    return (v.astype(np.float64) / nrm[:, None]).astype(np.float32)


def queries(B: int, dim: int, seed: int = 43, dist: int = 0) -> np.ndarray:
    return rows(seed, 0, B, dim, dist)


def query_tokens(B: int, nq: int, dim: int, seed: int = 44) -> np.ndarray:
    return rows(seed, 0, B * nq, dim).reshape(B, nq, dim)
