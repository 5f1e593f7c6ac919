"""Rademacher probe q_1 = s(seed, i)/sqrt(P)  (oracle; test infrastructure only).

PAPER.md P:312-316 (§4, SLQ with "random probes"); BASELINE north star: "a bit-identical
counter-based Rademacher probe generator on both sides".  The paper fixes no hash, so this
follows SURVEY.md §8(c2) reading #3/#4:

    s(seed, i) = -1 if top bit of splitmix64(splitmix64(seed) XOR i) is set, else +1
    splitmix64(x): x += 0x9E3779B97F4A7C15; z = (x ^ (x>>30)) * 0xBF58476D1CE4E5B9;
                   z = (z ^ (z>>27)) * 0x94D049BB133111EB; return z ^ (z>>31)   (mod 2^64)

i is the global canonical parameter index; P counts real parameters (no padding).
"""
from __future__ import annotations

import numpy as np

_M64 = (1 << 64) - 1


def splitmix64_int(x: int) -> int:
    """Scalar reference in Python integers (mod 2^64)."""
    x = (x + 0x9E3779B97F4A7C15) & _M64
    z = ((x ^ (x >> 30)) * 0xBF58476D1CE4E5B9) & _M64
    z = ((z ^ (z >> 27)) * 0x94D049BB133111EB) & _M64
    return z ^ (z >> 31)


def splitmix64(x: np.ndarray) -> np.ndarray:
    """Vectorised splitmix64 over uint64 (numpy uint64 arithmetic wraps mod 2^64)."""
    x = np.asarray(x, dtype=np.uint64)
    with np.errstate(over="ignore"):
        x = x + np.uint64(0x9E3779B97F4A7C15)
        z = (x ^ (x >> np.uint64(30))) * np.uint64(0xBF58476D1CE4E5B9)
        z = (z ^ (z >> np.uint64(27))) * np.uint64(0x94D049BB133111EB)
    return z ^ (z >> np.uint64(31))


def signs(seed: int, n: int, first: int = 0) -> np.ndarray:
    """s(seed, i) for i = first .. first+n-1, as float64 +-1."""
    key = np.uint64(splitmix64_int(seed & _M64))
    i = np.arange(first, first + n, dtype=np.uint64)
    top = splitmix64(key ^ i) >> np.uint64(63)
    return np.where(top == 1, -1.0, 1.0)


def rademacher_probe(seed: int, P: int) -> np.ndarray:
    """q_1 = s(seed, i)/sqrt(P), fp64, unit norm up to rounding."""
    return signs(seed, P) / np.sqrt(float(P))
