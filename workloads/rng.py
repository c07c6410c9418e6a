"""SplitMix64, the one named, portable PRNG every generator in this repo uses.

SPEC S:420 / S:424 ask for "a named, seedable, portable PRNG" with "defined
integer-draw semantics" so corpora regenerate byte-identically everywhere.
SplitMix64 (Steele, Lea, Flood 2014) is counter-based: value i of stream
``seed`` is ``mix(seed + (i+1) * GAMMA)``, so it vectorises in NumPy.

Integer draws are defined exactly (no floating point):
  * ``ints(n, lo, hi)``   -> lo + ((u >> 32) * (hi-lo+1) >> 32)     (inclusive)
  * ``bernoulli(n, p)``   -> (u >> 11) < round(p * 2**53)

This module holds no arithmetic of the RANC method; it only makes numbers.
"""
from __future__ import annotations

import numpy as np

GAMMA = np.uint64(0x9E3779B97F4A7C15)
_M1 = np.uint64(0xBF58476D1CE4E5B9)
_M2 = np.uint64(0x94D049BB133111EB)


def _mix(z: np.ndarray) -> np.ndarray:
    z = (z ^ (z >> np.uint64(30))) * _M1
    z = (z ^ (z >> np.uint64(27))) * _M2
    return z ^ (z >> np.uint64(31))


class SplitMix64:
    """A SplitMix64 stream; successive calls consume successive counters."""

    def __init__(self, seed: int):
        self.seed = np.uint64(seed & 0xFFFFFFFFFFFFFFFF)
        self.counter = 0

    def u64(self, n: int) -> np.ndarray:
        n = int(n)
        with np.errstate(over="ignore"):
            idx = np.arange(self.counter + 1, self.counter + 1 + n, dtype=np.uint64)
            out = _mix(self.seed + idx * GAMMA)
        self.counter += n
        return out

    def ints(self, n: int, lo: int, hi: int) -> np.ndarray:
        """n integers uniform on [lo, hi] (inclusive), int64."""
        span = np.uint64(hi - lo + 1)
        u = self.u64(n) >> np.uint64(32)
        with np.errstate(over="ignore"):
            v = (u * span) >> np.uint64(32)
        return v.astype(np.int64) + lo

    def bernoulli(self, n: int, p: float) -> np.ndarray:
        thr = np.uint64(int(round(p * (1 << 53))))
        return (self.u64(n) >> np.uint64(11)) < thr

    def choice_bits(self, shape, p: float) -> np.ndarray:
        size = int(np.prod(shape)) if len(shape) else 1
        return self.bernoulli(size, p).reshape(shape)

    def permutation(self, n: int) -> np.ndarray:
        """Fisher-Yates with the defined integer draws."""
        perm = np.arange(n, dtype=np.int64)
        for i in range(n - 1, 0, -1):
            j = int(self.ints(1, 0, i)[0])
            perm[i], perm[j] = perm[j], perm[i]
        return perm


def substream(seed: int, name: str) -> SplitMix64:
    """Deterministic named sub-stream: seed mixed with a stable hash of name."""
    h = 1469598103934665603
    for ch in name.encode():
        h = ((h ^ ch) * 1099511628211) & 0xFFFFFFFFFFFFFFFF
    base = SplitMix64(seed ^ h)
    return SplitMix64(int(base.u64(1)[0]))
