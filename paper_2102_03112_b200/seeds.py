"""Seed derivations of the reference's worker loop — pure Python, no CUDA.

Kept free of imports of the device library so that the CPU reference arm of
bench.py and the golden generator can use them without loading
libgradpack_b200.so.
"""
from __future__ import annotations

import math

GAMMA = 0x9E3779B97F4A7C15
MASK = (1 << 64) - 1


def mix64(z: int) -> int:
    """SplitMix64 finalizer (rng.hpp:25-31)."""
    z &= MASK
    z ^= z >> 30
    z = (z * 0xBF58476D1CE4E5B9) & MASK
    z ^= z >> 27
    z = (z * 0x94D049BB133111EB) & MASK
    return z ^ (z >> 31)


def hash64(x: int, seed: int) -> int:
    """rng.hpp:35-37"""
    return mix64((x ^ ((seed + GAMMA) & MASK)) & MASK)


def pipeline_seed(seed: int, worker: int, step: int) -> int:
    """Simulation::pipeline_seed (harness.cpp:201-203) over Problem::batch_seed (:47-51)."""
    key = ((worker & 0xFFFFFFFF) << 32) | (step & 0xFFFFFFFF)
    return hash64(0xC0DEC, hash64(key, hash64(0xDA7A, seed)))


def bucket_seed(seed: int, worker: int, step: int, bucket: int) -> int:
    """Seed of bucket b in the bucketed (C5) convention of dp.BucketedSparseAllgather."""
    return hash64(bucket, pipeline_seed(seed, worker, step))


def ratio_r(d: int, ratio: float) -> int:
    """r = max(1, llround(ratio * d)) (harness.cpp:212)."""
    x = ratio * d
    return max(1, int(math.floor(x + 0.5)))


def bucket_bounds(d: int, buckets: int) -> list[tuple[int, int]]:
    """[lo, hi) of each bucket: the first d % buckets buckets take one extra element."""
    base, rem = divmod(d, buckets)
    out, at = [], 0
    for b in range(buckets):
        n = base + (1 if b < rem else 0)
        out.append((at, at + n))
        at += n
    return out
