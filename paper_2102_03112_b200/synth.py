"""Synthetic gradients of the benchmark configurations (BASELINE.md §3 inputs).

g_w[i] = (float) CounterRng(hash64(w, hash64(0xBE7C, seed))).normal() — the
reference CLI's bench generator (gradpack_main.cpp:279-281) extended with the
rank, vectorised with numpy: draw i of a CounterRng stream is
mix64(seed + (i+1) * gamma), and normal() consumes two draws (rng.hpp:62-69).
NCF-style natural sparsity zeroes whole 64-wide rows with probability 0.4
(stream hash64(w, hash64(0x0DCF, seed))).
"""
from __future__ import annotations

import numpy as np

from .dp import hash64

GAMMA = np.uint64(0x9E3779B97F4A7C15)


def _mix64(z: np.ndarray) -> np.ndarray:
    z = z ^ (z >> np.uint64(30))
    z = z * np.uint64(0xBF58476D1CE4E5B9)
    z = z ^ (z >> np.uint64(27))
    z = z * np.uint64(0x94D049BB133111EB)
    return z ^ (z >> np.uint64(31))


def _draws(seed: int, start: int, n: int) -> np.ndarray:
    pos = np.arange(start + 1, start + n + 1, dtype=np.uint64)
    with np.errstate(over="ignore"):
        return _mix64(np.uint64(seed) + pos * GAMMA)


def _unit(seed: int, start: int, n: int) -> np.ndarray:
    return (_draws(seed, start, n) >> np.uint64(11)).astype(np.float64) * (2.0 ** -53)


def normal_f32(seed: int, n: int, chunk: int = 1 << 22) -> np.ndarray:
    out = np.empty(n, dtype=np.float32)
    for b in range(0, n, chunk):
        m = min(chunk, n - b)
        u = _unit(seed, 2 * b, 2 * m)
        u1 = 1.0 - u[0::2]
        u2 = u[1::2]
        out[b:b + m] = (np.sqrt(-2.0 * np.log(u1)) * np.cos(2.0 * np.pi * u2)).astype(np.float32)
    return out


def gradient(d: int, rank: int = 0, seed: int = 1) -> np.ndarray:
    return normal_f32(hash64(rank, hash64(0xBE7C, seed)), d)


def natural_sparse_gradient(d: int, rank: int = 0, seed: int = 1, zero_frac: float = 0.4,
                            row: int = 64) -> np.ndarray:
    g = gradient(d, rank, seed)
    rows = (d + row - 1) // row
    u = _unit(hash64(rank, hash64(0x0DCF, seed)), 0, rows)
    mask = np.repeat(u < zero_frac, row)[:d]
    g[mask] = 0.0
    return g


def _mix64_t(z):
    import torch
    m30, m27, m31 = (1 << 34) - 1, (1 << 37) - 1, (1 << 33) - 1
    z = z ^ ((z >> 30) & m30)
    z = z * -4658895280553007687  # 0xBF58476D1CE4E5B9 as int64
    z = z ^ ((z >> 27) & m27)
    z = z * -7723592293110705685  # 0x94D049BB133111EB as int64
    return z ^ ((z >> 31) & m31)


def _as_i64(x: int) -> int:
    x &= (1 << 64) - 1
    return x - (1 << 64) if x >= 1 << 63 else x


def gradient_torch(d: int, rank: int = 0, seed: int = 1, device="cuda", chunk: int = 1 << 24):
    """The same generator on the GPU (int64 two's-complement = u64 arithmetic,
    logical shifts by masking).  fp64 log/cos are the device's, so a rare
    element may differ from the host generator in the last f32 bit; used for
    benchmark inputs only (parity tests use the host/oracle generator)."""
    import torch
    s = _as_i64(hash64(rank, hash64(0xBE7C, seed)))
    g = _as_i64(0x9E3779B97F4A7C15)
    out = torch.empty(d, dtype=torch.float32, device=device)
    for b in range(0, d, chunk):
        m = min(chunk, d - b)
        pos = torch.arange(2 * b + 1, 2 * (b + m) + 1, dtype=torch.int64, device=device)
        z = _mix64_t(pos * g + s)
        u = ((z >> 11) & ((1 << 53) - 1)).to(torch.float64) * (2.0 ** -53)
        u1 = 1.0 - u[0::2]
        u2 = u[1::2]
        out[b:b + m] = (torch.sqrt(-2.0 * torch.log(u1)) * torch.cos(2.0 * np.pi * u2)).to(torch.float32)
    return out
