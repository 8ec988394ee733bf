"""Synthetic benchmark gradients, generated on the host.

g_w[i] = (float) CounterRng(hash64(w, hash64(0xBE7C, seed))).normal() — the
reference CLI's bench generator (tools/gradpack_main.cpp:279-281) extended
with the rank; NCF-style natural sparsity zeroes 64-wide rows with
probability 0.4 (stream hash64(w, hash64(0x0DCF, seed))).  The arithmetic is
csrc/inputs.c (libm log/cos, as the reference build), run on all host cores
over independent slices — CounterRng is counter based, so element i depends
only on (seed, i).  The same bytes feed the device arm (uploaded once), the
CPU reference arm and the committed goldens (tests/golden/), so the bench's
containers can be compared with the reference's.

Loads only libgp_inputs.so (plain C), never the CUDA library.
"""
from __future__ import annotations

import ctypes as C
import os
import subprocess
from concurrent.futures import ThreadPoolExecutor

import numpy as np

from .seeds import hash64

HERE = os.path.dirname(os.path.abspath(__file__))
SRC = os.path.join(HERE, "csrc", "inputs.c")
LIB = os.path.join(HERE, "libgp_inputs.so")


def build() -> str:
    if not os.path.exists(LIB) or os.path.getmtime(LIB) < os.path.getmtime(SRC):
        subprocess.run(["gcc", "-std=c11", "-O2", "-fPIC", "-shared", "-ffp-contract=off", SRC, "-o", LIB, "-lm"],
                       check=True)
    return LIB


_lib = None


def _l():
    global _lib
    if _lib is None:
        if not os.path.exists(LIB):
            build()
        L = C.CDLL(LIB)
        L.gpi_fill_normal_f32.argtypes = [C.c_uint64, C.c_uint64, C.c_void_p, C.c_uint64]
        L.gpi_fill_normal_f32.restype = None
        L.gpi_zero_rows.argtypes = [C.c_uint64, C.c_uint64, C.c_void_p, C.c_uint64, C.c_uint64, C.c_double]
        L.gpi_zero_rows.restype = None
        _lib = L
    return _lib


def _parallel(fn, n: int, chunk: int = 1 << 21) -> None:
    spans = [(b, min(chunk, n - b)) for b in range(0, n, chunk)]
    if len(spans) <= 1:
        for b, m in spans:
            fn(b, m)
        return
    with ThreadPoolExecutor(max_workers=min(len(spans), os.cpu_count() or 1)) as pool:
        list(pool.map(lambda s: fn(*s), spans))  # ctypes releases the GIL


def gradient_seed(rank: int = 0, seed: int = 1) -> int:
    return hash64(rank, hash64(0xBE7C, seed))


def normal_f32(stream_seed: int, n: int, first: int = 0) -> np.ndarray:
    """(float) CounterRng(stream_seed).normal() numbers [first, first + n)."""
    L = _l()
    out = np.empty(n, dtype=np.float32)
    base = out.ctypes.data
    _parallel(lambda b, m: L.gpi_fill_normal_f32(stream_seed, first + b, base + 4 * b, m), n)
    return out


def gradient(d: int, rank: int = 0, seed: int = 1, first: int = 0) -> np.ndarray:
    """Elements [first, first + d) of rank `rank`'s N(0,1) f32 gradient."""
    return normal_f32(gradient_seed(rank, seed), d, first)


def natural_sparse_gradient(d: int, rank: int = 0, seed: int = 1, zero_frac: float = 0.4, row: int = 64,
                            first: int = 0) -> np.ndarray:
    """The C3 input: the rank's gradient with whole 64-wide rows zeroed (support = nonzeros)."""
    g = gradient(d, rank, seed, first)
    L = _l()
    zs = hash64(rank, hash64(0x0DCF, seed))
    base = g.ctypes.data
    _parallel(lambda b, m: L.gpi_zero_rows(zs, first + b, base + 4 * b, m, row, zero_frac), d)
    return g
