"""ctypes bindings for the CPU checkers (TEST INFRASTRUCTURE ONLY).

Loads oracle/liboracle.so (the C restatement, gp_oracle.c) and, when it was
built, oracle/_ref/libgpref.so (the unmodified reference sources, see
oracle/Makefile).  Both export the same entry points under the prefixes
``gpo_`` and ``gpr_``; :class:`CpuCodec` wraps either one.

Only tests/, __graft_entry__.smoke() and bench.py's CPU legs may import this
module, and only as the checker / the timed CPU baseline.
"""
from __future__ import annotations

import ctypes as C
import os

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
ORACLE_SO = os.path.join(HERE, "liboracle.so")
REF_SO = os.path.join(HERE, "_ref", "libgpref.so")

GP_STATUS = {
    0: "OK", 1: "Error", 2: "DecodeError", 3: "TruncatedError", 4: "ChecksumError",
    5: "UnknownMethodError", 6: "CorruptPayloadError", 7: "FitError", 8: "CudaError",
    9: "Unsupported", 10: "Capacity",
}


class GpConfig(C.Structure):
    """gp_pipeline_config (include/gradpack_b200.h), mirror of PipelineConfig."""

    _fields_ = [
        ("index_method", C.c_uint8), ("value_method", C.c_uint8), ("pd_variant", C.c_uint8),
        ("slot_codec", C.c_uint8), ("degree", C.c_int32), ("max_segments", C.c_int32),
        ("quant_bits", C.c_int32), ("quant_bucket", C.c_uint32), ("fpr", C.c_double),
        ("seed", C.c_uint64),
    ]

    @classmethod
    def make(cls, index_method=0, value_method=0, fpr=0.01, degree=5, max_segments=0, seed=0,
             pd_variant=0, slot_codec=1, quant_bits=7, quant_bucket=512):
        return cls(index_method, value_method, pd_variant, slot_codec, degree, max_segments,
                   quant_bits, quant_bucket, fpr, seed)


class OracleError(Exception):
    def __init__(self, code: int, msg: str):
        super().__init__(f"{GP_STATUS.get(code, code)}: {msg}")
        self.code = code
        self.kind = GP_STATUS.get(code, str(code))


def _u8p(a):
    return a.ctypes.data_as(C.POINTER(C.c_uint8))


_P = C.POINTER
_u8 = C.c_uint8
_u32 = C.c_uint32
_u64 = C.c_uint64


class CpuCodec:
    """One of the two CPU checkers; prefix 'gpo' (restatement) or 'gpr' (reference)."""

    def __init__(self, path: str, prefix: str):
        self.path = path
        self.prefix = prefix
        self.lib = C.CDLL(path)
        L, p = self.lib, prefix
        self._f = {}

        def bind(name, argtypes, restype=C.c_int):
            fn = getattr(L, f"{p}_{name}")
            fn.argtypes = argtypes
            fn.restype = restype
            self._f[name] = fn

        bind("last_error", [], C.c_char_p)
        bind("free", [C.c_void_p], None)
        bind("top_r", [_P(C.c_float), _u64, _u64, _P(_u32)])
        bind("bloom_params", [C.c_double, _u64, _P(_u64), _P(_u32)])
        bind("crc32c", [_P(_u8), C.c_size_t], C.c_uint32)
        bind("bloom_build", [_P(_u32), _u64, C.c_double, _u64, _u64, _P(_P(_u8)), _P(C.c_size_t)])
        bind("positive_scan", [_P(_u8), C.c_size_t, _u64, _P(_P(_u32)), _P(_u64)])
        bind("bloom_select", [_P(_u8), C.c_size_t, _u64, _u64, C.c_int, _P(_P(_u32))])
        bind("conflict_sets", [_P(_u8), C.c_size_t, _u64, _P(_P(_u64)), _P(_P(_u64)),
                               _P(_P(_u32)), _P(_u64)])
        bind("value_compress", [_P(C.c_double), _u64, C.c_int, C.c_int, _P(_P(_u8)),
                                _P(C.c_size_t), _P(_P(_u32)), _P(_u64)])
        bind("compress_pack", [_u64, _P(_u32), _P(C.c_double), _u64, _P(C.c_float),
                               _P(GpConfig), _P(_P(_u8)), _P(C.c_size_t)])
        bind("encode_dense", [_P(C.c_float), _u64, _u64, _P(GpConfig), _P(_P(_u8)),
                              _P(C.c_size_t)])
        bind("decode", [_P(_u8), C.c_size_t, _P(_u64), _P(_P(_u32)), _P(_P(C.c_double)),
                        _P(_u64)])
        bind("decode_accumulate", [_P(_u8), C.c_size_t, _P(C.c_double), _u64, C.c_double])
        if prefix == "gpr":
            bind("volume", [_P(_u8), C.c_size_t, _P(_u64)])
            bind("random_r", [_u64, _u64, _u64, _P(_u32)])
            bind("encode_sparse64", [_u64, _P(_u32), _P(C.c_double), _u64, _P(C.c_double), _P(GpConfig),
                                     _P(_P(_u8)), _P(C.c_size_t)])
            bind("ef_step64", [_P(C.c_float), _P(C.c_double), _u64, _u64, _P(GpConfig), _P(_P(_u8)),
                               _P(C.c_size_t)])
        if prefix == "gpo":
            bind("rle_encode", [_P(_u32), _u64, _u64, _P(_P(_u8)), _P(C.c_size_t)])
            bind("bitmap_bytes", [_P(_u32), _u64, _u64, _P(_u8)])
            bind("mix64", [_u64], _u64)
            bind("hash64", [_u64, _u64], _u64)
            bind("pipeline_seed", [_u64, C.c_int, C.c_int], _u64)
            bind("rng_below_seq", [_u64, _u64, _u64, _P(_u64)])
            bind("fill_normal_f32", [_u64, _P(C.c_float), _u64], None)

    # ------------------------------------------------------------ helpers
    def _check(self, rc):
        if rc != 0:
            raise OracleError(rc, self._f["last_error"]().decode(errors="replace"))

    def _take(self, ptr, n, dtype):
        """Copy a malloc'd output array into numpy and free it."""
        n = int(n)
        if n == 0 or not ptr:
            if ptr:
                self._f["free"](C.cast(ptr, C.c_void_p))
            return np.zeros(0, dtype=dtype)
        ct = np.ctypeslib.as_ctypes_type(np.dtype(dtype))
        arr = np.ctypeslib.as_array(C.cast(ptr, C.POINTER(ct)), shape=(n,)).copy()
        self._f["free"](C.cast(ptr, C.c_void_p))
        return arr

    # ------------------------------------------------------------ API
    def top_r(self, g: np.ndarray, r: int) -> np.ndarray:
        g = np.ascontiguousarray(g, dtype=np.float32)
        out = np.zeros(r, dtype=np.uint32)
        self._check(self._f["top_r"](g.ctypes.data_as(_P(C.c_float)), g.size, r,
                                     out.ctypes.data_as(_P(_u32))))
        return out

    def random_r(self, d: int, r: int, seed: int) -> np.ndarray:
        """random_r (sparsify.cpp:48-58) with CounterRng(seed): the sorted support (reference build only)."""
        out = np.zeros(r, dtype=np.uint32)
        self._check(self._f["random_r"](d, r, seed, out.ctypes.data_as(_P(_u32))))
        return out

    def bloom_params(self, eps: float, r: int):
        m, k = _u64(), _u32()
        self._check(self._f["bloom_params"](eps, r, C.byref(m), C.byref(k)))
        return m.value, k.value

    def crc32c(self, data: bytes) -> int:
        a = np.frombuffer(bytes(data), dtype=np.uint8).copy() if len(data) else np.zeros(1, np.uint8)
        return int(self._f["crc32c"](_u8p(a), len(data)))

    def bloom_build(self, support, eps, seed_a, seed_b) -> bytes:
        s = np.ascontiguousarray(support, dtype=np.uint32)
        p, n = _P(_u8)(), C.c_size_t()
        self._check(self._f["bloom_build"](s.ctypes.data_as(_P(_u32)), s.size, eps, seed_a,
                                           seed_b, C.byref(p), C.byref(n)))
        return self._take(p, n.value, np.uint8).tobytes()

    def positive_scan(self, filt: bytes, d: int) -> np.ndarray:
        a = np.frombuffer(filt, dtype=np.uint8).copy()
        p, n = _P(_u32)(), _u64()
        self._check(self._f["positive_scan"](_u8p(a), a.size, d, C.byref(p), C.byref(n)))
        return self._take(p, n.value, np.uint32)

    def bloom_select(self, filt: bytes, d: int, r: int, index_method: int) -> np.ndarray:
        a = np.frombuffer(filt, dtype=np.uint8).copy()
        p = _P(_u32)()
        self._check(self._f["bloom_select"](_u8p(a), a.size, d, r, index_method, C.byref(p)))
        return self._take(p, r, np.uint32)

    def conflict_sets(self, filt: bytes, d: int):
        a = np.frombuffer(filt, dtype=np.uint8).copy()
        b, o, m, ns = _P(_u64)(), _P(_u64)(), _P(_u32)(), _u64()
        self._check(self._f["conflict_sets"](_u8p(a), a.size, d, C.byref(b), C.byref(o),
                                             C.byref(m), C.byref(ns)))
        bits = self._take(b, ns.value, np.uint64)
        offs = self._take(o, ns.value + 1, np.uint64)
        mem = self._take(m, int(offs[-1]) if offs.size else 0, np.uint32)
        return bits, offs, mem

    def value_compress(self, v: np.ndarray, degree=5, max_segments=0):
        v = np.ascontiguousarray(v, dtype=np.float64)
        f, fl, mp, ml = _P(_u8)(), C.c_size_t(), _P(_u32)(), _u64()
        self._check(self._f["value_compress"](v.ctypes.data_as(_P(C.c_double)), v.size, degree,
                                              max_segments, C.byref(f), C.byref(fl), C.byref(mp),
                                              C.byref(ml)))
        return self._take(f, fl.value, np.uint8).tobytes(), self._take(mp, ml.value, np.uint32)

    def compress_pack(self, d, support, cfg: GpConfig, values=None, dense=None) -> bytes:
        s = np.ascontiguousarray(support, dtype=np.uint32)
        vp = None
        if values is not None:
            values = np.ascontiguousarray(values, dtype=np.float64)
            vp = values.ctypes.data_as(_P(C.c_double))
        dp = None
        if dense is not None:
            dense = np.ascontiguousarray(dense, dtype=np.float32)
            dp = dense.ctypes.data_as(_P(C.c_float))
        p, n = _P(_u8)(), C.c_size_t()
        self._check(self._f["compress_pack"](d, s.ctypes.data_as(_P(_u32)), vp, s.size, dp,
                                             C.byref(cfg), C.byref(p), C.byref(n)))
        return self._take(p, n.value, np.uint8).tobytes()

    def encode_dense(self, g: np.ndarray, r: int, cfg: GpConfig) -> bytes:
        g = np.ascontiguousarray(g, dtype=np.float32)
        p, n = _P(_u8)(), C.c_size_t()
        self._check(self._f["encode_dense"](g.ctypes.data_as(_P(C.c_float)), g.size, r,
                                            C.byref(cfg), C.byref(p), C.byref(n)))
        return self._take(p, n.value, np.uint8).tobytes()

    def encode_sparse64(self, d: int, support, values, cfg: GpConfig, dense=None) -> bytes:
        """compress_gradient(sg, cfg, dense) + pack with f64 values (reference build only)."""
        s = np.ascontiguousarray(support, dtype=np.uint32)
        v = np.ascontiguousarray(values, dtype=np.float64)
        dp = None
        if dense is not None:
            dense = np.ascontiguousarray(dense, dtype=np.float64)
            dp = dense.ctypes.data_as(_P(C.c_double))
        p, n = _P(_u8)(), C.c_size_t()
        self._check(self._f["encode_sparse64"](d, s.ctypes.data_as(_P(_u32)), v.ctypes.data_as(_P(C.c_double)),
                                               s.size, dp, C.byref(cfg), C.byref(p), C.byref(n)))
        return self._take(p, n.value, np.uint8).tobytes()

    def ef_step64(self, g: np.ndarray, residual: np.ndarray, r: int, cfg: GpConfig) -> bytes:
        """One compensated worker step in f64 (harness.cpp:230-271); `residual` (f64) is updated in place."""
        g = np.ascontiguousarray(g, dtype=np.float32)
        assert residual.dtype == np.float64 and residual.flags.c_contiguous
        p, n = _P(_u8)(), C.c_size_t()
        self._check(self._f["ef_step64"](g.ctypes.data_as(_P(C.c_float)),
                                         residual.ctypes.data_as(_P(C.c_double)), g.size, r, C.byref(cfg),
                                         C.byref(p), C.byref(n)))
        return self._take(p, n.value, np.uint8).tobytes()

    def decode(self, data: bytes):
        """unpack + decompress_gradient → (d, support u32, values f64)."""
        a = np.frombuffer(bytes(data), dtype=np.uint8).copy() if len(data) else np.zeros(1, np.uint8)
        d, s, v, n = _u64(), _P(_u32)(), _P(C.c_double)(), _u64()
        self._check(self._f["decode"](_u8p(a), len(data), C.byref(d), C.byref(s), C.byref(v),
                                      C.byref(n)))
        return d.value, self._take(s, n.value, np.uint32), self._take(v, n.value, np.float64)

    def decode_accumulate(self, data: bytes, dense: np.ndarray, scale: float = 1.0):
        a = np.frombuffer(bytes(data), dtype=np.uint8).copy()
        assert dense.dtype == np.float64 and dense.flags.c_contiguous
        self._check(self._f["decode_accumulate"](_u8p(a), a.size,
                                                 dense.ctypes.data_as(_P(C.c_double)), dense.size,
                                                 scale))

    def volume(self, data: bytes) -> dict:
        """volume() of a packed container (reference build only)."""
        a = np.frombuffer(bytes(data), dtype=np.uint8).copy()
        out = np.zeros(7, dtype=np.uint64)
        self._check(self._f["volume"](_u8p(a), a.size, out.ctypes.data_as(_P(_u64))))
        keys = ["index_bits", "value_bits", "reorder_bits", "metadata_bits", "total_bits"]
        rep = {k: int(v) for k, v in zip(keys, out[:5])}
        rep["ratio_dense"], rep["ratio_sparse"] = out[5:7].view(np.float64).tolist()
        return rep

    # restatement-only helpers
    def rle_encode(self, support, d) -> bytes:
        s = np.ascontiguousarray(support, dtype=np.uint32)
        p, n = _P(_u8)(), C.c_size_t()
        self._check(self._f["rle_encode"](s.ctypes.data_as(_P(_u32)), s.size, d, C.byref(p),
                                          C.byref(n)))
        return self._take(p, n.value, np.uint8).tobytes()

    def bitmap_bytes(self, support, d) -> bytes:
        s = np.ascontiguousarray(support, dtype=np.uint32)
        out = np.zeros((d + 7) // 8, dtype=np.uint8)
        self._check(self._f["bitmap_bytes"](s.ctypes.data_as(_P(_u32)), s.size, d, _u8p(out)))
        return out.tobytes()

    def mix64(self, x):
        return int(self._f["mix64"](x))

    def hash64(self, x, seed):
        return int(self._f["hash64"](x, seed))

    def pipeline_seed(self, seed, worker, step):
        return int(self._f["pipeline_seed"](seed, worker, step))

    def below_seq(self, seed, bound, n):
        out = np.zeros(n, dtype=np.uint64)
        self._check(self._f["rng_below_seq"](seed, bound, n, out.ctypes.data_as(_P(_u64))))
        return out

    def normal_f32(self, seed, n):
        out = np.zeros(n, dtype=np.float32)
        self._f["fill_normal_f32"](seed, out.ctypes.data_as(_P(C.c_float)), n)
        return out


_cache = {}


def oracle() -> CpuCodec:
    """The C restatement (always available once `make -C oracle` ran)."""
    if "gpo" not in _cache:
        if not os.path.exists(ORACLE_SO):
            raise FileNotFoundError(f"{ORACLE_SO} missing: run `make -C oracle` (or build())")
        _cache["gpo"] = CpuCodec(ORACLE_SO, "gpo")
    return _cache["gpo"]


def reference() -> CpuCodec | None:
    """The reference's own sources built in oracle/_ref, or None when absent."""
    if "gpr" not in _cache:
        _cache["gpr"] = CpuCodec(REF_SO, "gpr") if os.path.exists(REF_SO) else None
    return _cache["gpr"]


def synthetic_gradient(d: int, rank: int = 0, seed: int = 1) -> np.ndarray:
    """Rank-w synthetic gradient (BASELINE.md §3 inputs):
    g_w[i] = (float) CounterRng(hash64(w, hash64(0xBE7C, seed))).normal()."""
    o = oracle()
    return o.normal_f32(o.hash64(rank, o.hash64(0xBE7C, seed)), d)
