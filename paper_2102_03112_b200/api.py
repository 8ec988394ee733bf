"""Host-side mirror of gradpack's compressor API over the B200 C-ABI.

Names, argument meaning and error behaviour follow the reference
(/root/reference/proj/include/gradpack/*.hpp):

  reference                                   here
  ------------------------------------------  -----------------------------------------
  IndexMethod / ValueMethod (container.hpp:23) IndexMethod / ValueMethod (same ids)
  PipelineConfig (pipeline.hpp:28-39)          PipelineConfig (same fields, defaults)
  top_r (sparsify.hpp:22)                      Codec.top_r
  compress_gradient + pack (pipeline.hpp:53,   Codec.compress / Codec.compress_support
    container.hpp:65)                            (device tensor in, packed bytes on device out)
  unpack + decompress_gradient (:59, :66)      Codec.decompress
  to_dense + harness mean (harness.cpp:274)    Codec.decode_accumulate
  Error / DecodeError / ... (errors.hpp:21-53)  the same exception classes

Device memory and streams come from torch; torch is plumbing here, every
byte of the path is computed by libgradpack_b200.so.
"""
from __future__ import annotations

import ctypes as C
import enum
from dataclasses import dataclass, field

import torch

from ._lib import GpConfig, GpVolume, lib


# ---------------------------------------------------------------- errors (errors.hpp:21-53)
class Error(RuntimeError):
    """gradpack::Error — base class of every error raised by this library."""


class DecodeError(Error):
    """A byte stream failed structural validation while decoding."""


class TruncatedError(DecodeError):
    """The stream ended before a complete structure could be read."""


class ChecksumError(DecodeError):
    """A stored checksum does not match the recomputed one."""


class UnknownMethodError(DecodeError):
    """A method or codec id is not in the registry."""


class CorruptPayloadError(DecodeError):
    """A payload parsed structurally but violates its own invariants."""


class FitError(Error):
    """An iterative fit failed to converge to a usable model."""


class CudaError(Error):
    """The CUDA runtime failed (no reference equivalent)."""


class UnsupportedMethodError(Error):
    """Method id registered in FORMAT.md but not implemented on the device path."""


class CapacityError(Error):
    """The context workspace or an output buffer is too small."""


_STATUS = {1: Error, 2: DecodeError, 3: TruncatedError, 4: ChecksumError, 5: UnknownMethodError,
           6: CorruptPayloadError, 7: FitError, 8: CudaError, 9: UnsupportedMethodError, 10: CapacityError}


# ---------------------------------------------------------------- method ids (container.hpp:23-43)
class IndexMethod(enum.IntEnum):
    None_ = 0
    Bitmap = 1
    Rle = 2
    Huffman = 3
    BloomP0 = 4
    BloomP1 = 5
    BloomP2 = 6
    BloomPd = 7
    BloomNaive = 8


class ValueMethod(enum.IntEnum):
    None_ = 0
    FitPoly = 1
    FitDexp = 2
    Quant = 3
    DeflateSlot = 4
    RawF64 = 5


@dataclass
class PipelineConfig:
    """gradpack::PipelineConfig (pipeline.hpp:28-39) with the same defaults."""

    index_method: IndexMethod = IndexMethod.None_
    value_method: ValueMethod = ValueMethod.None_
    fpr: float = 0.01
    pd_variant: int = 0
    degree: int = 5
    max_segments: int = 0
    quant_bits: int = 7
    quant_bucket: int = 512
    slot_codec: int = 1
    seed: int = 0

    def to_c(self) -> GpConfig:
        return GpConfig(int(self.index_method), int(self.value_method), int(self.pd_variant),
                        int(self.slot_codec), int(self.degree), int(self.max_segments),
                        int(self.quant_bits), int(self.quant_bucket), float(self.fpr),
                        int(self.seed) & 0xFFFFFFFFFFFFFFFF)


def _ptr(t: torch.Tensor | None):
    return None if t is None else C.c_void_p(t.data_ptr())


def _stream(stream=None):
    s = stream if stream is not None else torch.cuda.current_stream()
    return C.c_void_p(s.cuda_stream)


@dataclass
class Codec:
    """One device context (gp_ctx): a preallocated workspace for gradients of up
    to ``max_d`` elements on ``device``.  All calls enqueue on the current torch
    stream; ``status()`` synchronises and raises the first latched device error."""

    max_d: int
    device: int = 0
    _ctx: C.c_void_p = field(default=None, repr=False)

    def __post_init__(self):
        if not torch.cuda.is_available():
            raise CudaError("no CUDA device: the B200 path has no CPU fallback")
        torch.cuda.set_device(self.device)
        h = C.c_void_p()
        rc = lib.gp_ctx_create(self.device, self.max_d, C.byref(h))
        if rc != 0:
            raise _STATUS.get(rc, Error)(f"gp_ctx_create failed with status {rc}")
        self._ctx = h
        # 8-byte device scratch for container lengths / counts
        self._len = torch.zeros(4, dtype=torch.int64, device=f"cuda:{self.device}")

    def close(self):
        if self._ctx:
            lib.gp_ctx_destroy(self._ctx)
            self._ctx = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    # -------------------------------------------------------------- status
    def _raise(self, rc: int):
        if rc != 0:
            msg = lib.gp_last_error(self._ctx)
            raise _STATUS.get(rc, Error)(msg.decode(errors="replace") if msg else f"status {rc}")

    def status(self, stream=None):
        """Synchronise and raise the first device-side error, if any."""
        self._raise(lib.gp_ctx_status(self._ctx, _stream(stream)))

    @property
    def launches(self) -> int:
        return int(lib.gp_ctx_launch_count(self._ctx))

    def profile(self, on: bool = True):
        """Bracket every pipeline stage with CUDA events on its stream."""
        self._raise(lib.gp_ctx_profile(self._ctx, 1 if on else 0))

    def stage_times(self) -> dict:
        """{stage: (total ms, launches)} recorded since the last call (synchronises)."""
        n = 32
        ms = (C.c_double * n)()
        cnt = (C.c_uint64 * n)()
        self._raise(lib.gp_ctx_stage_times(self._ctx, ms, cnt, n))
        out = {}
        for i in range(n):
            name = lib.gp_stage_name(i)
            if name and cnt[i]:
                out[name.decode()] = (ms[i], int(cnt[i]))
        return out

    def set_seed_source(self, seed: torch.Tensor | None):
        """Read every encode's pipeline seed from the device word ``seed`` (int64,
        1 element) when the step executes — the hook that lets a captured CUDA
        graph replay with a new seed per step.  None restores cfg.seed."""
        if seed is not None:
            assert seed.dtype == torch.int64 and seed.is_cuda and seed.numel() >= 1
        self._raise(lib.gp_ctx_set_seed_source(self._ctx, _ptr(seed)))

    # -------------------------------------------------------------- encode
    @staticmethod
    def max_container_bytes(d: int, r: int, cfg: PipelineConfig) -> int:
        c = cfg.to_c()
        return int(lib.gp_max_container_bytes(d, r, C.byref(c)))

    def encode_into(self, grad: torch.Tensor, r: int, cfg: PipelineConfig, out: torch.Tensor,
                    length: torch.Tensor, support: torch.Tensor | None = None, stream=None):
        """Asynchronous top_r + compress_gradient + pack of ``grad`` (f32, device)
        into ``out`` (u8, device); the byte length lands in ``length`` (int64, device).
        With ``support`` given, that support replaces top_r (compress_gradient(sg, cfg, &dense))."""
        assert grad.dtype == torch.float32 and grad.is_cuda and grad.is_contiguous()
        assert out.dtype == torch.uint8 and out.is_cuda
        c = cfg.to_c()
        if support is None:
            rc = lib.gp_encode_topr(self._ctx, _ptr(grad), grad.numel(), r, C.byref(c), _ptr(out),
                                    out.numel(), _ptr(length), _stream(stream))
        else:
            assert support.dtype == torch.int32 and support.is_cuda
            rc = lib.gp_encode_support(self._ctx, _ptr(grad), grad.numel(), _ptr(support),
                                       support.numel(), C.byref(c), _ptr(out), out.numel(),
                                       _ptr(length), _stream(stream))
        self._raise(rc)

    def encode_ef_into(self, grad: torch.Tensor, residual: torch.Tensor, r: int, cfg: PipelineConfig,
                       out: torch.Tensor, length: torch.Tensor, stream=None):
        """Error-feedback step of the reference worker loop (harness.cpp:230, :250,
        :269-271), asynchronous: input = grad + residual; the container of
        top_r(input) goes to ``out`` (length word in ``length``); ``residual`` is
        overwritten with input - decode(container)."""
        for t in (grad, residual):
            assert t.dtype == torch.float32 and t.is_cuda and t.is_contiguous()
        assert residual.numel() == grad.numel() and out.dtype == torch.uint8 and out.is_cuda
        c = cfg.to_c()
        self._raise(lib.gp_encode_topr_ef(self._ctx, _ptr(grad), _ptr(residual), grad.numel(), r, C.byref(c),
                                          _ptr(out), out.numel(), _ptr(length), _stream(stream)))

    def encode_ef64_into(self, grad: torch.Tensor, residual: torch.Tensor, r: int, cfg: PipelineConfig,
                         out: torch.Tensor, length: torch.Tensor, stream=None):
        """encode_ef_into in the reference's own precision: ``residual`` is f64
        (Simulation::residual_), input = double(grad) + residual, top_r, the value
        codec and residual = input - decoded all in f64."""
        assert grad.dtype == torch.float32 and grad.is_cuda and grad.is_contiguous()
        assert residual.dtype == torch.float64 and residual.is_cuda and residual.is_contiguous()
        assert residual.numel() == grad.numel() and out.dtype == torch.uint8 and out.is_cuda
        c = cfg.to_c()
        self._raise(lib.gp_encode_topr_ef64(self._ctx, _ptr(grad), _ptr(residual), grad.numel(), r, C.byref(c),
                                            _ptr(out), out.numel(), _ptr(length), _stream(stream)))

    def compress_ef64(self, grad: torch.Tensor, residual: torch.Tensor, r: int, cfg: PipelineConfig) -> torch.Tensor:
        """encode_ef64_into, synchronised; returns the packed container (device u8)."""
        out = torch.empty(self.max_container_bytes(grad.numel(), r, cfg), dtype=torch.uint8, device=grad.device)
        self.encode_ef64_into(grad, residual, r, cfg, out, self._len[0:1])
        self.status()
        return out[: int(self._len[0].item())]

    def compress_sparse(self, d: int, support: torch.Tensor, values: torch.Tensor, cfg: PipelineConfig,
                        dense: torch.Tensor | None = None) -> torch.Tensor:
        """compress_gradient(sg, cfg, dense) + pack with the reference's f64 values
        (pipeline.cpp:146-221): ``support`` int32/uint32 [r] strictly increasing,
        ``values`` f64 [r], ``dense`` f64 [d] or None."""
        r = support.numel()
        assert values.dtype == torch.float64 and values.numel() == r
        if dense is not None:
            assert dense.dtype == torch.float64 and dense.numel() == d and dense.is_cuda
        dev = support.device if r else torch.device("cuda")
        out = torch.empty(self.max_container_bytes(d, max(r, 1), cfg), dtype=torch.uint8, device=dev)
        c = cfg.to_c()
        self._raise(lib.gp_encode_sparse(self._ctx, d, _ptr(support) if r else None, _ptr(values) if r else None,
                                         r, _ptr(dense), C.byref(c), _ptr(out), out.numel(), _ptr(self._len[0:1]),
                                         _stream(None)))
        self.status()
        return out[: int(self._len[0].item())]

    def compress_ef(self, grad: torch.Tensor, residual: torch.Tensor, r: int, cfg: PipelineConfig) -> torch.Tensor:
        """encode_ef_into, synchronised; returns the packed container (device u8)."""
        out = torch.empty(self.max_container_bytes(grad.numel(), r, cfg), dtype=torch.uint8, device=grad.device)
        self.encode_ef_into(grad, residual, r, cfg, out, self._len[0:1])
        self.status()
        return out[: int(self._len[0].item())]

    def compress(self, grad: torch.Tensor, r: int, cfg: PipelineConfig,
                 support: torch.Tensor | None = None) -> torch.Tensor:
        """top_r + compress_gradient + pack; returns the packed container (device u8)."""
        d = grad.numel()
        rr = r if support is None else support.numel()
        out = torch.empty(self.max_container_bytes(d, rr, cfg), dtype=torch.uint8, device=grad.device)
        self.encode_into(grad, r, cfg, out, self._len[0:1], support=support)
        self.status()
        return out[: int(self._len[0].item())]

    # -------------------------------------------------------------- decode
    def set_decode_overwrite(self, on: bool):
        """Following decodes write dense = scale * decoded (zeros off the support)
        instead of accumulating — zero + accumulate in one pass."""
        self._raise(lib.gp_ctx_set_decode_overwrite(self._ctx, 1 if on else 0))

    def decode_accumulate(self, container: torch.Tensor, dense: torch.Tensor, scale: float = 1.0,
                          length: int | None = None, hint: PipelineConfig | None = None, stream=None,
                          overwrite: bool = False):
        """Asynchronous unpack + decompress_gradient + dense[support] += scale * values
        (overwrite=True: dense = scale * decoded, zeros elsewhere)."""
        assert dense.dtype == torch.float32 and dense.is_cuda and dense.is_contiguous()
        if overwrite:
            self.set_decode_overwrite(True)
            try:
                return self.decode_accumulate(container, dense, scale, length, hint, stream)
            finally:
                self.set_decode_overwrite(False)
        if isinstance(length, torch.Tensor):  # device length word: fully asynchronous path
            assert hint is not None, "a device-side length needs a dispatch hint"
            c = hint.to_c()
            rc = lib.gp_decode_accumulate_dlen(self._ctx, _ptr(container), container.numel(), _ptr(length),
                                               C.byref(c), _ptr(dense), dense.numel(), float(scale),
                                               _stream(stream))
            self._raise(rc)
            return
        n = container.numel() if length is None else length
        if hint is None:
            rc = lib.gp_decode_accumulate(self._ctx, _ptr(container), n, _ptr(dense), dense.numel(),
                                          float(scale), _stream(stream))
        else:
            c = hint.to_c()
            rc = lib.gp_decode_accumulate_hint(self._ctx, _ptr(container), n, C.byref(c), _ptr(dense),
                                               dense.numel(), float(scale), _stream(stream))
        self._raise(rc)

    def set_index_event(self, event: torch.cuda.Event | None):
        """Encodes record ``event`` once their index payload (the Bloom filter) is final."""
        self._raise(lib.gp_ctx_set_index_event(self._ctx, C.c_void_p(event.cuda_event) if event is not None else None))

    def decode_index_prepare(self, filt: torch.Tensor, d: int, r: int, index_method: int, stream=None):
        """The Bloom index stage (positive scan + selection) of a container's filter
        payload ``filt``, into this context (for decode_accumulate_own)."""
        self._raise(lib.gp_decode_index_prepare(self._ctx, _ptr(filt), filt.numel(), d, r, int(index_method),
                                                _stream(stream)))

    def decode_accumulate_own(self, container: torch.Tensor, dense: torch.Tensor, length: torch.Tensor,
                              hint: PipelineConfig, scale: float = 1.0, stream=None):
        """Decode of a container whose index stage this context prepared."""
        h = hint.to_c()
        self._raise(lib.gp_decode_accumulate_own(self._ctx, _ptr(container), container.numel(), _ptr(length),
                                                 C.byref(h), _ptr(dense), dense.numel(), float(scale),
                                                 _stream(stream)))

    def decode_prepare(self, container: torch.Tensor, length: torch.Tensor, hint: PipelineConfig, stream=None):
        """Asynchronous decode without the final scatter (parse, CRC, index and value
        decode, validation) into this context; ``length`` is the device length word."""
        h = hint.to_c()
        self._raise(lib.gp_decode_prepare(self._ctx, _ptr(container), container.numel(), _ptr(length), C.byref(h),
                                          _stream(stream)))

    def decode_finish(self, container: torch.Tensor, dense: torch.Tensor, scale: float = 1.0, stream=None,
                      overwrite: bool = False):
        """dense[support] += scale * values of the container this context prepared
        (overwrite=True: dense = scale * decoded, zeros elsewhere)."""
        if overwrite:
            self.set_decode_overwrite(True)
            try:
                return self.decode_finish(container, dense, scale, stream)
            finally:
                self.set_decode_overwrite(False)
        self._raise(lib.gp_decode_finish(self._ctx, _ptr(container), _ptr(dense), dense.numel(), float(scale),
                                         _stream(stream)))

    def decompress(self, container: torch.Tensor, length: int | None = None):
        """unpack + decompress_gradient → (d, support int32 tensor, values float64 tensor)."""
        n = container.numel() if length is None else length
        cap = self.max_d
        dev = container.device
        sup = torch.empty(cap, dtype=torch.int32, device=dev)
        val = torch.empty(cap, dtype=torch.float64, device=dev)
        meta = torch.zeros(2, dtype=torch.int64, device=dev)
        rc = lib.gp_decode_sparse(self._ctx, _ptr(container), n, _ptr(sup), _ptr(val), cap,
                                  C.c_void_p(meta.data_ptr()), C.c_void_p(meta.data_ptr() + 8), _stream())
        self._raise(rc)
        self.status()
        cnt, d = (int(x) for x in meta.tolist())
        return d, sup[:cnt], val[:cnt]

    # -------------------------------------------------------------- components
    def top_r(self, grad: torch.Tensor, r: int):
        """top_r (sparsify.cpp:32-46) → (support int32, values f32), ascending support."""
        sup = torch.empty(r, dtype=torch.int32, device=grad.device)
        val = torch.empty(r, dtype=torch.float32, device=grad.device)
        self._raise(lib.gp_top_r(self._ctx, _ptr(grad), grad.numel(), r, _ptr(sup), _ptr(val), _stream()))
        self.status()
        return sup, val

    def crc32c(self, data: torch.Tensor) -> int:
        out = torch.zeros(1, dtype=torch.int64, device=data.device)
        self._raise(lib.gp_crc32c(self._ctx, _ptr(data), data.numel(), _ptr(out), _stream()))
        self.status()
        return int(out.item()) & 0xFFFFFFFF

    def bloom_positive_scan(self, filt: torch.Tensor, d: int) -> torch.Tensor:
        """positive_scan (bloom.cpp:123-128) of a serialized filter (device u8
        tensor, FORMAT.md:58-75) over [0, d) → ascending positives (int32)."""
        out = torch.empty(d, dtype=torch.int32, device=filt.device)
        count = torch.zeros(1, dtype=torch.int64, device=filt.device)
        self._raise(lib.gp_bloom_positive_scan(self._ctx, _ptr(filt), filt.numel(), d, _ptr(out), d, _ptr(count),
                                               _stream()))
        self.status()
        return out[: int(count.item())]

    def bloom_scan_range_into(self, filt: torch.Tensor, d: int, lo: int, hi: int, out: torch.Tensor,
                              count: torch.Tensor, stream=None):
        """Asynchronous positive_scan of a serialized filter over [lo, hi) only:
        the ascending positives (global coordinates) to ``out`` (int32), their
        number to ``count`` (int64, device)."""
        self._raise(lib.gp_bloom_scan_range(self._ctx, _ptr(filt), filt.numel(), d, lo, hi, _ptr(out), out.numel(),
                                            _ptr(count), _stream(stream)))

    def decode_index_from_positions(self, filt: torch.Tensor, d: int, r: int, index_method: int,
                                    positions: torch.Tensor, count: torch.Tensor, stream=None):
        """The decode index stage (selection) from a complete positive list; finish
        with decode_accumulate_own on this context."""
        self._raise(lib.gp_decode_index_from_positions(self._ctx, _ptr(filt), filt.numel(), d, r, int(index_method),
                                                       _ptr(positions), _ptr(count), _stream(stream)))

    def bloom_select(self, filt: torch.Tensor, d: int, r: int, index_method: int) -> torch.Tensor:
        """p1_select / p2_select (bloom.cpp:140-154, :175-222) over the positives
        of a serialized filter, seeded derive_selection_seed(seed_a, seed_b)."""
        out = torch.empty(r, dtype=torch.int32, device=filt.device)
        self._raise(lib.gp_bloom_select(self._ctx, _ptr(filt), filt.numel(), d, r, int(index_method), _ptr(out),
                                        _stream()))
        self.status()
        return out


def pipeline_seed_device(seed_out: torch.Tensor, step: torch.Tensor, seed: int, worker: int, buckets: int = 0,
                         stream=None):
    """seed_out[0] = Simulation::pipeline_seed(seed, worker, step[0]) on the device
    (harness.cpp:201-203), enqueued on ``stream``; with buckets > 0,
    seed_out[b] = hash64(b, that seed) for every bucket."""
    assert seed_out.numel() >= max(1, buckets)
    rc = lib.gp_pipeline_seed_device(_ptr(seed_out), _ptr(step), int(seed) & 0xFFFFFFFFFFFFFFFF, int(worker),
                                     int(buckets), _stream(stream))
    if rc != 0:
        raise _STATUS.get(rc, Error)("gp_pipeline_seed_device failed")


def volume(container: bytes) -> dict:
    """volume (container.cpp:148-243) of a packed container held on the host:
    exact bit accounting; bits per nonzero = total_bits / r."""
    buf = (C.c_uint8 * max(1, len(container))).from_buffer_copy(bytes(container) or b"\0")
    rep = GpVolume()
    rc = lib.gp_volume(buf, len(container), C.byref(rep))
    if rc != 0:
        raise _STATUS.get(rc, Error)(f"volume: status {rc}")
    return {f: getattr(rep, f) for f, _ in GpVolume._fields_}


def bloom_params(epsilon: float, r: int) -> tuple[int, int]:
    """bloom_params (bloom.cpp:22-31) → (m, k)."""
    m, k = C.c_uint64(), C.c_uint32()
    rc = lib.gp_bloom_params(float(epsilon), int(r), C.byref(m), C.byref(k))
    if rc != 0:
        raise Error("bloom_params: epsilon must be in (0, 1) and r >= 1")
    return m.value, k.value
