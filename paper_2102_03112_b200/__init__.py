"""paper_2102_03112_b200 — B200-native DeepReduce sparse-gradient encode → exchange → decode.

A drop-in for the reference's compressor path (gradpack: top_r,
compress_gradient, pack, unpack, decompress_gradient, FORMAT.md wire format),
computed by hand-written sm_100a kernels in libgradpack_b200.so behind the
C-ABI of include/gradpack_b200.h.
"""
from .api import (  # noqa: F401
    CapacityError, ChecksumError, Codec, CorruptPayloadError, CudaError, DecodeError, Error, FitError,
    IndexMethod, PipelineConfig, TruncatedError, UnknownMethodError, UnsupportedMethodError, ValueMethod,
    bloom_params, volume,
)
