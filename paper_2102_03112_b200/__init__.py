"""paper_2102_03112_b200 — B200-native DeepReduce sparse-gradient encode → exchange → decode.

A drop-in for the reference's compressor path (gradpack: top_r,
compress_gradient, pack, unpack, decompress_gradient, FORMAT.md wire format),
computed by hand-written sm_100a kernels in libgradpack_b200.so behind the
C-ABI of include/gradpack_b200.h.

The device API is loaded lazily (PEP 562): ``import paper_2102_03112_b200.seeds``
or ``.inputs`` (pure host helpers) does not load the CUDA library, while any
attribute of the API below does — and fails loudly when the library is missing.
"""
_API = (
    "CapacityError", "ChecksumError", "Codec", "CorruptPayloadError", "CudaError", "DecodeError", "Error", "FitError",
    "IndexMethod", "PipelineConfig", "TruncatedError", "UnknownMethodError", "UnsupportedMethodError", "ValueMethod",
    "bloom_params", "volume",
)
__all__ = list(_API)


def __getattr__(name):
    if name in _API:
        from . import api
        return getattr(api, name)
    raise AttributeError(f"module {__name__!r} has no attribute {name!r}")
