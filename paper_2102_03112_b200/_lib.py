"""ctypes binding of the in-tree CUDA library (libgradpack_b200.so).

The product path has no CPU fallback: importing this module on a box where
the library was not built raises, and every call fails loudly when no CUDA
device is usable.  Build with ``python -m paper_2102_03112_b200.build``.
"""
from __future__ import annotations

import ctypes as C
import os
import re

HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(HERE, "libgradpack_b200.so")
HEADER = os.path.join(os.path.dirname(HERE), "include", "gradpack_b200.h")

if not os.path.exists(LIB_PATH):
    raise ImportError(f"{LIB_PATH} is missing; build it with `python -m paper_2102_03112_b200.build` "
                      "(the B200 path has no CPU fallback)")


class GpConfig(C.Structure):
    """gp_pipeline_config — POD mirror of gradpack::PipelineConfig (pipeline.hpp:28-39)."""

    _fields_ = [
        ("index_method", C.c_uint8), ("value_method", C.c_uint8), ("pd_variant", C.c_uint8),
        ("slot_codec", C.c_uint8), ("degree", C.c_int32), ("max_segments", C.c_int32),
        ("quant_bits", C.c_int32), ("quant_bucket", C.c_uint32), ("fpr", C.c_double),
        ("seed", C.c_uint64),
    ]


class GpVolume(C.Structure):
    """gp_volume_report — VolumeReport (container.hpp:75-83)."""

    _fields_ = [("index_bits", C.c_uint64), ("value_bits", C.c_uint64), ("reorder_bits", C.c_uint64),
                ("metadata_bits", C.c_uint64), ("total_bits", C.c_uint64), ("ratio_dense", C.c_double),
                ("ratio_sparse", C.c_double)]


_P = C.POINTER
_vp = C.c_void_p
_u64 = C.c_uint64

lib = C.CDLL(LIB_PATH)

_SIGS = {
    "gp_pipeline_config_default": ([_P(GpConfig)], None),
    "gp_ctx_create": ([C.c_int, _u64, _P(_vp)], C.c_int),
    "gp_ctx_destroy": ([_vp], None),
    "gp_last_error": ([_vp], C.c_char_p),
    "gp_ctx_status": ([_vp, _vp], C.c_int),
    "gp_ctx_launch_count": ([_vp], _u64),
    "gp_ctx_profile": ([_vp, C.c_int], C.c_int),
    "gp_ctx_stage_times": ([_vp, _P(C.c_double), _P(_u64), C.c_int], C.c_int),
    "gp_stage_name": ([C.c_int], C.c_char_p),
    "gp_max_container_bytes": ([_u64, _u64, _P(GpConfig)], _u64),
    "gp_encode_topr": ([_vp, _vp, _u64, _u64, _P(GpConfig), _vp, _u64, _vp, _vp], C.c_int),
    "gp_ctx_set_seed_source": ([_vp, _vp], C.c_int),
    "gp_pipeline_seed_device": ([_vp, _vp, _u64, C.c_uint32, C.c_uint32, _vp], C.c_int),
    "gp_encode_topr_ef": ([_vp, _vp, _vp, _u64, _u64, _P(GpConfig), _vp, _u64, _vp, _vp], C.c_int),
    "gp_encode_support": ([_vp, _vp, _u64, _vp, _u64, _P(GpConfig), _vp, _u64, _vp, _vp], C.c_int),
    "gp_encode_topr_ef64": ([_vp, _vp, _vp, _u64, _u64, _P(GpConfig), _vp, _u64, _vp, _vp], C.c_int),
    "gp_encode_sparse": ([_vp, _u64, _vp, _vp, _u64, _vp, _P(GpConfig), _vp, _u64, _vp, _vp], C.c_int),
    "gp_decode_accumulate": ([_vp, _vp, _u64, _vp, _u64, C.c_float, _vp], C.c_int),
    "gp_decode_accumulate_hint": ([_vp, _vp, _u64, _P(GpConfig), _vp, _u64, C.c_float, _vp], C.c_int),
    "gp_decode_accumulate_dlen": ([_vp, _vp, _u64, _vp, _P(GpConfig), _vp, _u64, C.c_float, _vp], C.c_int),
    "gp_ctx_set_index_event": ([_vp, _vp], C.c_int),
    "gp_ctx_set_decode_overwrite": ([_vp, C.c_int], C.c_int),
    "gp_decode_index_prepare": ([_vp, _vp, _u64, _u64, _u64, C.c_int, _vp], C.c_int),
    "gp_decode_accumulate_own": ([_vp, _vp, _u64, _vp, _P(GpConfig), _vp, _u64, C.c_float, _vp], C.c_int),
    "gp_decode_prepare": ([_vp, _vp, _u64, _vp, _P(GpConfig), _vp], C.c_int),
    "gp_decode_finish": ([_vp, _vp, _vp, _u64, C.c_float, _vp], C.c_int),
    "gp_decode_sparse":([_vp, _vp, _u64, _vp, _vp, _u64, _vp, _vp, _vp], C.c_int),
    "gp_top_r": ([_vp, _vp, _u64, _u64, _vp, _vp, _vp], C.c_int),
    "gp_crc32c": ([_vp, _vp, _u64, _vp, _vp], C.c_int),
    "gp_bloom_positive_scan": ([_vp, _vp, _u64, _u64, _vp, _u64, _vp, _vp], C.c_int),
    "gp_bloom_select": ([_vp, _vp, _u64, _u64, _u64, C.c_int, _vp, _vp], C.c_int),
    "gp_bloom_scan_range": ([_vp, _vp, _u64, _u64, _u64, _u64, _vp, _u64, _vp, _vp], C.c_int),
    "gp_decode_index_from_positions": ([_vp, _vp, _u64, _u64, _u64, C.c_int, _vp, _vp, _vp], C.c_int),
    "gp_volume": ([_vp, _u64, _P(GpVolume)], C.c_int),
    "gp_bloom_params": ([C.c_double, _u64, _P(_u64), _P(C.c_uint32)], C.c_int),
}

for _name, (_args, _res) in _SIGS.items():
    _fn = getattr(lib, _name)
    _fn.argtypes = _args
    _fn.restype = _res


def header_symbols() -> list[str]:
    """Every function the C-ABI header declares (for the export-table test)."""
    with open(HEADER) as f:
        text = f.read()
    return sorted(set(re.findall(r"^GP_API\s+[\w\s\*]+?\b(gp_\w+)\s*\(", text, flags=re.M)))
