"""Container helpers shared by the config-size golden generator
(tools/make_config_goldens.py) and its parity tests (tests/test_gpu_configs.py).
TEST INFRASTRUCTURE ONLY.  Layouts: FORMAT.md "Container" and "Fit payload"."""
from __future__ import annotations

import hashlib
import json
import os
import struct

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
GOLDEN = os.path.join(HERE, "golden", "configs.json")


def sha(b) -> str:
    if isinstance(b, np.ndarray):
        b = np.ascontiguousarray(b).tobytes()
    return hashlib.sha256(bytes(b)).hexdigest()


def split(c: bytes) -> dict:
    """Header fields and payload slices of a packed container (container.cpp:58-82)."""
    assert c[:4] == b"DRC1"
    ver, im, vm, flags = struct.unpack_from("<HBBB", c, 4)
    d, r, il, vl, rl = struct.unpack_from("<QQQQQ", c, 9)
    o = 49
    return dict(version=ver, index_method=im, value_method=vm, flags=flags, d=d, r=r, il=il, vl=vl, rl=rl,
                header=c[:49], index=c[o:o + il], value=c[o + il:o + il + vl],
                reorder=c[o + il + vl:o + il + vl + rl], crc=c[o + il + vl + rl:o + il + vl + rl + 4])


def parse_fit(p: bytes) -> dict:
    """serialize_fit layout (curvefit.cpp:285-298)."""
    kind = p[0]
    (S,) = struct.unpack_from("<H", p, 1)
    bounds = list(struct.unpack_from(f"<{S}I", p, 3))
    o = 3 + 4 * S
    degree = p[o]
    cps = degree + 1 if kind == 0 else 4
    coeffs = np.frombuffer(p, dtype="<f4", count=S * cps, offset=o + 1).reshape(S, cps).astype(np.float64)
    (l,) = struct.unpack_from("<I", p, o + 1 + 4 * S * cps)
    return dict(kind=kind, S=S, bounds=bounds, degree=degree, coeffs=coeffs, l=l)


def repack(parts: dict, value: bytes, crc32c) -> bytes:
    """The container with its value payload replaced (header lengths and CRC redone)."""
    h = bytearray(parts["header"])
    struct.pack_into("<Q", h, 33, len(value))
    body = bytes(parts["index"]) + bytes(value) + bytes(parts["reorder"])
    return bytes(h) + body + struct.pack("<I", crc32c(body))


def load() -> dict:
    with open(GOLDEN) as f:
        return json.load(f)


def coeff_close(a: np.ndarray, b: np.ndarray) -> bool:
    """SURVEY §8(a) exactness contract for f32 fit coefficients:
    |Δc| <= 1e-5·|c_ref| + 1e-6·max|c_seg| (the absolute floor covers cancellation)."""
    tol = 1e-5 * np.abs(b) + 1e-6 * np.abs(b).max(axis=1, keepdims=True)
    return bool(np.all(np.abs(a - b) <= tol))
