"""Error feedback (memory compensation) — test infrastructure only.

CPU restatement of the compensation lines of the reference worker loop, in the
f32 arithmetic of the device path (gp_encode_topr_ef):

  harness.cpp:230      input = g + residual            -> fl32(g + e)
  harness.cpp:242-251  top_r(input) + compress_gradient(sg, cfg, &input) + pack
  harness.cpp:257-258  unpack + decompress_gradient + to_dense
  harness.cpp:269-271  residual = input - decoded      -> fl32(input[s] - fl32(v_s))
                                                          on the decoded support,
                                                          input elsewhere

The reference keeps `input` and `residual` in f64 (Eigen VectorXd); this
path is f32 end to end (its gradients are f32), so the restatement is the
harness semantics at f32 precision.  `codec` is a CpuCodec: the C oracle or
the reference build (oracle/_ref), which must agree bit for bit.
"""
from __future__ import annotations

import numpy as np


def ef_step(codec, g: np.ndarray, e: np.ndarray, r: int, cfg) -> tuple[bytes, np.ndarray]:
    """One worker's compensated encode: returns (container bytes, new residual)."""
    inp = (np.asarray(g, np.float32) + np.asarray(e, np.float32)).astype(np.float32)
    c = codec.encode_dense(inp, r, cfg)
    return c, residual_after(codec, inp, c)


def residual_after(codec, inp: np.ndarray, container: bytes) -> np.ndarray:
    """input - to_dense(decode(container)) with one f32 rounding per coordinate."""
    _, sup, val = codec.decode(container)
    res = np.array(inp, np.float32, copy=True)
    res[sup] = (inp[sup] - val.astype(np.float32)).astype(np.float32)
    return res
