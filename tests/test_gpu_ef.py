"""Error feedback on the device (gp_encode_topr_ef) vs the CPU oracle.

Bit-exact: container bytes (every non-fit method; fit coefficients are a
tolerance artefact, see test_gpu_fit.py) and the new residual, which must equal
fl32(input - fl32(v)) on the container's decoded support (decoded by the
oracle) and the input elsewhere — for all methods, fit included, since the
residual is defined by the container actually sent.
"""
import numpy as np
import pytest
import torch

from oracle.bindings import GpConfig, synthetic_gradient
from oracle.ef import residual_after

pytestmark = pytest.mark.gpu

NONE, BITMAP, RLE, P0, P1, P2, PD, NAIVE = 0, 1, 2, 4, 5, 6, 7, 8
V_NONE, V_FIT, V_F64 = 0, 1, 5
CASES = [(BITMAP, V_NONE), (RLE, V_NONE), (NONE, V_F64), (BITMAP, V_FIT), (P0, V_FIT), (P1, V_NONE),
         (P2, V_FIT), (P2, V_NONE), (PD, V_NONE), (NAIVE, V_NONE), (NAIVE, V_FIT), (BITMAP, 3), (P2, 3), (RLE, 4)]


@pytest.fixture(scope="module")
def codec():
    from paper_2102_03112_b200 import Codec
    c = Codec(max_d=1 << 20)
    yield c
    c.close()


@pytest.mark.parametrize("im,vm", CASES)
def test_ef_steps_bit_exact(codec, oracle, im, vm):
    from paper_2102_03112_b200 import PipelineConfig
    d, r = 200_003, 2_000
    kw = dict(slot_codec=0) if vm == 4 else {}
    cfg = PipelineConfig(index_method=im, value_method=vm, fpr=0.01, seed=21, **kw)
    ocfg = GpConfig.make(im, vm, fpr=0.01, seed=21, **kw)
    e = torch.zeros(d, dtype=torch.float32, device="cuda")
    for step in range(3):
        g = synthetic_gradient(d, rank=step + 1)
        e_prev = e.cpu().numpy()
        inp = (g + e_prev).astype(np.float32)
        c = codec.compress_ef(torch.from_numpy(g).cuda(), e, r, cfg).cpu().numpy().tobytes()
        if vm != V_FIT:
            assert c == oracle.encode_dense(inp, r, ocfg), f"step {step}: container bytes differ"
        want = residual_after(oracle, inp, c)
        got = e.cpu().numpy()
        assert np.array_equal(got, want), f"step {step}: residual differs at {np.flatnonzero(got != want)[:5]}"


def test_ef_matches_plain_encode_then_decode(codec):
    """The own-container shortcut (no index replay) equals encode + full decode."""
    from paper_2102_03112_b200 import PipelineConfig
    d, r = 300_000, 3_000
    cfg = PipelineConfig(index_method=P2, value_method=V_FIT, fpr=0.001, seed=3)
    g = torch.from_numpy(synthetic_gradient(d, rank=2)).cuda()
    e0 = torch.from_numpy(synthetic_gradient(d, rank=3) * np.float32(0.05)).cuda()
    e = e0.clone()
    c_ef = codec.compress_ef(g, e, r, cfg)
    inp = g + e0
    c = codec.compress(inp, r, cfg)
    assert torch.equal(c, c_ef)
    want = inp.clone()
    codec.decode_accumulate(c, want, scale=-1.0)
    codec.status()
    assert torch.equal(e, want)
