"""The reference's f64 value semantics on the device, against the reference
build (oracle/_ref):

* gp_encode_topr_ef64 — the compensated worker step of Simulation::step in
  f64 (harness.cpp:230 input = g + residual, :242-251 top_r + compress +
  pack, :257-258 decode, :269-271 residual = input - decoded; residual_ is a
  VectorXd, gradient.hpp:29).  Three steps per method: containers
  byte-identical and residuals bit-identical to the reference loop (fit
  methods: structure exact, coefficients within the SURVEY §8(a) tolerance,
  and the residual bit-identical to input - decode(the device's container)).
* gp_encode_sparse — compress_gradient(sg, cfg, dense) with Vector values that
  are not f32-representable (pipeline.cpp:146-221), with and without the dense
  vector (Bloom policies: gather_values, pipeline.cpp:38-54).
"""
import numpy as np
import pytest
import torch

from golden_util import coeff_close, parse_fit, split
from oracle.bindings import GpConfig, synthetic_gradient

pytestmark = pytest.mark.gpu

NONE, BITMAP, RLE, HUFF, P0, P1, P2, PD, NAIVE = 0, 1, 2, 3, 4, 5, 6, 7, 8
V_NONE, V_FIT, V_QUANT, V_SLOT, V_F64 = 0, 1, 3, 4, 5
CASES = [(BITMAP, V_NONE), (RLE, V_NONE), (NONE, V_F64), (HUFF, V_NONE), (BITMAP, V_FIT), (P0, V_FIT),
         (P1, V_NONE), (P2, V_FIT), (P2, V_NONE), (PD, V_NONE), (NAIVE, V_NONE), (NAIVE, V_FIT), (BITMAP, V_QUANT),
         (P2, V_QUANT), (RLE, V_SLOT)]


@pytest.fixture(scope="module")
def codec():
    from paper_2102_03112_b200 import Codec
    c = Codec(max_d=1 << 20)
    yield c
    c.close()


def _cfgs(im, vm, seed):
    from paper_2102_03112_b200 import PipelineConfig
    kw = dict(slot_codec=0) if vm == V_SLOT else {}
    return (PipelineConfig(index_method=im, value_method=vm, fpr=0.01, seed=seed, **kw),
            GpConfig.make(im, vm, fpr=0.01, seed=seed, **kw))


def _fit_close(a: bytes, b: bytes):
    p, q = split(a), split(b)
    assert p["header"][:9] == q["header"][:9] and p["index"] == q["index"] and p["reorder"] == q["reorder"]
    fa, fb = parse_fit(p["value"]), parse_fit(q["value"])
    for k in ("kind", "S", "bounds", "degree", "l"):
        assert fa[k] == fb[k], k
    assert coeff_close(fa["coeffs"], fb["coeffs"])


@pytest.mark.parametrize("im,vm", CASES)
def test_ef64_steps_match_the_reference_loop(codec, reference, im, vm):
    d, r = 200_003, 2_000
    e_ref = np.zeros(d, np.float64)
    e = torch.zeros(d, dtype=torch.float64, device="cuda")
    for step in range(3):
        cfg, ocfg = _cfgs(im, vm, seed=21 + step)
        g = synthetic_gradient(d, rank=step + 1)
        e_prev = e.cpu().numpy()
        want = reference.ef_step64(g, e_ref, r, ocfg)  # e_ref <- the reference's new residual
        got = codec.compress_ef64(torch.from_numpy(g).cuda(), e, r, cfg).cpu().numpy().tobytes()
        e_got = e.cpu().numpy()
        if vm == V_FIT:
            _fit_close(got, want)
            # the residual of the container actually sent, in f64
            _, sup, val = reference.decode(got)
            want_e = g.astype(np.float64) + e_prev
            want_e[sup] = want_e[sup] - val
            assert np.array_equal(e_got, want_e), f"step {step}: residual differs"
            e_ref = e_got.copy()  # carry the device's state (the fits differ within tolerance)
        else:
            assert got == want, f"step {step}: container differs"
            assert np.array_equal(e_got, e_ref), f"step {step}: residual differs at {np.flatnonzero(e_got != e_ref)[:5]}"


def test_ef64_top_r_uses_f64_order(codec, reference):
    """Inputs whose f32 roundings tie but whose f64 values do not: the
    selection follows the f64 order (harness.cpp:242 on a VectorXd)."""
    d, r = 100_000, 1_000
    g = np.full(d, 1.0, np.float32)
    res = np.zeros(d, np.float64)
    res[::7] = 1e-12 * np.arange(res[::7].size)  # below f32 resolution at 1.0
    cfg, ocfg = _cfgs(NONE, V_F64, seed=3)
    e = torch.from_numpy(res.copy()).cuda()
    got = codec.compress_ef64(torch.from_numpy(g).cuda(), e, r, cfg).cpu().numpy().tobytes()
    want = reference.ef_step64(g, res, r, ocfg)
    assert got == want
    assert np.array_equal(e.cpu().numpy(), res)


SPARSE_CASES = [(NONE, V_NONE), (NONE, V_F64), (BITMAP, V_NONE), (RLE, V_F64), (HUFF, V_NONE), (BITMAP, V_FIT),
                (BITMAP, V_QUANT), (RLE, V_SLOT), (P0, V_NONE), (P1, V_F64), (P2, V_QUANT), (P2, V_FIT),
                (PD, V_NONE), (NAIVE, V_F64)]


@pytest.mark.parametrize("im,vm", SPARSE_CASES)
@pytest.mark.parametrize("with_dense", [False, True])
def test_encode_sparse_f64_values(codec, reference, im, vm, with_dense):
    rng = np.random.default_rng(im * 10 + vm)
    d, r = 50_003, 500
    sup = np.sort(rng.choice(d, size=r, replace=False)).astype(np.uint32)
    dense = rng.standard_normal(d)                  # full-precision doubles
    vals = dense[sup] * (1.0 + 1e-3 * rng.standard_normal(r))  # sg values differ from the dense ones
    cfg, ocfg = _cfgs(im, vm, seed=77)
    want = reference.encode_sparse64(d, sup, vals, ocfg, dense=dense if with_dense else None)
    got = codec.compress_sparse(d, torch.from_numpy(sup.astype(np.int32)).cuda(), torch.from_numpy(vals).cuda(),
                                cfg, dense=torch.from_numpy(dense).cuda() if with_dense else None)
    got = got.cpu().numpy().tobytes()
    if vm == V_FIT:
        _fit_close(got, want)
    else:
        assert got == want


def test_encode_sparse_empty_support(codec, reference):
    """compress_gradient of an empty support: legal for index NONE with raw
    values (pipeline.cpp:152-154), an Error otherwise."""
    from paper_2102_03112_b200 import Error
    empty_i = torch.zeros(0, dtype=torch.int32, device="cuda")
    empty_v = torch.zeros(0, dtype=torch.float64, device="cuda")
    for vm in (V_NONE, V_F64):
        cfg, ocfg = _cfgs(NONE, vm, seed=1)
        got = codec.compress_sparse(10, empty_i, empty_v, cfg).cpu().numpy().tobytes()
        assert got == reference.encode_sparse64(10, np.zeros(0, np.uint32), np.zeros(0), ocfg)
    for im, vm in ((BITMAP, V_NONE), (NONE, V_FIT)):
        cfg, _ = _cfgs(im, vm, seed=1)
        with pytest.raises(Error):
            codec.compress_sparse(10, empty_i, empty_v, cfg)
