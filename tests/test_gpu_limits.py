"""Reference-legal inputs at the edges of the wire format, on the device.

* Fit degrees 8..60 (fit_poly accepts [0, 60], curvefit.cpp:130) and models of
  more than 64 segments (part_budget caps at 0xffff, curvefit.cpp:424-428;
  serialize_fit at 0xffff, :287): the device decodes containers the
  reference build (oracle/_ref) wrote bit for bit, and its own encode of the
  same values has the reference's model structure (kind, segment bounds,
  degree, sign split — fp64 segmentation is exact) with reconstructed values
  within tolerance.  Coefficients are compared only where the problem is
  well conditioned (degree 8): the reference solves a monomial Vandermonde
  system with column-pivoted QR, which at high degree is ill-conditioned, so
  two correct solvers agree only in the values they reproduce.
* Conflict sets of more than 254 members (conflict_sets keeps them in an
  unbounded std::map, bloom.cpp:156-173): P2 containers whose filter is so
  small that hundreds of positives share every bit, encoded and decoded bit
  for bit against the oracle.
"""
import numpy as np
import pytest
import torch

from golden_util import coeff_close, parse_fit, split
from oracle.bindings import GpConfig, synthetic_gradient

pytestmark = pytest.mark.gpu

NONE, BITMAP, P2 = 0, 1, 6
V_FIT = 1


@pytest.fixture(scope="module")
def codec():
    from paper_2102_03112_b200 import Codec
    c = Codec(max_d=1 << 21)
    yield c
    c.close()


def _dev(b: bytes):
    return torch.from_numpy(np.frombuffer(b, np.uint8).copy()).cuda()


def _decode_equal(codec, cpu, c: bytes):
    d, sup, val = codec.decompress(_dev(c))
    od, osup, oval = cpu.decode(c)
    assert d == od
    assert np.array_equal(sup.cpu().numpy().astype(np.uint32), osup)
    assert np.array_equal(val.cpu().numpy(), oval)
    return osup, oval


FIT_CASES = [  # (d, r, scale, degree, max_segments)
    (100_003, 1_000, 1.0, 8, 0),
    (100_003, 1_000, 1.0, 8, 40),
    (200_003, 4_000, 1e4, 5, 0),      # part_budget > 64 on each sign part
    (200_003, 4_000, 1e4, 8, 0),
    (200_003, 4_000, 1.0, 3, 300),    # a 300-segment cap split across the parts
    (60_001, 600, 1.0, 12, 0),
    (60_001, 600, 1.0, 20, 4),
    (60_001, 600, 1.0, 60, 0),
]


@pytest.mark.parametrize("d,r,scale,degree,max_segments", FIT_CASES)
def test_fit_wide_models(codec, reference, d, r, scale, degree, max_segments):
    from paper_2102_03112_b200 import PipelineConfig
    g = (synthetic_gradient(d, rank=4) * np.float32(scale)).astype(np.float32)
    for im in (BITMAP, NONE):
        ocfg = GpConfig.make(im, V_FIT, degree=degree, max_segments=max_segments, seed=5)
        ref_c = reference.encode_dense(g, r, ocfg)
        ref_fit = parse_fit(split(ref_c)["value"])
        if scale > 1.0 and max_segments == 0:
            assert ref_fit["S"] > 64, "the case must exercise more than 64 segments"
        if max_segments:
            assert ref_fit["S"] == max_segments
        # the reference's container decodes bit for bit
        _, ref_v = _decode_equal(codec, reference, ref_c)
        # the device's own encode: same structure, values within tolerance
        cfg = PipelineConfig(index_method=im, value_method=V_FIT, degree=degree, max_segments=max_segments, seed=5)
        c = codec.compress(torch.from_numpy(g).cuda(), r, cfg).cpu().numpy().tobytes()
        p, q = split(c), split(ref_c)
        assert p["index"] == q["index"] and p["reorder"] == q["reorder"]
        fit = parse_fit(p["value"])
        for k in ("kind", "S", "bounds", "degree", "l"):
            assert fit[k] == ref_fit[k], k
        if degree <= 8:
            assert coeff_close(fit["coeffs"], ref_fit["coeffs"])
        _, sup, val = codec.decompress(_dev(c))
        v = val.cpu().numpy()
        if degree <= 12:
            assert np.max(np.abs(v - ref_v)) <= 1e-4 * np.max(np.abs(ref_v))
        elif degree <= 20:  # ill-conditioned: both reconstructions follow the data equally well
            y = g[sup.cpu().numpy()].astype(np.float64)
            e_dev, e_ref = np.sqrt(np.mean((v - y) ** 2)), np.sqrt(np.mean((ref_v - y) ** 2))
            assert np.isfinite(e_dev) and e_dev <= 1.5 * e_ref + 1e-6 * np.max(np.abs(y))
        # degree 60 over ~30k-point segments: x^60 in f32 monomials reproduces
        # nothing in either implementation (the reference's own reconstruction
        # error is ~1e34 here); structure and bit-exact decode are the contract


def test_fit_too_many_segments_is_an_error(codec):
    """More than 0xffff segments: serialize_fit's Error (curvefit.cpp:287)."""
    from paper_2102_03112_b200 import Error, PipelineConfig
    d = 300_000
    g = synthetic_gradient(d, rank=2)
    cfg = PipelineConfig(index_method=NONE, value_method=V_FIT, degree=0, max_segments=70_000, seed=1)
    with pytest.raises(Error):
        codec.compress(torch.from_numpy(g).cuda(), d, cfg)


@pytest.mark.parametrize("d,r,fpr", [(300_000, 2_000, 0.8), (200_000, 1_000, 0.9), (1_000_000, 10_000, 0.95)])
def test_p2_large_conflict_sets(codec, oracle, d, r, fpr):
    from paper_2102_03112_b200 import PipelineConfig
    g = synthetic_gradient(d, rank=6)
    sup = oracle.top_r(g, r)
    filt = oracle.bloom_build(sup, fpr, 0x77, 0x99)
    _, offs, _ = oracle.conflict_sets(filt, d)
    assert int(np.diff(offs.astype(np.int64)).max()) >= 255, "the case must build sets of >= 255 members"
    f = _dev(filt)
    got = codec.bloom_select(f, d, r, P2).cpu().numpy().astype(np.uint32)
    assert np.array_equal(got, oracle.bloom_select(filt, d, r, P2))
    for seed in (3, 4):
        cfg = PipelineConfig(index_method=P2, value_method=0, fpr=fpr, seed=seed)
        c = codec.compress(torch.from_numpy(g).cuda(), r, cfg).cpu().numpy().tobytes()
        assert c == oracle.encode_dense(g, r, GpConfig.make(P2, 0, fpr=fpr, seed=seed))
        _decode_equal(codec, oracle, c)
