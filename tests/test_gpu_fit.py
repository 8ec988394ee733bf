"""Value codec (fit-poly) parity on the B200, through the C-ABI.

Bit-exact: sort map / reorder payload, sign split, segment bounds, degree,
index payload, and every decode of a given container (fp64 Horner without
FMA).  Tolerance (north star): the f32 fit coefficients,
|dc| <= 1e-5 |c| + 1e-6 * max|c_segment|, and values reconstructed from a
GPU-encoded container, |dv| <= 1e-5 * max|v|.
"""
import struct

import numpy as np
import pytest
import torch

from oracle.bindings import GpConfig, synthetic_gradient

pytestmark = pytest.mark.gpu

BITMAP, P0, P2, PD = 1, 4, 6, 7
V_FIT = 1


@pytest.fixture(scope="module")
def codec():
    from paper_2102_03112_b200 import Codec
    c = Codec(max_d=1 << 22)
    yield c
    c.close()


def _dev(b):
    return torch.from_numpy(np.frombuffer(b, np.uint8).copy()).cuda()


def _split(c: bytes):
    il, vl, rl = struct.unpack_from("<QQQ", c, 25)
    idx = c[49:49 + il]
    val = c[49 + il:49 + il + vl]
    reo = c[49 + il + vl:49 + il + vl + rl]
    return c[:49], idx, val, reo


def _fit_fields(v: bytes):
    S = struct.unpack_from("<H", v, 1)[0]
    bounds = struct.unpack_from(f"<{S}I", v, 3)
    deg = v[3 + 4 * S]
    coeffs = np.frombuffer(v[4 + 4 * S:len(v) - 4], "<f4").reshape(S, deg + 1)
    l = struct.unpack_from("<I", v, len(v) - 4)[0]
    return v[0], S, bounds, deg, coeffs, l


def _check_container(got: bytes, want: bytes, oracle):
    gh, gi, gv, gr = _split(got)
    wh, wi, wv, wr = _split(want)
    assert gh[:49] == wh[:49], "header (lengths, methods, d, r)"
    assert gi == wi, "index payload"
    assert gr == wr, "reorder payload"
    gk, gS, gb, gd, gc, gl = _fit_fields(gv)
    wk, wS, wb, wd, wc, wl = _fit_fields(wv)
    assert (gk, gS, gb, gd, gl) == (wk, wS, wb, wd, wl), "fit structure"
    scale = np.abs(wc).max(axis=1, keepdims=True)
    assert np.all(np.abs(gc - wc) <= 1e-5 * np.abs(wc) + 1e-6 * scale), (gc, wc)
    # values reconstructed from the GPU container vs from the oracle container
    _, s1, v1 = oracle.decode(got)
    _, s2, v2 = oracle.decode(want)
    assert np.array_equal(s1, s2)
    assert np.max(np.abs(v1 - v2)) <= 1e-5 * max(1e-30, np.abs(v2).max())


@pytest.mark.parametrize("im", [BITMAP, P0, 5, P2, PD])
def test_fit_encode_matches_oracle(codec, oracle, im):
    from paper_2102_03112_b200 import PipelineConfig
    for d, r, fpr, deg, ms in [(1000, 10, 0.01, 5, 0), (65539, 655, 0.001, 5, 0), (269722, 2697, 0.01, 3, 0),
                               (1_000_000, 10_000, 0.01, 5, 0), (1_000_000, 10_000, 0.001, 5, 8),
                               (300_000, 3_000, 0.01, 1, 0), (20_000, 200, 0.01, 0, 4)]:
        g = synthetic_gradient(d, rank=d % 11)
        cfg = PipelineConfig(index_method=im, value_method=V_FIT, fpr=fpr, degree=deg, max_segments=ms, seed=d)
        got = codec.compress(torch.from_numpy(g).cuda(), r, cfg).cpu().numpy().tobytes()
        want = oracle.encode_dense(g, r, GpConfig.make(im, V_FIT, fpr=fpr, degree=deg, max_segments=ms, seed=d))
        _check_container(got, want, oracle)


def test_fit_scaled_and_positive_only(codec, oracle):
    from paper_2102_03112_b200 import PipelineConfig
    for scale, absval in [(1e-3, False), (1e3, False), (1.0, True)]:
        g = synthetic_gradient(200_000, rank=5) * np.float32(scale)
        if absval:
            g = np.abs(g)
        cfg = PipelineConfig(index_method=BITMAP, value_method=V_FIT, seed=3)
        got = codec.compress(torch.from_numpy(g).cuda(), 2000, cfg).cpu().numpy().tobytes()
        want = oracle.encode_dense(g, 2000, GpConfig.make(BITMAP, V_FIT, seed=3))
        _check_container(got, want, oracle)


@pytest.mark.parametrize("im", [BITMAP, P0, P2])
def test_fit_decode_bit_exact(codec, oracle, im):
    for d, r, deg, ms in [(5000, 50, 5, 0), (269722, 2697, 5, 0), (1_000_000, 10_000, 2, 6)]:
        g = synthetic_gradient(d, rank=1)
        c = oracle.encode_dense(g, r, GpConfig.make(im, V_FIT, fpr=0.01, degree=deg, max_segments=ms, seed=9))
        gd, sup, val = codec.decompress(_dev(c))
        od, osup, oval = oracle.decode(c)
        assert gd == od and np.array_equal(sup.cpu().numpy().astype(np.uint32), osup)
        assert np.array_equal(val.cpu().numpy(), oval)


def test_fit_decode_errors(codec, oracle):
    from oracle.bindings import OracleError
    from paper_2102_03112_b200 import Error
    g = synthetic_gradient(5000, rank=4)
    c = oracle.encode_dense(g, 60, GpConfig.make(BITMAP, V_FIT, seed=1))
    _, il, vl, rl = 0, *struct.unpack_from("<QQQ", c, 25)
    vo = 49 + il
    muts = []
    for pos in [vo, vo + 1, vo + 3, vo + vl - 1, vo + vl - 4, 49 + il + vl]:  # kind, S, bound, split, reorder
        b = bytearray(c)
        b[pos] ^= 0x40
        body = bytes(b[49:-4])
        b[-4:] = struct.pack("<I", oracle.crc32c(body))  # re-seal so the CRC passes
        muts.append(bytes(b))
    for bad in muts:
        try:
            oracle.decode(bad)
            continue  # mutation happened to stay valid
        except OracleError as oe:
            kind = oe.kind
        dense = torch.zeros(5000, dtype=torch.float32, device="cuda")
        with pytest.raises(Error) as ge:
            codec.decode_accumulate(_dev(bad), dense)
            codec.status()
        assert type(ge.value).__name__ == kind
        assert float(dense.abs().sum()) == 0.0
