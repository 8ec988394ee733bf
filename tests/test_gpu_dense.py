"""The dense-selection fast path (csrc/dense.cu) against the CPU oracle.

Encode: bitmap + raw f32 with r >= d/4 runs the speculative one-pass nonzero
encoder; when r equals the nonzero count its container must be the oracle's
byte for byte, and when it does not (the speculation misses) the general
top-r path must produce the oracle's container instead.  Decode: bitmap + raw
containers decode through the fused count/scan/scatter path, bit-exact in
accumulate and overwrite mode, and with the reference's error classes (no
dense write on a failed popcount check)."""
import numpy as np
import pytest
import torch

from oracle.bindings import GpConfig, OracleError, synthetic_gradient

pytestmark = pytest.mark.gpu

BITMAP, V_NONE, V_F64 = 1, 0, 5


@pytest.fixture(scope="module")
def codec():
    from paper_2102_03112_b200 import Codec
    c = Codec(max_d=1 << 21)
    yield c
    c.close()


def _cfg(im, vm, seed=3):
    from paper_2102_03112_b200 import PipelineConfig
    return PipelineConfig(index_method=im, value_method=vm, seed=seed)


def _sparse(d, frac, rank, row=64, neg_zero=False):
    g = synthetic_gradient(d, rank=rank)
    rng = np.random.default_rng(rank)
    rows = (d + row - 1) // row
    g[np.repeat(rng.random(rows) < frac, row)[:d]] = 0.0
    if neg_zero:  # -0.0 is a zero key (|g| = 0): never selected while r = nnz
        z = np.flatnonzero(g == 0)
        g[z[::3]] = np.float32(-0.0)
    return g


CASES = [(8192, 0.4, 1), (8193, 0.4, 2), (100_003, 0.4, 3), (1_000_000, 0.4, 4), (1_048_576, 0.0, 5),
         (2_000_001, 0.7, 6), (65_536 * 3 + 17, 0.4, 7)]


@pytest.mark.parametrize("d,frac,rank", CASES)
def test_nz_encode_equals_oracle(codec, oracle, d, frac, rank):
    g = _sparse(d, frac, rank, neg_zero=(rank % 2 == 0))
    nnz = int(np.count_nonzero(g))
    c = codec.compress(torch.from_numpy(g).cuda(), nnz, _cfg(BITMAP, V_NONE)).cpu().numpy().tobytes()
    assert c == oracle.encode_dense(g, nnz, GpConfig.make(BITMAP, V_NONE, seed=3))


@pytest.mark.parametrize("delta", [-1, +1, -777])
def test_speculation_miss_falls_back(codec, oracle, delta):
    g = _sparse(300_000, 0.4, 11)
    r = int(np.count_nonzero(g)) + delta  # r >= d/4 but not the nonzero count
    c = codec.compress(torch.from_numpy(g).cuda(), r, _cfg(BITMAP, V_NONE)).cpu().numpy().tobytes()
    assert c == oracle.encode_dense(g, r, GpConfig.make(BITMAP, V_NONE, seed=3))


def test_dense_input_half_selection(codec, oracle):
    g = synthetic_gradient(500_000, rank=12)  # no zeros: r = d/2 is a genuine top-r
    r = 250_000
    c = codec.compress(torch.from_numpy(g).cuda(), r, _cfg(BITMAP, V_NONE)).cpu().numpy().tobytes()
    assert c == oracle.encode_dense(g, r, GpConfig.make(BITMAP, V_NONE, seed=3))


def _want_dense(oracle, c, d, scale, base):
    _, sup, val = oracle.decode(c)
    want = base.copy()
    # scale is a power of two: the f32 product is exact and the sum rounds once, as fmaf does
    want[sup] = np.float32(scale) * val.astype(np.float32) + want[sup]
    return want


@pytest.mark.parametrize("vm", [V_NONE, V_F64])
@pytest.mark.parametrize("d,r", [(1, 1), (7, 3), (8192, 4000), (100_003, 1000), (1_000_000, 600_000)])
def test_fused_bitmap_decode(codec, oracle, vm, d, r):
    g = synthetic_gradient(d, rank=d % 7)
    c = oracle.encode_dense(g, r, GpConfig.make(BITMAP, vm, seed=1))
    dev = torch.from_numpy(np.frombuffer(c, np.uint8).copy()).cuda()
    base = synthetic_gradient(d, rank=99)
    for scale in (1.0, 0.25, -1.0):
        dense = torch.from_numpy(base.copy()).cuda()
        codec.decode_accumulate(dev, dense, scale=scale)
        codec.status()
        assert np.array_equal(dense.cpu().numpy().view(np.uint32),
                              _want_dense(oracle, c, d, scale, base).view(np.uint32))
        dense = torch.from_numpy(base.copy()).cuda()
        codec.decode_accumulate(dev, dense, scale=scale, overwrite=True)
        codec.status()
        assert np.array_equal(dense.cpu().numpy().view(np.uint32),
                              _want_dense(oracle, c, d, scale, np.zeros(d, np.float32)).view(np.uint32))


def test_fused_decode_errors_leave_dense_untouched(codec, oracle):
    from paper_2102_03112_b200 import CorruptPayloadError
    d, r = 100_000, 30_000
    g = synthetic_gradient(d, rank=4)
    c = bytearray(oracle.encode_dense(g, r, GpConfig.make(BITMAP, V_NONE, seed=1)))
    # clear one set bit of the bitmap and re-seal the CRC: popcount != r (pipeline.cpp:242-243)
    body = 49
    i = next(k for k in range(body, body + (d + 7) // 8) if c[k])
    c[i] &= c[i] - 1
    crc = oracle.crc32c(bytes(c[49:-4]))
    c[-4:] = crc.to_bytes(4, "little")
    with pytest.raises(OracleError, match="CorruptPayload"):
        oracle.decode(bytes(c))
    dense = torch.full((d,), 7.0, device="cuda")
    codec.decode_accumulate(torch.from_numpy(np.frombuffer(bytes(c), np.uint8).copy()).cuda(), dense)
    with pytest.raises(CorruptPayloadError):
        codec.status()
    assert bool((dense == 7.0).all())


def test_dense_length_mismatch_is_an_error(codec, oracle):
    from paper_2102_03112_b200 import Error
    d, r = 50_000, 20_000
    c = oracle.encode_dense(synthetic_gradient(d, rank=2), r, GpConfig.make(BITMAP, V_NONE, seed=1))
    dev = torch.from_numpy(np.frombuffer(c, np.uint8).copy()).cuda()
    for n in (d - 1, d + 1):
        dense = torch.zeros(n, device="cuda")
        codec.decode_accumulate(dev, dense)
        with pytest.raises(Error):
            codec.status()
        assert bool((dense == 0).all())
