"""CUDA path vs the CPU oracle, through the C-ABI (pytest -m gpu on a B200).

Bit-exact: supports, container bytes, CRCs, decoded supports and raw values.
Tolerance (stated per test): the f32 dense accumulate against the oracle's
f64 to_dense.
"""
import numpy as np
import pytest
import torch

from oracle.bindings import GpConfig, OracleError, synthetic_gradient

pytestmark = pytest.mark.gpu

NONE, BITMAP, RLE, P0, P1, P2, PD, NAIVE = 0, 1, 2, 4, 5, 6, 7, 8
V_NONE, V_FIT, V_F64 = 0, 1, 5

EXC_NAME = {"Error": "Error", "DecodeError": "DecodeError", "TruncatedError": "TruncatedError",
            "ChecksumError": "ChecksumError", "UnknownMethodError": "UnknownMethodError",
            "CorruptPayloadError": "CorruptPayloadError"}


@pytest.fixture(scope="module")
def codec():
    from paper_2102_03112_b200 import Codec
    c = Codec(max_d=1 << 22)
    yield c
    c.close()


def _dev(a):
    return torch.from_numpy(np.array(a, copy=True)).cuda()


def _cfg(im, vm, **kw):
    from paper_2102_03112_b200 import PipelineConfig
    return PipelineConfig(index_method=im, value_method=vm, **kw)


def _grads():
    rng = np.random.default_rng(0)
    out = []
    for d in [1, 2, 3, 7, 64, 1000, 4097, 65536 + 3, 269722, 1_000_000]:
        g = synthetic_gradient(d, rank=d % 5)
        out.append(g)
    ties = np.round(synthetic_gradient(100_003, rank=9) * 4).astype(np.float32)  # heavy magnitude ties
    out.append(ties)
    z = synthetic_gradient(300_000, rank=1)
    z[rng.random(z.size) < 0.4] = 0.0  # natural sparsity, zeros tie at key 0
    out.append(z)
    const = np.full(50_000, -1.5, np.float32)  # every key equal
    out.append(const)
    return out


def _rs(d):
    return sorted({1, max(1, d // 100), max(1, d // 3), d})


def test_top_r_bit_exact(codec, oracle):
    for g in _grads():
        for r in _rs(g.size):
            sup, val = codec.top_r(_dev(g), r)
            want = oracle.top_r(g, r)
            assert np.array_equal(sup.cpu().numpy().astype(np.uint32), want), (g.size, r)
            assert np.array_equal(val.cpu().numpy().view(np.uint32), g[want].view(np.uint32))


def test_top_r_dense_selections(codec, oracle):
    """r > d/16 takes the counted candidates path (topr.cu): natural sparsity
    with r = nnz and its neighbours, 64-wide zero rows (C3's shape), half-dense
    ties, and an input pointer that is not 16-byte aligned."""
    rng = np.random.default_rng(5)
    for d in [4096 * 3 + 17, 100_000, 1_000_003]:
        g = synthetic_gradient(d, rank=2)
        rows = rng.random((d + 63) // 64) < 0.4
        g[np.repeat(rows, 64)[:d]] = 0.0
        nnz = int(np.count_nonzero(g))
        ties = np.round(g * 2).astype(np.float32)
        for x in (g, ties):
            for r in sorted({nnz - 1, nnz, min(d, nnz + 1), d // 16 + 1, d // 2}):
                sup, val = codec.top_r(_dev(x), r)
                want = oracle.top_r(x, r)
                assert np.array_equal(sup.cpu().numpy().astype(np.uint32), want), (d, r)
        buf = _dev(np.concatenate([np.zeros(1, np.float32), g]))
        sup, _ = codec.top_r(buf[1:], nnz)
        assert np.array_equal(sup.cpu().numpy().astype(np.uint32), oracle.top_r(g, nnz)), d


def test_crc32c_bit_exact(codec, oracle):
    rng = np.random.default_rng(1)
    for n in [0, 1, 9, 1023, 1024, 1025, 262143, 262144, 262145, 3_000_001]:
        data = rng.integers(0, 256, n, dtype=np.uint8) if n else np.zeros(1, np.uint8)
        t = _dev(data)
        got = codec.crc32c(t[:n])
        assert got == oracle.crc32c(data[:n].tobytes()), n
    assert codec.crc32c(_dev(np.frombuffer(b"123456789", np.uint8))) == 0xE3069283
    # misaligned starts and ends, ranges inside one 64-byte line, and ranges
    # past one row of the fixed grid (148 x 1024 lanes x 64 B) — several rows
    big = rng.integers(0, 256, 25_000_000 + 200, dtype=np.uint8)
    t = _dev(big)
    for off, n in [(1, 5), (3, 60), (63, 2), (17, 64), (5, 127), (13, 9_699_329), (0, 9_699_328), (7, 25_000_000),
                   (64, 19_398_656 + 3), (33, 1_260_001),
                   # crc_tail (ranges up to 8 MiB): the init-term bytes across words and chunks,
                   # one grid row exactly, one chunk past it, several Horner rows
                   (2, 4), (1, 3), (61, 4), (62, 67), (60, 130), (9, 148 * 256 * 64), (11, 148 * 256 * 64 + 1),
                   (6, 7_999_999), (4, 8 << 20)]:
        assert codec.crc32c(t[off:off + n]) == oracle.crc32c(big[off:off + n].tobytes()), (off, n)


@pytest.mark.parametrize("im,vm", [(NONE, V_NONE), (BITMAP, V_NONE), (BITMAP, V_F64), (NONE, V_F64)])
def test_encode_bytes_bit_exact(codec, oracle, im, vm):
    for g in _grads():
        for r in _rs(g.size):
            cfg = _cfg(im, vm, seed=r)
            got = codec.compress(_dev(g), r, cfg).cpu().numpy().tobytes()
            want = oracle.encode_dense(g, r, GpConfig.make(im, vm, seed=r))
            assert got == want, (im, vm, g.size, r)


@pytest.mark.parametrize("im,vm", [(NONE, V_NONE), (BITMAP, V_NONE), (BITMAP, V_F64), (NONE, V_F64)])
def test_decode_bit_exact(codec, oracle, im, vm):
    for g in _grads():
        for r in _rs(g.size):
            c = oracle.encode_dense(g, r, GpConfig.make(im, vm))
            d, sup, val = codec.decompress(_dev(np.frombuffer(c, np.uint8)))
            od, osup, oval = oracle.decode(c)
            assert d == od
            assert np.array_equal(sup.cpu().numpy().astype(np.uint32), osup)
            assert np.array_equal(val.cpu().numpy(), oval)


def test_decode_accumulate_mean(codec, oracle):
    # f32 accumulate of N peers in rank order vs the oracle's f64 sum; tolerance:
    # |err| <= 4 ulp(f32) of the magnitude of the largest term at each coordinate.
    d, r, n = 200_000, 2_000, 4
    dense = torch.zeros(d, dtype=torch.float32, device="cuda")
    ref = np.zeros(d, np.float64)
    for w in range(n):
        g = synthetic_gradient(d, rank=w)
        c = oracle.encode_dense(g, r, GpConfig.make(BITMAP, V_NONE))
        codec.decode_accumulate(_dev(np.frombuffer(c, np.uint8)), dense, scale=1.0 / n)
        oracle.decode_accumulate(c, ref, 1.0 / n)
    codec.status()
    got = dense.cpu().numpy().astype(np.float64)
    assert np.allclose(got, ref, rtol=0, atol=4 * np.finfo(np.float32).eps * np.abs(ref).max())


def _mutations(c: bytes):
    out = [c[:3], b"XRC1" + c[4:], c[:4] + b"\x02\x00" + c[6:], c[:-1], c + b"\x00",
           c[:49] + bytes([c[49] ^ 1]) + c[50:], c[:6] + b"\x09" + c[7:], c[:8] + b"\x02" + c[9:],
           c[:40]]
    return out


def test_decode_error_classes_match_oracle(codec, oracle):
    from paper_2102_03112_b200 import Error
    g = synthetic_gradient(5000, rank=2)
    for im, vm in [(NONE, V_NONE), (BITMAP, V_NONE), (BITMAP, V_F64)]:
        c = oracle.encode_dense(g, 50, GpConfig.make(im, vm))
        for bad in _mutations(c):
            with pytest.raises(OracleError) as oe:
                oracle.decode(bad)
            dense = torch.zeros(5000, dtype=torch.float32, device="cuda")
            t = _dev(np.frombuffer(bad, np.uint8)) if len(bad) else torch.zeros(1, dtype=torch.uint8, device="cuda")
            with pytest.raises(Error) as ge:
                codec.decode_accumulate(t, dense, length=len(bad))
                codec.status()
            assert type(ge.value).__name__ == oe.value.kind, (im, vm, len(bad), ge.value, oe.value)
            assert float(dense.abs().sum()) == 0.0  # a failed decode never touches the output


BLOOM_CASES = [(P0, V_NONE), (P1, V_NONE), (P2, V_NONE), (PD, V_NONE), (NAIVE, V_NONE), (P2, V_F64)]


@pytest.mark.parametrize("im,vm", BLOOM_CASES)
@pytest.mark.parametrize("fpr", [0.1, 0.01, 0.001])
def test_bloom_encode_bytes_bit_exact(codec, oracle, im, vm, fpr):
    for d, r in [(1000, 10), (65536 + 3, 655), (269722, 2697), (1_000_000, 10_000)]:
        g = synthetic_gradient(d, rank=d % 7)
        for seed in (1, 12345):
            cfg = _cfg(im, vm, fpr=fpr, seed=seed, pd_variant=seed % 3)
            got = codec.compress(_dev(g), r, cfg).cpu().numpy().tobytes()
            want = oracle.encode_dense(g, r, GpConfig.make(im, vm, fpr=fpr, seed=seed, pd_variant=seed % 3))
            assert len(got) == len(want), (im, vm, fpr, d, r, seed)
            assert got == want, (im, vm, fpr, d, r, seed)


@pytest.mark.parametrize("im,vm", BLOOM_CASES)
def test_bloom_decode_bit_exact(codec, oracle, im, vm):
    for d, r, fpr in [(5000, 50, 0.3), (269722, 2697, 0.01), (1_000_000, 10_000, 0.001)]:
        g = synthetic_gradient(d, rank=3)
        c = oracle.encode_dense(g, r, GpConfig.make(im, vm, fpr=fpr, seed=d, pd_variant=2))
        gd, sup, val = codec.decompress(_dev(np.frombuffer(c, np.uint8)))
        od, osup, oval = oracle.decode(c)
        assert gd == od and np.array_equal(sup.cpu().numpy().astype(np.uint32), osup)
        assert np.array_equal(val.cpu().numpy(), oval)


@pytest.mark.parametrize("d,r,eps", [(50_000, 500, 0.01), (300_000, 3_000, 0.001), (1_000_000, 10_000, 0.05)])
def test_bloom_components_bit_exact(codec, oracle, d, r, eps):
    """gp_bloom_positive_scan / gp_bloom_select on a bare serialized filter."""
    g = synthetic_gradient(d, rank=3)
    sup = oracle.top_r(g, r)
    filt = oracle.bloom_build(sup, eps, 0x1234, 0x5678)
    f = _dev(np.frombuffer(filt, np.uint8))
    pos = codec.bloom_positive_scan(f, d).cpu().numpy().astype(np.uint32)
    assert np.array_equal(pos, oracle.positive_scan(filt, d))
    for im in (P1, P2):
        got = codec.bloom_select(f, d, r, im).cpu().numpy().astype(np.uint32)
        assert np.array_equal(got, oracle.bloom_select(filt, d, r, im)), im


def test_bloom_components_errors(codec, oracle):
    from paper_2102_03112_b200 import CorruptPayloadError, Error
    d, r = 20_000, 200
    sup = oracle.top_r(synthetic_gradient(d, rank=1), r)
    filt = bytearray(oracle.bloom_build(sup, 0.01, 1, 2))
    f = _dev(np.frombuffer(bytes(filt), np.uint8))
    with pytest.raises(Error):  # |P| < r for the selection
        codec.bloom_select(f, d, d, P2)
    bad = bytearray(filt)
    bad[8] = bad[9] = 0  # k = 0
    with pytest.raises(CorruptPayloadError):
        codec.bloom_positive_scan(_dev(np.frombuffer(bytes(bad), np.uint8)), d)
