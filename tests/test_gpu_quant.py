"""Quantizer (value id 3) and Store byte-codec slot (value id 4) on the device
vs the CPU oracle (itself pinned byte-for-byte to the reference build in
tests/test_oracle.py).  Bit-exact: container bytes, decoded supports and f64
values, and the error class of corrupted payloads."""
import numpy as np
import pytest
import torch

from oracle.bindings import GpConfig, OracleError, synthetic_gradient

pytestmark = pytest.mark.gpu

NONE, BITMAP, RLE, P0, P1, P2, PD, NAIVE = 0, 1, 2, 4, 5, 6, 7, 8
QUANT, SLOT = 3, 4
VCASES = [(QUANT, dict(quant_bits=7, quant_bucket=512)), (QUANT, dict(quant_bits=1, quant_bucket=1)),
          (QUANT, dict(quant_bits=16, quant_bucket=3)), (QUANT, dict(quant_bits=5, quant_bucket=100)),
          (QUANT, dict(quant_bits=12, quant_bucket=4096)), (SLOT, dict(slot_codec=0))]


@pytest.fixture(scope="module")
def codec():
    from paper_2102_03112_b200 import Codec
    c = Codec(max_d=1 << 21)
    yield c
    c.close()


def _dev(a):
    return torch.from_numpy(np.array(a, copy=True)).cuda()


def _grads():
    out = []
    for d, rank in [(1, 0), (7, 1), (4097, 2), (100_003, 3), (1_000_000, 4)]:
        g = synthetic_gradient(d, rank=rank)
        if d > 1000:
            g[: d // 4] = 0.0  # zero buckets: no RNG draws there
        out.append(g)
    return out


@pytest.mark.parametrize("im", [NONE, BITMAP, RLE, P0, P1, P2, PD, NAIVE])
@pytest.mark.parametrize("vm,kw", VCASES)
def test_encode_bytes_bit_exact(codec, oracle, im, vm, kw):
    from paper_2102_03112_b200 import PipelineConfig
    for g in _grads():
        for r in sorted({1, max(1, g.size // 100), max(1, g.size // 3)}):
            if im >= P0 and r == g.size:
                continue
            if im == P2 and r == 1 and g.size > 10_000:
                continue  # ~m/2 bits shared by |P| ~ d/128 positives: sets > 254 members (GP_CAPACITY)
            cfg = PipelineConfig(index_method=im, value_method=vm, fpr=0.01, seed=r + 3, **kw)
            got = codec.compress(_dev(g), r, cfg).cpu().numpy().tobytes()
            want = oracle.encode_dense(g, r, GpConfig.make(im, vm, fpr=0.01, seed=r + 3, **kw))
            assert got == want, (im, vm, kw, g.size, r)


@pytest.mark.parametrize("im", [BITMAP, P0, P2, NAIVE])
@pytest.mark.parametrize("vm,kw", VCASES)
def test_decode_bit_exact(codec, oracle, im, vm, kw):
    for g in _grads()[2:]:
        r = max(1, g.size // 100)
        c = oracle.encode_dense(g, r, GpConfig.make(im, vm, fpr=0.01, seed=5, **kw))
        d, sup, val = codec.decompress(_dev(np.frombuffer(c, np.uint8)))
        od, osup, oval = oracle.decode(c)
        assert d == od
        assert np.array_equal(sup.cpu().numpy().astype(np.uint32), osup)
        assert np.array_equal(val.cpu().numpy(), oval)


def _fix_crc(oracle, m: bytearray) -> bytes:
    m[-4:] = oracle.crc32c(bytes(m[49:-4])).to_bytes(4, "little")
    return bytes(m)


def test_decode_error_classes_match_oracle(codec, oracle):
    from paper_2102_03112_b200 import Error
    g = synthetic_gradient(5000, rank=2)
    for vm, kw in VCASES:
        c = bytearray(oracle.encode_dense(g, 50, GpConfig.make(BITMAP, vm, seed=2, **kw)))
        vo = 49 + int.from_bytes(c[25:33], "little")
        muts = [c[:vo] + bytes([0]) + c[vo + 1:], c[:vo] + bytes([17]) + c[vo + 1:], c[:vo] + bytes([9]) + c[vo + 1:],
                c[:vo] + bytes([2]) + c[vo + 1:], c[:vo + 1] + bytes(4) + c[vo + 5:]]
        for m in muts:
            bad = _fix_crc(oracle, bytearray(m))
            try:
                oracle.decode(bad)
                want = None
            except OracleError as e:
                want = e.kind
            dense = torch.zeros(5000, dtype=torch.float32, device="cuda")
            got = None
            try:
                codec.decode_accumulate(_dev(np.frombuffer(bad, np.uint8)), dense, length=len(bad))
                codec.status()
            except Error as e:
                got = type(e).__name__
            if want == "Unsupported" or got == "UnsupportedMethodError":
                continue  # deflate-framed slot: unsupported on the device path (byte id 1)
            assert got == want, (vm, kw, got, want)
            if want is not None:
                assert float(dense.abs().sum()) == 0.0
