"""RLE index codec (id 2) on the B200 vs the CPU oracle: bytes, decode, and the
reference's error classes for malformed run streams (codecs.cpp:52-70)."""
import struct

import numpy as np
import pytest
import torch

from oracle.bindings import GpConfig, OracleError, synthetic_gradient

pytestmark = pytest.mark.gpu

RLE = 2
V_NONE, V_FIT, V_F64 = 0, 1, 5


@pytest.fixture(scope="module")
def codec():
    from paper_2102_03112_b200 import Codec
    c = Codec(max_d=1 << 22)
    yield c
    c.close()


def _dev(b):
    return torch.from_numpy(np.frombuffer(b, np.uint8).copy()).cuda()


def _grads():
    rng = np.random.default_rng(3)
    out = []
    for d in [1, 2, 9, 130, 1000, 70_000, 269_722]:
        out.append(synthetic_gradient(d, rank=d % 3))
    rows = synthetic_gradient(500_000, rank=2)
    mask = np.repeat(rng.random(500_000 // 64 + 1) < 0.4, 64)[:500_000]
    rows[mask] = 0.0  # 64-wide zero rows: long runs (multi-group varints)
    out.append(rows)
    return out


def _rs(g):
    d = g.size
    nz = int(np.count_nonzero(g))
    return sorted({1, max(1, d // 100), max(1, d // 2), d, max(1, nz)})


@pytest.mark.parametrize("vm", [V_NONE, V_F64, V_FIT])
def test_rle_encode_bytes(codec, oracle, vm):
    from paper_2102_03112_b200 import PipelineConfig
    for g in _grads():
        for r in _rs(g):
            got = codec.compress(torch.from_numpy(g).cuda(), r, PipelineConfig(index_method=RLE, value_method=vm,
                                                                             degree=2)).cpu().numpy().tobytes()
            want = oracle.encode_dense(g, r, GpConfig.make(RLE, vm, degree=2))
            if vm == V_FIT:  # fit coefficients are tolerance-checked in test_gpu_fit; compare the index payload
                il = struct.unpack_from("<Q", want, 25)[0]
                assert got[:49 + il] == want[:49 + il], (g.size, r)
            else:
                assert got == want, (g.size, r)


@pytest.mark.parametrize("vm", [V_NONE, V_FIT])
def test_rle_decode(codec, oracle, vm):
    for g in _grads():
        for r in _rs(g):
            c = oracle.encode_dense(g, r, GpConfig.make(RLE, vm, degree=2))
            d, sup, val = codec.decompress(_dev(c))
            od, osup, oval = oracle.decode(c)
            assert d == od and np.array_equal(sup.cpu().numpy().astype(np.uint32), osup)
            assert np.array_equal(val.cpu().numpy(), oval)


def _reseal(c: bytes, index_payload: bytes) -> bytes:
    il_old, vl, rl = struct.unpack_from("<QQQ", c, 25)
    body = index_payload + c[49 + il_old:49 + il_old + vl + rl]
    hdr = bytearray(c[:49])
    struct.pack_into("<Q", hdr, 25, len(index_payload))
    from oracle.bindings import oracle as _o
    return bytes(hdr) + body + struct.pack("<I", _o().crc32c(body))


def test_rle_malformed_streams(codec, oracle):
    from paper_2102_03112_b200 import Error
    g = synthetic_gradient(3000, rank=1)
    c = oracle.encode_dense(g, 40, GpConfig.make(RLE, V_NONE))
    il = struct.unpack_from("<Q", c, 25)[0]
    p = c[49:49 + il]
    bad_payloads = [
        p[:-1],                      # truncated
        p + b"\x00",                 # >= 8 slack bits
        p[:-1] + b"\x02",            # nonzero slack
        bytes([p[0] & 1]) + b"\x00\x00",   # zero-length run
        bytes([1 | (0x7F << 1) & 0xFF, 0xFF] + [0xFF] * 11 + [0]),  # varint over 10 groups
        bytes([0x01, 0x10]),         # polarity + one run too short, stream ends
        b"",                         # no polarity bit
        bytes([0xFF, 0xFF, 0xFF, 0xFF, 0x0F, 0x00]),  # run longer than d
    ]
    seen = set()
    for bp in bad_payloads:
        bad = _reseal(c, bp)
        with pytest.raises(OracleError) as oe:
            oracle.decode(bad)
        dense = torch.zeros(3000, dtype=torch.float32, device="cuda")
        with pytest.raises(Error) as ge:
            codec.decode_accumulate(_dev(bad), dense)
            codec.status()
        assert type(ge.value).__name__ == oe.value.kind, (bp, ge.value, oe.value)
        assert float(dense.abs().sum()) == 0.0
        seen.add(oe.value.kind)
    assert {"TruncatedError", "CorruptPayloadError"} <= seen
