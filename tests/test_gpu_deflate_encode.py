"""Deflate byte-codec slot ENCODED on the device (csrc/deflate.cu; byte_compress,
codecs.cpp:244-266).  The stream is a valid zlib stream of the 4n f32 value
bytes — Python's zlib (the decoder the reference's uncompress is) inflates it
to exactly those bytes, the reference build decodes the container to the same
support and values, and so does the device's own inflate — while its bytes
differ from zlib's compress2 (a different, chunk-parallel encoder; DESIGN.md
§3).  Everything outside the slot body (header ids, index payload, framing) is
the reference's."""
import struct
import zlib

import numpy as np
import pytest
import torch

from golden_util import split
from oracle.bindings import GpConfig, synthetic_gradient

pytestmark = pytest.mark.gpu

NONE, BITMAP, RLE, P0, P2 = 0, 1, 2, 4, 6
SLOT = 4


@pytest.fixture(scope="module")
def codec():
    from paper_2102_03112_b200 import Codec
    c = Codec(max_d=1 << 21)
    yield c
    c.close()


def _check(codec, reference, c: bytes, want_ref: bytes, values_f32: np.ndarray):
    p, q = split(c), split(want_ref)
    assert p["header"][:25] == q["header"][:25] and p["index"] == q["index"] and p["reorder"] == q["reorder"]
    body = p["value"]
    assert body[0] == 1 and struct.unpack_from("<Q", body, 1)[0] == 4 * values_f32.size
    raw = zlib.decompress(body[9:])
    assert raw == values_f32.astype("<f4").tobytes(), "the zlib stream does not inflate to the value bytes"
    # decoders: the reference build (zlib uncompress) and the device inflate
    d1, s1, v1 = reference.decode(c)
    d2, s2, v2 = reference.decode(want_ref)
    assert d1 == d2 and np.array_equal(s1, s2) and np.array_equal(v1, v2)
    dd, sd, vd = codec.decompress(torch.from_numpy(np.frombuffer(c, np.uint8).copy()).cuda())
    assert dd == d1 and np.array_equal(sd.cpu().numpy().astype(np.uint32), s1)
    assert np.array_equal(vd.cpu().numpy(), v1)
    return len(body) - 9


@pytest.mark.parametrize("im", [BITMAP, RLE, P0, P2])
@pytest.mark.parametrize("d,r", [(1_000, 1), (20_000, 200), (300_000, 8_192), (1_000_000, 100_003)])
def test_deflate_encode_round_trips(codec, reference, im, d, r):
    from paper_2102_03112_b200 import PipelineConfig
    g = synthetic_gradient(d, rank=d % 7)
    cfg = PipelineConfig(index_method=im, value_method=SLOT, fpr=0.01, seed=11, slot_codec=1)
    c = codec.compress(torch.from_numpy(g).cuda(), r, cfg).cpu().numpy().tobytes()
    want = reference.encode_dense(g, r, GpConfig.make(im, SLOT, fpr=0.01, seed=11, slot_codec=1))
    _, sup, val = reference.decode(want)
    n = _check(codec, reference, c, want, val.astype(np.float32))
    zl = len(split(want)["value"]) - 9
    assert n <= 4 * val.size + 5 * (4 * val.size // 32768 + 1) + 6  # never more than stored blocks
    if val.size >= 50_000:  # literal-only Huffman vs zlib level 6 on gradient floats
        assert n <= 1.08 * zl, (n, zl)


@pytest.mark.parametrize("kind", ["zeros", "constant", "two", "ramp"])
def test_deflate_encode_degenerate_byte_distributions(codec, reference, kind):
    """single-symbol and few-symbol chunks (package-merge's partner code, stored fallbacks)"""
    from paper_2102_03112_b200 import PipelineConfig
    d = 200_000
    sup = np.arange(0, d, 2, dtype=np.uint32)
    n = sup.size
    vals = {"zeros": np.zeros(n), "constant": np.full(n, 1.5), "two": np.where(np.arange(n) % 3, 1.0, -2.0),
            "ramp": np.arange(n, dtype=np.float64)}[kind]
    cfg = PipelineConfig(index_method=BITMAP, value_method=SLOT, seed=2, slot_codec=1)
    c = codec.compress_sparse(d, torch.from_numpy(sup.astype(np.int32)).cuda(), torch.from_numpy(vals).cuda(), cfg)
    c = c.cpu().numpy().tobytes()
    want = reference.encode_sparse64(d, sup, vals, GpConfig.make(BITMAP, SLOT, seed=2, slot_codec=1))
    _check(codec, reference, c, want, vals.astype(np.float32))


def test_deflate_encode_empty_sequence(codec, reference):
    from paper_2102_03112_b200 import PipelineConfig
    cfg = PipelineConfig(index_method=NONE, value_method=SLOT, slot_codec=1)
    e_i = torch.zeros(0, dtype=torch.int32, device="cuda")
    e_v = torch.zeros(0, dtype=torch.float64, device="cuda")
    c = codec.compress_sparse(10, e_i, e_v, cfg).cpu().numpy().tobytes()
    want = reference.encode_sparse64(10, np.zeros(0, np.uint32), np.zeros(0), GpConfig.make(NONE, SLOT, slot_codec=1))
    _check(codec, reference, c, want, np.zeros(0, np.float32))
