"""CPU check of the Deflate-slot test vectors used by tests/test_gpu_deflate.py:
the reference build (oracle/_ref, gradpack over the image's zlib) accepts every
well-formed stream with the same values as the Store-codec container, ignores
bytes after the Adler-32 trailer, and rejects each hand-built malformed stream
with CorruptPayloadError — so the GPU test compares the device against a
checker whose verdicts are pinned here."""
import numpy as np

from oracle.bindings import GpConfig, synthetic_gradient
from test_gpu_deflate import BITMAP, SLOT, _error_cases, _raw_of, _ref_decode, _streams, _with_body


def test_streams_decode_like_store(reference):
    g = synthetic_gradient(3000, rank=1)
    g[:1500] = np.round(g[:1500] * 8) / 8
    base = reference.encode_dense(g, 300, GpConfig.make(BITMAP, SLOT, seed=1, slot_codec=0))
    d0, s0, v0 = reference.decode(base)
    raw = _raw_of(base)
    for name, body in _streams(raw):
        for tail in (b"", b"\x00trailing"):
            got = _ref_decode(reference, _with_body(reference, base, body + tail, len(raw)))
            assert not isinstance(got, str), (name, got)
            assert got[0] == d0 and np.array_equal(got[1], s0) and np.array_equal(got[2], v0), name


def test_store_and_codec_ids(reference):
    g = synthetic_gradient(500, rank=2)
    base = reference.encode_dense(g, 20, GpConfig.make(BITMAP, SLOT, seed=1, slot_codec=0))
    raw = _raw_of(base)
    assert not isinstance(_ref_decode(reference, _with_body(reference, base, raw, len(raw), codec_id=0)), str)
    assert _ref_decode(reference, _with_body(reference, base, raw, len(raw), codec_id=2)) == "UnknownMethodError"
    assert _ref_decode(reference, _with_body(reference, base, b"", 0, codec_id=1)) == "CorruptPayloadError"


def test_malformed_streams_rejected(reference):
    g = synthetic_gradient(2000, rank=4)
    base = reference.encode_dense(g, 64, GpConfig.make(BITMAP, SLOT, seed=1, slot_codec=0))
    raw = _raw_of(base)
    for name, body in _error_cases(raw).items():
        assert _ref_decode(reference, _with_body(reference, base, body, len(raw))) == "CorruptPayloadError", name
