"""Deflate byte-codec slot (value id 4, byte codec 1) decoded on the device
(csrc/inflate.cu) against the reference build itself (oracle/_ref: gradpack's
byte_decompress over the image's zlib, codecs.cpp:268-290).  Bit-exact
supports and f64 values; for streams that zlib rejects, the same error class
(CorruptPayloadError).  Streams come from the reference's own encoder
(compress2 at Z_DEFAULT_COMPRESSION) and from Python's zlib at every level and
strategy (stored, fixed-Huffman, dynamic, RLE, Huffman-only blocks, small
windows), plus hand-built and mutated streams for the error paths."""
import random
import zlib

import numpy as np
import pytest
import torch

from oracle.bindings import GpConfig, OracleError, synthetic_gradient

pytestmark = pytest.mark.gpu

BITMAP, RLE, P0, P2, NAIVE = 1, 2, 4, 6, 8
SLOT = 4


@pytest.fixture(scope="module")
def codec():
    from paper_2102_03112_b200 import Codec
    c = Codec(max_d=1 << 20)
    yield c
    c.close()


def _dev(b: bytes):
    return torch.from_numpy(np.frombuffer(bytes(b), np.uint8).copy()).cuda()


def _device_decode(codec, c: bytes):
    """(d, support, values) or the exception class name."""
    from paper_2102_03112_b200 import Error
    try:
        d, sup, val = codec.decompress(_dev(c))
        return d, sup.cpu().numpy().astype(np.uint32), val.cpu().numpy()
    except Error as e:
        return type(e).__name__


def _ref_decode(ref, c: bytes):
    try:
        return ref.decode(c)
    except OracleError as e:
        return e.kind


def _same(got, want):
    if isinstance(want, str) or isinstance(got, str):
        return got == want
    return got[0] == want[0] and np.array_equal(got[1], want[1]) and np.array_equal(got[2], want[2])


def _with_body(ref, c: bytes, body: bytes, raw_len: int, codec_id: int = 1) -> bytes:
    """Container c with its value payload replaced by [codec_id][raw_len][body], CRC fixed."""
    il = int.from_bytes(c[25:33], "little")
    vl = int.from_bytes(c[33:41], "little")
    rl = int.from_bytes(c[41:49], "little")
    payload = bytes([codec_id]) + raw_len.to_bytes(8, "little") + body
    m = bytearray(c[:33]) + len(payload).to_bytes(8, "little") + c[41:49] + c[49:49 + il] + payload
    m += c[49 + il + vl:49 + il + vl + rl]
    m += ref.crc32c(bytes(m[49:])).to_bytes(4, "little")
    return bytes(m)


def _raw_of(c: bytes) -> bytes:
    il = int.from_bytes(c[25:33], "little")
    vl = int.from_bytes(c[33:41], "little")
    return c[49 + il + 9:49 + il + vl]  # Store slot body = the raw f32 bytes


@pytest.mark.parametrize("im", [BITMAP, RLE, P0, P2, NAIVE])
def test_reference_deflate_containers(codec, reference, im):
    """Containers the reference's encoder writes (zlib compress2, level 6)."""
    for d, r in [(1, 1), (100, 7), (5000, 50), (100_003, 1000), (400_000, 40_000)]:
        g = synthetic_gradient(d, rank=3)
        if d > 1000:
            g[: d // 3] = np.round(g[: d // 3] * 4) / 4  # repetitive bytes: real matches, not just literals
        c = reference.encode_dense(g, r, GpConfig.make(im, SLOT, fpr=0.01, seed=9, slot_codec=1))
        want = _ref_decode(reference, c)
        assert not isinstance(want, str)
        assert _same(_device_decode(codec, c), want), (im, d, r)


def _streams(raw: bytes):
    yield "level0", zlib.compress(raw, 0)
    for lvl in (1, 3, 6, 9):
        yield f"level{lvl}", zlib.compress(raw, lvl)
    for name, strat in [("fixed", zlib.Z_FIXED), ("huffman_only", zlib.Z_HUFFMAN_ONLY), ("rle", zlib.Z_RLE),
                        ("filtered", zlib.Z_FILTERED)]:
        o = zlib.compressobj(6, zlib.DEFLATED, 15, 8, strat)
        yield name, o.compress(raw) + o.flush()
    for wbits in (9, 10, 12):
        o = zlib.compressobj(9, zlib.DEFLATED, wbits)
        yield f"wbits{wbits}", o.compress(raw) + o.flush()
    o = zlib.compressobj(6)  # several blocks: full flushes put stored/empty blocks between them
    parts = [o.compress(raw[k:k + 4000]) + o.flush(zlib.Z_FULL_FLUSH) for k in range(0, len(raw), 4000)]
    yield "flushes", b"".join(parts) + o.flush()


def test_python_zlib_streams(codec, reference):
    """Every block type and code shape Python's zlib emits, same bytes as the reference decodes."""
    for d, r, seed in [(3000, 300, 1), (60_000, 20_000, 2)]:
        g = synthetic_gradient(d, rank=seed)
        g[: d // 2] = np.round(g[: d // 2] * 8) / 8
        base = reference.encode_dense(g, r, GpConfig.make(BITMAP, SLOT, seed=1, slot_codec=0))
        raw = _raw_of(base)
        assert len(raw) == 4 * r
        for name, body in _streams(raw):
            c = _with_body(reference, base, body, len(raw))
            want = _ref_decode(reference, c)
            assert not isinstance(want, str), name
            assert _same(_device_decode(codec, c), want), (name, d)
            # bytes after the Adler-32 trailer are ignored by uncompress
            c2 = _with_body(reference, base, body + b"\x00garbage", len(raw))
            assert _same(_device_decode(codec, c2), _ref_decode(reference, c2)), name


def test_raw_length_mismatches(codec, reference):
    """Streams that inflate to fewer / more bytes than raw_len, and raw_len != 4·count."""
    g = synthetic_gradient(10, rank=1)
    base = reference.encode_dense(g, 1, GpConfig.make(BITMAP, SLOT, seed=1, slot_codec=0))
    for body, raw_len in [(zlib.compress(b""), 4), (zlib.compress(_raw_of(base)), 4),
                          (zlib.compress(_raw_of(base) * 2), 4), (zlib.compress(_raw_of(base)[:3]), 4),
                          (zlib.compress(_raw_of(base)), 8)]:
        c = _with_body(reference, base, body, raw_len)
        assert _same(_device_decode(codec, c), _ref_decode(reference, c))


def _error_cases(raw: bytes) -> dict:
    """One malformed stream per zlib rejection rule the device mirrors."""
    good = zlib.compress(raw, 6)
    fixed = zlib.compressobj(6, zlib.DEFLATED, 15, 8, zlib.Z_FIXED)
    fixed = fixed.compress(raw) + fixed.flush()
    return {
        "truncated_header": good[:1],
        "bad_fcheck": bytes([good[0], good[1] ^ 1]) + good[2:],
        "cm7": bytes([0x77, (31 - (0x7700 % 31)) % 31]) + good[2:],
        "cinfo8": bytes([0x88, (31 - (0x8800 % 31)) % 31]) + good[2:],
        "fdict": bytes([0x78, 0xBB]) + b"\x00\x00\x00\x01" + good[2:],
        "btype3": good[:2] + bytes([0x07]) + good[3:],
        "stored_nlen": good[:2] + bytes([0x01, 0x05, 0x00, 0x00, 0x00]) + b"x" * 5,
        "no_trailer": good[:-4],
        "bad_adler": good[:-1] + bytes([good[-1] ^ 0x5A]),
        "truncated_body": good[: len(good) // 2],
        "short_output": zlib.compress(raw[:-4]),
        "long_output": zlib.compress(raw + b"\x00" * 4),
        "far_distance": bytes([0x78, 0x01]) + _fixed_block_far(),
        "fixed_truncated": fixed[:-6],
        "empty": b"",
    }


def test_error_paths(codec, reference):
    """Hand-built malformed streams: each rejected by zlib and by the device with the same class."""
    g = synthetic_gradient(2000, rank=4)
    base = reference.encode_dense(g, 64, GpConfig.make(BITMAP, SLOT, seed=1, slot_codec=0))
    raw = _raw_of(base)
    for name, body in _error_cases(raw).items():
        c = _with_body(reference, base, body, len(raw))
        want = _ref_decode(reference, c)
        assert want == "CorruptPayloadError", (name, want)
        assert _device_decode(codec, c) == want, name


def _fixed_block_far() -> bytes:
    """A final fixed-Huffman block whose first symbol is a match (distance 1 with no output yet)."""
    bits = []

    def put(v, n):  # LSB-first fields
        bits.extend((v >> k) & 1 for k in range(n))

    def put_code(code, n):  # Huffman codes MSB-first
        bits.extend((code >> (n - 1 - k)) & 1 for k in range(n))

    put(1, 1)
    put(1, 2)
    put_code(0b0000001, 7)  # length symbol 257 (length 3)
    put_code(0, 5)          # distance symbol 0 (distance 1)
    put_code(0, 7)          # end of block
    out = bytearray()
    for k in range(0, len(bits), 8):
        out.append(sum(b << j for j, b in enumerate(bits[k:k + 8])))
    return bytes(out) + b"\x00\x00\x00\x00"


def test_mutated_streams_match_reference(codec, reference):
    """Random byte mutations of valid streams (CRC re-fixed): accept/reject and values agree with zlib."""
    rng = random.Random(7)
    g = synthetic_gradient(3000, rank=5)
    g[:1500] = np.round(g[:1500] * 4) / 4
    base = reference.encode_dense(g, 400, GpConfig.make(BITMAP, SLOT, seed=1, slot_codec=0))
    raw = _raw_of(base)
    streams = [body for _, body in _streams(raw)]
    n_ok = n_bad = 0
    for it in range(400):
        body = bytearray(rng.choice(streams))
        for _ in range(rng.choice([1, 1, 2, 3])):
            k = rng.randrange(len(body))
            if rng.random() < 0.5:
                body[k] ^= 1 << rng.randrange(8)
            else:
                body[k] = rng.randrange(256)
        if rng.random() < 0.3:  # make the Adler check pass so the decoder's own checks decide
            inner = bytes(body[:-4])
            try:
                out = zlib.decompressobj().decompress(inner)
                body = bytearray(inner + zlib.adler32(out).to_bytes(4, "big"))
            except zlib.error:
                pass
        c = _with_body(reference, base, bytes(body), len(raw))
        want = _ref_decode(reference, c)
        got = _device_decode(codec, c)
        assert _same(got, want), (it, got if isinstance(got, str) else "values", want if isinstance(want, str) else "values")
        n_ok += not isinstance(want, str)
        n_bad += isinstance(want, str)
    assert n_bad > 50


def test_decode_accumulate(codec, reference):
    g = synthetic_gradient(50_000, rank=6)
    c = reference.encode_dense(g, 5000, GpConfig.make(P2, SLOT, fpr=0.01, seed=4, slot_codec=1))
    want = np.zeros(50_000, np.float64)
    reference.decode_accumulate(c, want, 0.5)
    dense = torch.zeros(50_000, dtype=torch.float32, device="cuda")
    codec.decode_accumulate(_dev(c), dense, scale=0.5)
    codec.status()
    assert np.array_equal(dense.cpu().numpy(), want.astype(np.float32))
