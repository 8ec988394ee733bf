"""Pins the CPU oracle (oracle/gp_oracle.c) before anything is checked against it.

Two independent anchors:
  1. the reference's own known-answer vectors, transcribed
     with their file:line;
  2. the unmodified reference sources built in oracle/_ref (skipped when that
     build is absent, e.g. on the GPU box where /root/reference does not exist).
"""
import struct

import numpy as np
import pytest

from oracle.bindings import GpConfig, OracleError, synthetic_gradient

NONE, BITMAP, RLE, P0, P1, P2, PD, NAIVE = 0, 1, 2, 4, 5, 6, 7, 8
V_NONE, V_FIT, V_F64 = 0, 1, 5


# ---------------------------------------------------------------- known answers
def test_crc32c_check_value(oracle):
    # FORMAT.md:42, test_container.cpp:148-152
    assert oracle.crc32c(b"123456789") == 0xE3069283
    assert oracle.crc32c(b"") == 0


@pytest.mark.parametrize("eps,r,m,k", [
    (0.5, 1, 2, 1), (1e-3, 1000, 14378, 10), (1e-2, 100, 959, 7), (1e-9, 100, 4314, 30),
    (1e-4, 100, 1918, 14), (1e-4, 10000, 191702, 14), (1e-3, 100, 1438, 10),
    (1e-2, 10000, 95851, 7)])
def test_bloom_params_table(oracle, eps, r, m, k):
    # test_bloom.cpp:24-42 (frozen against a 60-digit evaluation)
    assert oracle.bloom_params(eps, r) == (m, k)


def test_bloom_params_rejects(oracle):
    for eps, r in [(0.0, 10), (1.0, 10), (0.5, 0)]:  # test_bloom.cpp:44-48
        with pytest.raises(OracleError) as e:
            oracle.bloom_params(eps, r)
        assert e.value.kind == "Error"


def test_raw_container_bytes(oracle):
    # test_container.cpp:154-172: the 69-byte raw/raw container, CRC EC F0 F4 CB
    cfg = GpConfig.make(NONE, V_NONE)
    got = oracle.compress_pack(4, [1, 3], cfg, values=[1.5, -2.0])
    expect = bytes([ord("D"), ord("R"), ord("C"), ord("1"), 1, 0, 0, 0, 0,
                    4, 0, 0, 0, 0, 0, 0, 0, 2, 0, 0, 0, 0, 0, 0, 0,
                    8, 0, 0, 0, 0, 0, 0, 0, 8, 0, 0, 0, 0, 0, 0, 0, 0, 0, 0, 0, 0, 0, 0, 0,
                    1, 0, 0, 0, 3, 0, 0, 0, 0x00, 0x00, 0xC0, 0x3F, 0x00, 0x00, 0x00, 0xC0,
                    0xEC, 0xF0, 0xF4, 0xCB])
    assert got == expect


def test_bitmap_bytes_lsb_first(oracle):
    assert oracle.bitmap_bytes([0, 9], 16) == bytes([0x01, 0x02])  # test_gradient.cpp:81-89


def test_rle_bit_counts(oracle):
    # test_codecs.cpp:58-82: runs 1,8,1,6 → 1 + 8*4 bits = 5 bytes; varint(300) = 2 groups
    assert len(oracle.rle_encode([0, 9], 16)) == 5
    assert len(oracle.rle_encode([], 300)) == 3
    assert len(oracle.rle_encode(list(range(300)), 300)) == 3
    p = oracle.rle_encode([0, 9], 16)
    assert p == bytes([0x03, 0x10, 0x02, 0x0C, 0x00])


def test_fit_payload_exact_line(oracle):
    # test_curvefit.cpp:314-321: an exact line round trips in place
    fit, mp = oracle.value_compress(np.array([6.5, 6.0, 5.5, 5.0]), degree=1)
    assert mp.size == 0
    kind, segs = fit[0], struct.unpack_from("<H", fit, 1)[0]
    assert (kind, segs) == (0, 1)
    assert struct.unpack_from("<I", fit, len(fit) - 4)[0] == 4  # sign split


def test_fit_reorder_map(oracle):
    # test_curvefit.cpp:324-331
    _, mp = oracle.value_compress(np.array([5.0, 6.5, 5.5, 6.0]), degree=1)
    assert mp.tolist() == [1, 3, 2, 0]
    # test_curvefit.cpp:57-73: ties keep original order, zero is nonnegative
    _, mp = oracle.value_compress(np.array([1.0, 2.0, 1.0, 0.0, -1.0]), degree=0)
    assert mp.tolist() == [1, 0, 2, 3, 4]


def test_micro_container_72_bits(oracle):
    # acceptance.cpp:453-464: 8-entry tensor, bitmap + one degree-1 segment = 72 data bits
    cfg = GpConfig.make(BITMAP, V_FIT, degree=1, max_segments=1)
    b = oracle.compress_pack(8, [0, 1, 2, 3], cfg, values=[6.4, 5.8, 5.2, 4.6])
    from oracle.bindings import CpuCodec  # noqa: F401  (volume via the reference below)
    # index 8 bits + 2 coefficients * 32 bits; no reorder (already descending)
    il, vl, rl = struct.unpack_from("<QQQ", b, 25)
    assert (il, rl) == (1, 0)
    assert vl == 1 + 2 + 4 + 1 + 8 + 4


def test_top_r_tie_rule(oracle):
    # test_sparsify.cpp:32-38: magnitude ties keep the lower index
    assert oracle.top_r(np.array([2.0, -2.0, 1.0], np.float32), 1).tolist() == [0]
    assert oracle.top_r(np.array([1.0, -2.0, 3.0, 0.0], np.float32), 2).tolist() == [1, 2]
    assert oracle.top_r(np.array([0.0, -1.0, 0.0], np.float32), 3).tolist() == [0, 1, 2]


def test_positive_scan_vanishing_fpr(oracle):
    # test_bloom.cpp:162-166
    support = [10, 200, 3000, 9999]
    f = oracle.bloom_build(support, 1e-9, 77, 78)
    assert oracle.positive_scan(f, 10000).tolist() == support


def test_bloom_serialize_layout(oracle):
    f = oracle.bloom_build([5], 0.5, 0x1111, 0x2222)  # m = 2, k = 1
    m, k = struct.unpack_from("<QH", f, 0)
    assert (m, k) == (2, 1)
    assert struct.unpack_from("<QQ", f, 10) == (0x1111, 0x2222)
    assert len(f) == 26 + 1


def test_decode_error_classes(oracle):
    cfg = GpConfig.make(NONE, V_NONE)
    good = oracle.compress_pack(4, [1, 3], cfg, values=[1.5, -2.0])
    cases = {
        good[:3]: "TruncatedError",
        b"XRC1" + good[4:]: "CorruptPayloadError",
        good[:4] + b"\x02\x00" + good[6:]: "DecodeError",
        good[:-1]: "TruncatedError",
        good + b"\x00": "CorruptPayloadError",
        good[:49] + b"\x02" + good[50:]: "ChecksumError",
        good[:6] + b"\x09" + good[7:]: "UnknownMethodError",
        good[:8] + b"\x02" + good[9:]: "CorruptPayloadError",
    }
    for bad, kind in cases.items():
        with pytest.raises(OracleError) as e:
            oracle.decode(bad)
        assert e.value.kind == kind, (bad, e.value)
    for cut in range(len(good)):  # every prefix is a decode error (test_container.cpp:200-206)
        with pytest.raises(OracleError) as e:
            oracle.decode(good[:cut])
        assert e.value.kind in ("TruncatedError", "CorruptPayloadError")


def test_p0_exact_round_trip(oracle):
    # acceptance.cpp:192-223 in miniature: P0 decode reproduces the top-r values exactly
    g = synthetic_gradient(20000, rank=0)
    r = 200
    for seed in range(5):
        cfg = GpConfig.make(P0, V_NONE, fpr=0.01, seed=seed)
        d, sup, val = oracle.decode(oracle.encode_dense(g, r, cfg))
        top = oracle.top_r(g, r)
        pos = np.searchsorted(sup, top)
        assert np.array_equal(sup[pos], top)
        assert np.array_equal(val[pos], g[top].astype(np.float64))


# ---------------------------------------------------------------- vs the reference build
def _cfgs():
    out = []
    for im in (NONE, BITMAP, RLE, P0, P1, P2, PD, NAIVE):
        for vm in (V_NONE, V_F64, V_FIT):
            out.append((im, vm))
    return out


@pytest.mark.parametrize("im,vm", _cfgs())
def test_oracle_matches_reference_containers(oracle, reference, im, vm):
    rng = np.random.default_rng(im * 16 + vm)
    for trial in range(4):
        d = int(rng.integers(50, 3000))
        g = synthetic_gradient(d, rank=trial, seed=im * 100 + vm)
        if trial == 3:
            g[::7] = 0.0  # ties at zero
        r = int(max(1, round(d * rng.choice([0.01, 0.05, 0.2]))))
        cfg = GpConfig.make(im, vm, fpr=float(rng.choice([0.01, 0.001, 0.1])),
                            degree=int(rng.integers(0, 6)), seed=int(rng.integers(0, 2**63)),
                            max_segments=int(rng.choice([0, 0, 3])), pd_variant=trial % 3)
        a = oracle.encode_dense(g, r, cfg)
        b = reference.encode_dense(g, r, cfg)
        assert a == b, (im, vm, d, r, trial)
        da, sa, va = oracle.decode(a)
        db, sb, vb = reference.decode(b)
        assert da == db and np.array_equal(sa, sb)
        assert np.array_equal(va, vb)


def test_top_r_matches_reference(oracle, reference):
    rng = np.random.default_rng(7)
    for trial in range(20):
        d = int(rng.integers(1, 5000))
        g = synthetic_gradient(d, rank=trial)
        if trial % 3 == 0:
            g = np.round(g * 2).astype(np.float32)  # many magnitude ties
        r = int(rng.integers(1, d + 1))
        assert np.array_equal(oracle.top_r(g, r), reference.top_r(g, r))


def test_selection_matches_reference(oracle, reference):
    rng = np.random.default_rng(11)
    for trial in range(12):
        d = int(rng.integers(1000, 50000))
        r = int(rng.integers(5, max(6, d // 50)))
        support = np.sort(rng.choice(d, size=r, replace=False)).astype(np.uint32)
        eps = float(rng.choice([0.3, 0.1, 0.01, 0.001]))
        f = oracle.bloom_build(support, eps, int(rng.integers(0, 2**63)), int(rng.integers(0, 2**63)))
        assert f == reference.bloom_build(support, eps, *np.frombuffer(f[10:26], "<u8").tolist())
        assert np.array_equal(oracle.positive_scan(f, d), reference.positive_scan(f, d))
        for im in (P1, P2):
            assert np.array_equal(oracle.bloom_select(f, d, r, im), reference.bloom_select(f, d, r, im))
        ob, oo, om = oracle.conflict_sets(f, d)
        rb, ro, rm = reference.conflict_sets(f, d)
        assert np.array_equal(ob, rb) and np.array_equal(oo, ro) and np.array_equal(om, rm)


def test_value_codec_matches_reference(oracle, reference):
    rng = np.random.default_rng(5)
    for trial in range(30):
        n = int(rng.integers(1, 3000))
        v = rng.standard_normal(n) * (10.0 ** rng.integers(-3, 2))
        if trial % 4 == 0:
            v = np.abs(v)
        v = v.astype(np.float32).astype(np.float64)
        deg = int(rng.integers(0, 6))
        ms = int(rng.choice([0, 0, 1, 4, 9]))
        fo, mo = oracle.value_compress(v, deg, ms)
        fr, mr = reference.value_compress(v, deg, ms)
        assert np.array_equal(mo, mr)
        # bounds, degree, sign split are exact; coefficients agree to f32 rounding
        # (the shim QR and the restatement QR are the same algorithm)
        assert fo[:3] == fr[:3] and fo[-4:] == fr[-4:]
        segs = struct.unpack_from("<H", fo, 1)[0]
        assert fo[3:3 + 4 * segs + 1] == fr[3:3 + 4 * segs + 1]
        co = np.frombuffer(fo[4 + 4 * segs:-4], "<f4")
        cr = np.frombuffer(fr[4 + 4 * segs:-4], "<f4")
        assert np.allclose(co, cr, rtol=1e-5, atol=1e-6 * np.abs(cr).max())


QUANT_CASES = [(3, dict(quant_bits=7, quant_bucket=512)), (3, dict(quant_bits=1, quant_bucket=1)),
               (3, dict(quant_bits=16, quant_bucket=3)), (3, dict(quant_bits=5, quant_bucket=100)),
               (4, dict(slot_codec=0))]


@pytest.mark.parametrize("im", [0, 1, 2, 4, 5, 6, 7, 8])
@pytest.mark.parametrize("vm,kw", QUANT_CASES)
def test_quant_and_store_slot_match_reference(oracle, im, vm, kw):
    """Quantizer (codecs.cpp:290-368) and the Store byte-codec slot
    (codecs.cpp:244-288): containers and decodes byte-identical to the
    reference build, including zero buckets (no draws) and 1-bit codes."""
    from oracle.bindings import GpConfig, reference, synthetic_gradient
    ref = reference()
    if ref is None:
        pytest.skip("oracle/_ref not built")
    d, r = 20_000, 300
    g = synthetic_gradient(d, rank=im)
    g[:5000] = 0.0  # all-zero buckets when the support reaches them
    cfg = GpConfig.make(im, vm, seed=9, **kw)
    a, b = oracle.encode_dense(g, r, cfg), ref.encode_dense(g, r, cfg)
    assert a == b
    _, sa, va = oracle.decode(a)
    _, sb, vb = ref.decode(b)
    assert np.array_equal(sa, sb) and np.array_equal(va, vb)


def test_quant_decode_errors_match_reference(oracle):
    from oracle.bindings import GpConfig, OracleError, reference, synthetic_gradient
    ref = reference()
    if ref is None:
        pytest.skip("oracle/_ref not built")
    g = synthetic_gradient(5_000, rank=1)
    for vm, kw in QUANT_CASES:
        c = bytearray(oracle.encode_dense(g, 50, GpConfig.make(1, vm, seed=2, **kw)))
        il = int.from_bytes(c[25:33], "little")
        vo = 49 + il
        muts = [bytes(c[:vo]) + bytes([0]) + bytes(c[vo + 1:]), bytes(c[:vo]) + bytes([17]) + bytes(c[vo + 1:]),
                bytes(c[:vo]) + bytes([9]) + bytes(c[vo + 1:]), bytes(c[:vo + 1]) + bytes(4) + bytes(c[vo + 5:])]
        for m in muts:
            m = bytearray(m)
            m[-4:] = oracle.crc32c(bytes(m[49:-4])).to_bytes(4, "little")  # valid CRC: reach the payload checks
            m = bytes(m)
            outs = []
            for cod in (oracle, ref):
                try:
                    cod.decode(m)
                    outs.append("ok")
                except OracleError as e:
                    outs.append(e.code)
            assert outs[0] == outs[1], (vm, kw, outs)


def test_driver_random_r_matches_reference():
    """drivers.random_r (the sweep's random-r sparsifier) against sparsify.cpp:48-58."""
    from oracle.bindings import reference
    from paper_2102_03112_b200.drivers import random_r
    ref = reference()
    if ref is None:
        pytest.skip("oracle/_ref not built")
    for d, r, seed in [(10, 10, 1), (1000, 10, 2), (5000, 2500, 3), (70_000, 700, 4)]:
        assert np.array_equal(random_r(d, r, seed), ref.random_r(d, r, seed))


@pytest.mark.parametrize("d", [1, 2, 7, 255, 256, 257, 1000, 65536, 65537, 100_003, 2_000_000])
def test_huffman_index_matches_reference(oracle, d):
    """Huffman index (codecs.cpp:72-242, pipeline.cpp:179-184, :254-258): the
    canonical table derived from d alone, MSB-first codes, byte-identical."""
    from oracle.bindings import GpConfig, reference, synthetic_gradient
    ref = reference()
    if ref is None:
        pytest.skip("oracle/_ref not built")
    g = synthetic_gradient(d, rank=d % 7)
    for r in sorted({1, max(1, d // 100), max(1, d // 3), d}):
        if r > 100_000:
            continue
        cfg = GpConfig.make(3, 0, seed=4)
        a, b = oracle.encode_dense(g, r, cfg), ref.encode_dense(g, r, cfg)
        assert a == b, r
        _, sa, va = oracle.decode(a)
        _, sb, vb = ref.decode(b)
        assert np.array_equal(sa, sb) and np.array_equal(va, vb)


def test_huffman_decode_errors_match_reference(oracle):
    from oracle.bindings import GpConfig, OracleError, reference, synthetic_gradient
    ref = reference()
    if ref is None:
        pytest.skip("oracle/_ref not built")
    rng = np.random.default_rng(3)
    for d, r in [(1000, 10), (70_000, 300), (300, 300)]:
        c = bytearray(oracle.encode_dense(synthetic_gradient(d, rank=1), r, GpConfig.make(3, 0, seed=2)))
        il = int.from_bytes(c[25:33], "little")
        muts = []
        for _ in range(12):  # bit flips inside the index payload
            m = bytearray(c)
            pos = 49 + int(rng.integers(0, il))
            m[pos] ^= 1 << int(rng.integers(0, 8))
            muts.append(m)
        for cut in (1, 2):  # index payload shortened (lengths rewritten)
            m = bytearray(c[:49 + il - cut] + c[49 + il:])
            m[25:33] = (il - cut).to_bytes(8, "little")
            muts.append(m)
        m = bytearray(c[:49 + il] + b"\x00" + c[49 + il:])  # one trailing byte
        m[25:33] = (il + 1).to_bytes(8, "little")
        muts.append(m)
        for m in muts:
            m[-4:] = oracle.crc32c(bytes(m[49:-4])).to_bytes(4, "little")
            outs = []
            for cod in (oracle, ref):
                try:
                    _, s, v = cod.decode(bytes(m))
                    outs.append(("ok", s.tobytes(), v.tobytes()))
                except OracleError as e:
                    outs.append(e.code)
            assert outs[0] == outs[1], (d, r, outs[0] if not isinstance(outs[0], tuple) else "ok",
                                        outs[1] if not isinstance(outs[1], tuple) else "ok")
