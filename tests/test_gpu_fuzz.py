"""Randomised corruption of valid containers, every method on the device:
the GPU decoder must agree with the oracle (or, for fit-dexp, the reference
build) on the outcome of every mutated container — the same error class, or
the same decoded sparse gradient.  Mutations flip bits or bytes inside one
payload and re-seal the CRC, so the checks past the checksum are exercised.
Documented device capacity limits (GP_CAPACITY) are the only allowed
divergence, besides host allocation failures of the CPU checkers
on absurd Bloom filter widths."""
import numpy as np
import pytest
import torch

from oracle.bindings import GpConfig, OracleError, reference, synthetic_gradient

pytestmark = pytest.mark.gpu

METHODS = [(0, 0, {}), (1, 0, {}), (2, 0, {}), (3, 0, {}), (1, 5, {}), (1, 1, {}), (2, 3, dict(quant_bits=6)),
           (1, 4, dict(slot_codec=0)), (4, 0, {}), (5, 0, {}), (6, 0, {}), (7, 0, dict(pd_variant=2)),
           (6, 1, {}), (3, 3, dict(quant_bits=3, quant_bucket=17))]


@pytest.fixture(scope="module")
def codec():
    from paper_2102_03112_b200 import Codec
    c = Codec(max_d=1 << 18)
    yield c
    c.close()


def _outcome_cpu(cod, blob):
    try:
        _, s, v = cod.decode(blob)
        return ("ok", s.astype(np.uint32).tobytes(), v.tobytes())
    except OracleError as e:
        return e.kind


def _outcome_gpu(codec, blob):
    from paper_2102_03112_b200 import Error
    try:
        _, s, v = codec.decompress(torch.from_numpy(np.frombuffer(blob, np.uint8).copy()).cuda())
        return ("ok", s.cpu().numpy().astype(np.uint32).tobytes(), v.cpu().numpy().tobytes())
    except Error as e:
        return {"CapacityError": "Capacity", "UnsupportedMethodError": "Unsupported"}.get(type(e).__name__,
                                                                                         type(e).__name__)


@pytest.mark.parametrize("im,vm,kw", METHODS)
def test_mutated_containers_agree(codec, oracle, im, vm, kw):
    rng = np.random.default_rng(1000 * im + vm)
    d, r = 20_000, 150
    g = synthetic_gradient(d, rank=im + vm)
    c = bytearray(oracle.encode_dense(g, r, GpConfig.make(im, vm, fpr=0.05, seed=11, **kw)))
    il, vl, rl = (int.from_bytes(c[o:o + 8], "little") for o in (25, 33, 41))
    regions = [(49, il), (49 + il, vl), (49 + il + vl, rl)]
    regions = [(a, n) for a, n in regions if n > 0]
    checked = 0
    for t in range(80):
        m = bytearray(c)
        a, n = regions[t % len(regions)]
        pos = a + int(rng.integers(0, n))
        if t % 3 == 0:
            m[pos] = int(rng.integers(0, 256))
        else:
            m[pos] ^= 1 << int(rng.integers(0, 8))
        m[-4:] = oracle.crc32c(bytes(m[49:-4])).to_bytes(4, "little")
        blob = bytes(m)
        want = _outcome_cpu(oracle, blob)
        got = _outcome_gpu(codec, blob)
        if got == "Capacity":
            continue
        if want == "Error" and im >= 4 and a == 49 and pos - a < 8:
            # an absurd filter width m: the CPU checkers fail allocating the filter
            # (std::bad_alloc in the reference, before any payload check); the
            # device applies the next format check (the payload is short)
            continue
        assert got == want, (im, vm, t, pos - a, got if isinstance(got, str) else "ok",
                             want if isinstance(want, str) else "ok")
        checked += 1
    assert checked >= 60


def test_mutated_dexp_containers_agree(codec):
    ref = reference()
    if ref is None:
        pytest.skip("oracle/_ref missing")
    rng = np.random.default_rng(7)
    d, r = 20_000, 300
    c = bytearray(ref.encode_dense(synthetic_gradient(d, rank=2), r, GpConfig.make(1, 2, seed=3)))
    il, vl = (int.from_bytes(c[o:o + 8], "little") for o in (25, 33))
    for t in range(30):
        m = bytearray(c)
        pos = 49 + il + int(rng.integers(0, vl))
        m[pos] ^= 1 << int(rng.integers(0, 8))
        from oracle.bindings import oracle as _o
        m[-4:] = _o().crc32c(bytes(m[49:-4])).to_bytes(4, "little")
        blob = bytes(m)
        want = _outcome_cpu(ref, blob)
        got = _outcome_gpu(codec, blob)
        if isinstance(want, tuple) and isinstance(got, tuple):
            assert got[1] == want[1]
            gv, wv = np.frombuffer(got[2]), np.frombuffer(want[2])
            assert np.allclose(gv, wv, rtol=1e-12, atol=0, equal_nan=True)
        else:
            assert got == want, (t, got if isinstance(got, str) else "ok", want if isinstance(want, str) else "ok")
