"""Huffman index (id 3) on the device vs the CPU oracle (pinned byte-for-byte
to the reference build in tests/test_oracle.py): container bytes, decoded
supports, and the error class of corrupted streams (bit flips, truncation,
trailing bytes) — the chunked speculative decoder must report the first error
in stream order as the sequential decoder does."""
import numpy as np
import pytest
import torch

from oracle.bindings import GpConfig, OracleError, synthetic_gradient

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def codec():
    from paper_2102_03112_b200 import Codec
    c = Codec(max_d=1 << 22)
    yield c
    c.close()


def _dev(a):
    return torch.from_numpy(np.array(a, copy=True)).cuda()


@pytest.mark.parametrize("d", [1, 2, 7, 255, 256, 257, 1000, 65536, 65537, 100_003, 1_000_000, 4_000_000])
def test_encode_decode_bit_exact(codec, oracle, d):
    from paper_2102_03112_b200 import PipelineConfig
    g = synthetic_gradient(d, rank=d % 5)
    for r in sorted({1, max(1, d // 100), max(1, d // 3), d}):
        if r > 1_500_000:
            continue
        for vm in (0, 1):
            cfg = PipelineConfig(index_method=3, value_method=vm, seed=r)
            got = codec.compress(_dev(g), r, cfg).cpu().numpy().tobytes()
            want = oracle.encode_dense(g, r, GpConfig.make(3, vm, seed=r))
            if vm == 0:
                assert got == want, (d, r)
            c = want
            dd, sup, val = codec.decompress(_dev(np.frombuffer(c, np.uint8)))
            od, osup, oval = oracle.decode(c)
            assert dd == od
            assert np.array_equal(sup.cpu().numpy().astype(np.uint32), osup)
            assert np.array_equal(val.cpu().numpy(), oval)


def test_decode_error_classes_match_oracle(codec, oracle):
    from paper_2102_03112_b200 import Error
    rng = np.random.default_rng(11)
    for d, r in [(1000, 10), (70_000, 300), (300, 300), (2_000_000, 5_000)]:
        c = bytearray(oracle.encode_dense(synthetic_gradient(d, rank=2), r, GpConfig.make(3, 0, seed=2)))
        il = int.from_bytes(c[25:33], "little")
        muts = []
        for _ in range(16):
            m = bytearray(c)
            pos = 49 + int(rng.integers(0, il))
            m[pos] ^= 1 << int(rng.integers(0, 8))
            muts.append(m)
        for cut in (1, 3):
            m = bytearray(c[:49 + il - cut] + c[49 + il:])
            m[25:33] = (il - cut).to_bytes(8, "little")
            muts.append(m)
        m = bytearray(c[:49 + il] + b"\x00" + c[49 + il:])
        m[25:33] = (il + 1).to_bytes(8, "little")
        muts.append(m)
        for m in muts:
            m[-4:] = oracle.crc32c(bytes(m[49:-4])).to_bytes(4, "little")
            bad = bytes(m)
            try:
                _, osup, oval = oracle.decode(bad)
                want = None
            except OracleError as e:
                want = e.kind
            dense = torch.zeros(d, dtype=torch.float32, device="cuda")
            got = None
            try:
                codec.decode_accumulate(_dev(np.frombuffer(bad, np.uint8)), dense, length=len(bad))
                codec.status()
            except Error as e:
                got = type(e).__name__
            assert got == want, (d, r, got, want)
            if want is None:
                ref = np.zeros(d, np.float32)
                ref[osup.astype(np.int64)] = oval.astype(np.float32)
                assert np.array_equal(dense.cpu().numpy(), ref)
            else:
                assert float(dense.abs().sum()) == 0.0


def test_huffman_in_dp_graph_and_ef(oracle):
    from oracle.ef import ef_step
    from paper_2102_03112_b200 import Codec, PipelineConfig
    from paper_2102_03112_b200.dp import SparseAllgather, pipeline_seed
    d, r = 120_000, 1_500
    codec = Codec(max_d=d)
    ex = SparseAllgather(codec, d, r, PipelineConfig(index_method=3, value_method=0), ef="f32", graph=True)
    g = torch.empty(d, dtype=torch.float32, device="cuda")
    e = np.zeros(d, np.float32)
    for step in range(3):
        gh = synthetic_gradient(d, rank=step)
        g.copy_(torch.from_numpy(gh))
        ex.step(g, step=step)
        torch.cuda.synchronize()
        codec.status()
        c, e = ef_step(oracle, gh, e, r, GpConfig.make(3, 0, seed=pipeline_seed(1, 0, step)))
        assert bytes(ex.out[: int(ex.length.item())].cpu().numpy()) == c
        assert np.array_equal(ex.residual.cpu().numpy(), e)
    codec.close()


def test_sequential_fallback_path(codec, oracle, monkeypatch):
    """With no settling rounds the chunk check fails and the single-thread
    decoder runs: same supports, same error classes."""
    from paper_2102_03112_b200 import Error
    monkeypatch.setenv("GP_HUFF_FIX_ROUNDS", "0")
    for d, r in [(50_000, 500), (3000, 3000)]:
        c = oracle.encode_dense(synthetic_gradient(d, rank=4), r, GpConfig.make(3, 0, seed=9))
        _, sup, val = codec.decompress(_dev(np.frombuffer(c, np.uint8)))
        _, osup, oval = oracle.decode(c)
        assert np.array_equal(sup.cpu().numpy().astype(np.uint32), osup)
        m = bytearray(c)
        il = int.from_bytes(m[25:33], "little")
        m = bytearray(m[:49 + il - 1] + m[49 + il:])
        m[25:33] = (il - 1).to_bytes(8, "little")
        m[-4:] = oracle.crc32c(bytes(m[49:-4])).to_bytes(4, "little")
        with pytest.raises(OracleError) as oe:
            oracle.decode(bytes(m))
        with pytest.raises(Error) as ge:
            codec.decompress(_dev(np.frombuffer(bytes(m), np.uint8)))
        assert type(ge.value).__name__ == oe.value.kind
