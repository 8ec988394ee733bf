"""The DP step on one GPU (N = 1): SparseAllgather / BucketedSparseAllgather
against the oracle's encode → decode of the same pipeline seed, and the
host-buffer HostPipeline (overlapped copies) against the plain device step."""
import numpy as np
import pytest
import torch

from oracle.bindings import GpConfig, synthetic_gradient

pytestmark = pytest.mark.gpu

BITMAP, P2 = 1, 6
V_NONE, V_FIT = 0, 1


def _pcfg(im, vm, **kw):
    from paper_2102_03112_b200 import PipelineConfig
    return PipelineConfig(index_method=im, value_method=vm, **kw)


@pytest.mark.parametrize("im,vm,fpr", [(BITMAP, V_NONE, 0.01), (P2, V_FIT, 0.001)])
def test_dp_step_matches_oracle(oracle, im, vm, fpr):
    from paper_2102_03112_b200 import Codec
    from paper_2102_03112_b200.dp import SparseAllgather, pipeline_seed
    d, r = 300_000, 3_000
    g = synthetic_gradient(d, rank=0)
    codec = Codec(max_d=d)
    ex = SparseAllgather(codec, d, r, _pcfg(im, vm, fpr=fpr))
    dense = ex.step(torch.from_numpy(g).cuda(), step=5).cpu().numpy()
    codec.status()
    c = oracle.encode_dense(g, r, GpConfig.make(im, vm, fpr=fpr, seed=pipeline_seed(1, 0, 5)))
    assert bytes(ex.out[: int(ex.length.item())].cpu().numpy()) == c
    ref = np.zeros(d, np.float64)
    oracle.decode_accumulate(c, ref, 1.0)
    # one f32 term per coordinate: the decoded value rounded to f32 (fit values are f64)
    assert np.array_equal(dense, ref.astype(np.float32))
    codec.close()


def test_host_pipeline_matches_device_step():
    from paper_2102_03112_b200 import Codec
    from paper_2102_03112_b200.dp import HostPipeline, SparseAllgather
    d, r = 400_000, 4_000
    codec = Codec(max_d=d)
    ex = SparseAllgather(codec, d, r, _pcfg(P2, V_FIT, fpr=0.001))
    grads = [synthetic_gradient(d, rank=w) for w in range(3)]
    want = []
    for i, g in enumerate(grads):
        want.append(ex.step(torch.from_numpy(g).cuda(), step=i).cpu().numpy().copy())
    codec.status()
    pipe = HostPipeline(ex, d)
    ins = [torch.from_numpy(g).pin_memory() for g in grads]
    outs = [torch.empty(d, dtype=torch.float32).pin_memory() for _ in grads]
    for i in range(3):
        pipe.submit(ins[i], outs[i], step=i)
    pipe.drain()
    codec.status()
    for i in range(3):
        assert np.array_equal(outs[i].numpy(), want[i])
    codec.close()


def test_bucketed_step_is_bucketwise():
    from paper_2102_03112_b200 import Codec
    from paper_2102_03112_b200.dp import BucketedSparseAllgather, SparseAllgather
    d, ratio, buckets = 600_001, 0.01, 4
    g = torch.from_numpy(synthetic_gradient(d, rank=2)).cuda()
    cfg = _pcfg(BITMAP, V_NONE)
    bex = BucketedSparseAllgather(lambda dm: Codec(max_d=dm), d, ratio, cfg, buckets, streams=2)
    got = bex.step(g, step=3).clone()
    torch.cuda.synchronize()
    for c in bex.codecs:
        c.status()
    from dataclasses import replace
    for b, (lo, hi) in enumerate(bex.bounds):
        codec = Codec(max_d=hi - lo)
        one = SparseAllgather(codec, hi - lo, bex.rs[b], cfg)
        want = one.step_seeded(g[lo:hi], replace(cfg, seed=bex.bucket_seed(1, 3, b)))
        assert torch.equal(got[lo:hi], want)
        codec.close()


def test_dp_step_with_error_feedback_matches_oracle(oracle):
    """ef="f32": three compensated steps at N = 1 against the oracle's f32 worker loop."""
    from oracle.ef import ef_step
    from paper_2102_03112_b200 import Codec
    from paper_2102_03112_b200.dp import SparseAllgather, pipeline_seed
    d, r = 250_000, 2_500
    codec = Codec(max_d=d)
    ex = SparseAllgather(codec, d, r, _pcfg(P2, V_NONE, fpr=0.001), ef="f32")
    e = np.zeros(d, np.float32)
    for step in range(3):
        g = synthetic_gradient(d, rank=step)
        dense = ex.step(torch.from_numpy(g).cuda(), step=step).cpu().numpy()
        codec.status()
        c, e = ef_step(oracle, g, e, r, GpConfig.make(P2, V_NONE, fpr=0.001, seed=pipeline_seed(1, 0, step)))
        assert bytes(ex.out[: int(ex.length.item())].cpu().numpy()) == c
        assert np.array_equal(ex.residual.cpu().numpy(), e)
        ref = np.zeros(d, np.float64)
        oracle.decode_accumulate(c, ref, 1.0)
        assert np.array_equal(dense, ref.astype(np.float32))
    codec.close()


def test_concurrent_peer_decode_equals_sequential():
    """The N > 1 decode split (gp_decode_prepare on per-peer contexts/streams,
    gp_decode_finish in rank order) equals sequential decode_accumulate bit for
    bit; exercised on one GPU with containers of 5 simulated ranks."""
    from paper_2102_03112_b200 import Codec
    from paper_2102_03112_b200.dp import SparseAllgather, pipeline_seed
    from dataclasses import replace
    d, r, n = 200_000, 2_000, 5
    cfg = _pcfg(P2, V_FIT, fpr=0.001)
    enc = Codec(max_d=d)
    ex = SparseAllgather(enc, d, r, cfg, decode_codecs=[Codec(max_d=d) for _ in range(2)])
    outs, sizes = [], []
    for w in range(n):
        enc.encode_into(torch.from_numpy(synthetic_gradient(d, rank=w)).cuda(), r,
                        replace(cfg, seed=pipeline_seed(1, w, 0)), ex.out, ex.length)
        torch.cuda.synchronize()
        sizes.append(int(ex.length.item()))
        outs.append(ex.out[: sizes[-1]].clone())
    mx = max(sizes)
    ex.recv = torch.zeros(n * mx, dtype=torch.uint8, device="cuda")
    ex.sizes = torch.tensor(sizes, dtype=torch.int64, device="cuda")
    for j in range(n):
        ex.recv[j * mx: j * mx + sizes[j]] = outs[j]
    got = torch.zeros(d, dtype=torch.float32, device="cuda")
    ex._decode_concurrent(n, mx, got, torch.cuda.current_stream())
    want = torch.zeros(d, dtype=torch.float32, device="cuda")
    for j in range(n):
        enc.decode_accumulate(outs[j], want, scale=1.0 / n, hint=cfg)
    torch.cuda.synchronize()
    for c in ex.dec:
        c.status()
    assert torch.equal(got, want)


def test_dp_step_with_f64_error_feedback_matches_the_reference_loop(reference):
    """ef=True (f64, the reference's precision): three compensated steps at N = 1
    bit-identical to the reference build's own loop (harness.cpp:230-271)."""
    from paper_2102_03112_b200 import Codec
    from paper_2102_03112_b200.dp import SparseAllgather, pipeline_seed
    d, r = 250_000, 2_500
    codec = Codec(max_d=d)
    ex = SparseAllgather(codec, d, r, _pcfg(P2, V_NONE, fpr=0.001), ef=True)
    e = np.zeros(d, np.float64)
    try:
        for step in range(3):
            g = synthetic_gradient(d, rank=step)
            ex.step(torch.from_numpy(g).cuda(), step=step)
            codec.status()
            c = reference.ef_step64(g, e, r, GpConfig.make(P2, V_NONE, fpr=0.001, seed=pipeline_seed(1, 0, step)))
            assert bytes(ex.out[: int(ex.length.item())].cpu().numpy()) == c
            assert np.array_equal(ex.residual.cpu().numpy(), e)
    finally:
        codec.close()
