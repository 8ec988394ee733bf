"""The N = 1 DP step as one CUDA graph (SparseAllgather(graph=True)): replays
with the per-step pipeline seed computed on the device must equal eager steps
bit for bit — containers, dense means and error-feedback residuals — and the
host-buffer pipeline must run unchanged over it."""
import numpy as np
import pytest
import torch

from oracle.bindings import synthetic_gradient

pytestmark = pytest.mark.gpu

CASES = [dict(index_method=6, value_method=1, fpr=0.001), dict(index_method=1, value_method=0),
         dict(index_method=4, value_method=3, fpr=0.01), dict(index_method=5, value_method=0),
         dict(index_method=2, value_method=5)]


@pytest.mark.parametrize("ef", [False, True])
@pytest.mark.parametrize("kw", CASES)
def test_graph_replay_equals_eager(kw, ef):
    from paper_2102_03112_b200 import Codec, PipelineConfig
    from paper_2102_03112_b200.dp import SparseAllgather
    d, r = 300_001, 3_000
    cfg = PipelineConfig(**kw)
    ca, cb = Codec(max_d=d), Codec(max_d=d)
    eager = SparseAllgather(ca, d, r, cfg, ef=ef)
    graph = SparseAllgather(cb, d, r, cfg, ef=ef, graph=True)
    assert graph.graph
    g = torch.empty(d, dtype=torch.float32, device="cuda")  # stable input buffer (one graph)
    for step in [4, 5, 9, 5]:
        g.copy_(torch.from_numpy(synthetic_gradient(d, rank=step)))
        want = eager.step(g, step=step).clone()
        got = graph.step(g, step=step).clone()
        torch.cuda.synchronize()
        ca.status()
        cb.status()
        n = int(eager.length.item())
        assert int(graph.length.item()) == n
        assert torch.equal(eager.out[:n], graph.out[:n]), f"step {step}: containers differ"
        assert torch.equal(want, got), f"step {step}: dense means differ"
        if ef:
            assert torch.equal(eager.residual, graph.residual)
    assert len(graph.graphs) == 1 and graph.kernels_per_step > 5
    ca.close()
    cb.close()


def test_host_pipeline_over_graphs():
    from paper_2102_03112_b200 import Codec, PipelineConfig
    from paper_2102_03112_b200.dp import HostPipeline, SparseAllgather
    d, r = 200_000, 2_000
    cfg = PipelineConfig(index_method=6, value_method=1, fpr=0.001)
    ca, cb = Codec(max_d=d), Codec(max_d=d)
    eager = SparseAllgather(ca, d, r, cfg)
    graph = SparseAllgather(cb, d, r, cfg, graph=True)
    grads = [synthetic_gradient(d, rank=w) for w in range(4)]
    want = [eager.step(torch.from_numpy(g).cuda(), step=i).cpu().numpy().copy() for i, g in enumerate(grads)]
    pipe = HostPipeline(graph, d)
    ins = [torch.from_numpy(g).pin_memory() for g in grads]
    outs = [torch.empty(d, dtype=torch.float32).pin_memory() for _ in grads]
    for i in range(4):
        pipe.submit(ins[i], outs[i], step=i)
    pipe.drain()
    cb.status()
    for i in range(4):
        assert np.array_equal(outs[i].numpy(), want[i])
    assert len(graph.graphs) == 2  # one per double-buffer slot
    ca.close()
    cb.close()


@pytest.mark.parametrize("ef", [False, True])
def test_bucketed_graph_equals_eager(ef):
    from paper_2102_03112_b200 import Codec, PipelineConfig
    from paper_2102_03112_b200.dp import BucketedSparseAllgather
    d, ratio, buckets = 800_003, 0.005, 5
    cfg = PipelineConfig(index_method=6, value_method=1, fpr=0.001, max_segments=8)
    eager = BucketedSparseAllgather(lambda dm: Codec(max_d=dm), d, ratio, cfg, buckets, streams=3, ef=ef)
    graph = BucketedSparseAllgather(lambda dm: Codec(max_d=dm), d, ratio, cfg, buckets, streams=3, ef=ef, graph=True)
    assert graph.graph
    g = torch.empty(d, dtype=torch.float32, device="cuda")
    for step in [2, 3, 7]:
        g.copy_(torch.from_numpy(synthetic_gradient(d, rank=step)))
        want = eager.step(g, step=step).clone()
        got = graph.step(g, step=step).clone()
        torch.cuda.synchronize()
        for c in eager.codecs + graph.codecs:
            c.status()
        for ea, eb in zip(eager.ex, graph.ex):
            n = int(ea.length.item())
            assert int(eb.length.item()) == n and torch.equal(ea.out[:n], eb.out[:n])
            if ef:
                assert torch.equal(ea.residual, eb.residual)
        assert torch.equal(want, got), f"step {step}"
    assert len(graph.graphs) == 1


@pytest.mark.parametrize("ef", [False, True])
@pytest.mark.parametrize("graph", [False, True])
@pytest.mark.parametrize("kw", [dict(index_method=6, value_method=1, fpr=0.001), dict(index_method=4, value_method=0),
                                dict(index_method=5, value_method=3), dict(index_method=7, value_method=0, pd_variant=1)])
def test_early_index_decode_equals_plain(kw, graph, ef):
    """The own container's Bloom index stage run early on a second context
    (gp_decode_index_prepare + gp_decode_accumulate_own) equals the plain
    encode → decode step bit for bit."""
    from paper_2102_03112_b200 import Codec, PipelineConfig
    from paper_2102_03112_b200.dp import SparseAllgather
    d, r = 300_001, 3_000
    cfg = PipelineConfig(**kw)
    ca, cb, ce = Codec(max_d=d), Codec(max_d=d), Codec(max_d=d)
    plain = SparseAllgather(ca, d, r, cfg, ef=ef)
    early = SparseAllgather(cb, d, r, cfg, graph=graph, early_codec=ce, ef=ef)
    assert early.early is not None
    g = torch.empty(d, dtype=torch.float32, device="cuda")
    for step in [1, 2, 6]:
        g.copy_(torch.from_numpy(synthetic_gradient(d, rank=step)))
        want = plain.step(g, step=step).clone()
        got = early.step(g, step=step).clone()
        torch.cuda.synchronize()
        for c in (ca, cb, ce):
            c.status()
        n = int(plain.length.item())
        assert int(early.length.item()) == n and torch.equal(plain.out[:n], early.out[:n])
        assert torch.equal(want, got), f"step {step}"
        if ef:
            assert torch.equal(plain.residual, early.residual)
    for c in (ca, cb, ce):
        c.close()
