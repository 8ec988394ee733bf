"""The N = 2 exchange on the CUDA codec: two processes share the GPU over gloo
(the only two-rank transport one GPU allows; NCCL needs a device per rank).

Each rank runs paper_2102_03112_b200.dp.SparseAllgather — encode, sizes-first
allgather, padded payload allgather, rank-order decode with scale 1/2 — with
the Bloom positive scans sharded by coordinate range (shard_scan, the default
at N > 1) or not.  Both ranks must hold the same dense mean
(harness.cpp:287-288), bit-identical to the same worker loop replayed in one
process through the codec (encode with Simulation::pipeline_seed(1, rank,
step), decode in rank order), whose pieces the parity suites pin to the
reference; with compensation the f64 residuals must match too.
"""
import os
import socket

import numpy as np
import pytest
import torch
import torch.multiprocessing as mp

from oracle.bindings import synthetic_gradient

pytestmark = pytest.mark.gpu

CASES = {  # name: (index, value, fpr)
    "p2fit": (6, 1, 0.001),
    "p0fit": (4, 1, 0.01),
    "p1raw": (5, 0, 0.01),
    "bitmap": (1, 0, 0.01),
}


def _port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _worker(rank, world, port, name, d, r, steps, shard, ef, q):
    import torch.distributed as dist
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    from paper_2102_03112_b200 import Codec, PipelineConfig
    from paper_2102_03112_b200.dp import SparseAllgather
    im, vm, fpr = CASES[name]
    codec = Codec(max_d=d)
    ex = SparseAllgather(codec, d, r, PipelineConfig(index_method=im, value_method=vm, fpr=fpr), ef=ef,
                         shard_scan=shard)
    g = torch.from_numpy(synthetic_gradient(d, rank=rank)).cuda()
    outs, res = [], []
    for step in range(steps):
        outs.append(ex.step(g, step=step).cpu().numpy().copy())
        ex.check()
        res.append(ex.residual.cpu().numpy().copy() if ex.residual is not None else None)
    q.put((rank, outs, res, bool(ex.shard)))
    codec.close()
    dist.destroy_process_group()


def _replay(name, d, r, steps, world, ef):
    from paper_2102_03112_b200 import Codec, PipelineConfig
    from paper_2102_03112_b200.seeds import pipeline_seed
    im, vm, fpr = CASES[name]
    codec = Codec(max_d=d)
    grads = [torch.from_numpy(synthetic_gradient(d, rank=k)).cuda() for k in range(world)]
    res = [torch.zeros(d, dtype=torch.float64, device="cuda") for _ in range(world)]
    means, resids = [], []
    try:
        for step in range(steps):
            cs = []
            for k in range(world):
                cfg = PipelineConfig(index_method=im, value_method=vm, fpr=fpr, seed=pipeline_seed(1, k, step))
                cs.append(codec.compress_ef64(grads[k], res[k], r, cfg) if ef else codec.compress(grads[k], r, cfg))
            mean = torch.zeros(d, dtype=torch.float32, device="cuda")
            for k in range(world):
                codec.decode_accumulate(cs[k], mean, scale=1.0 / world)
            codec.status()
            means.append(mean.cpu().numpy())
            resids.append([x.cpu().numpy().copy() for x in res])
    finally:
        codec.close()
    return means, resids


@pytest.mark.parametrize("name,shard,ef", [("p2fit", True, False), ("p2fit", False, False), ("p0fit", True, False),
                                           ("p1raw", True, True), ("bitmap", None, True)])
def test_world2_on_one_gpu_matches_the_worker_loop(name, shard, ef):
    world, d, r, steps = 2, 400_003, 4_000, 3
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _port()
    procs = [ctx.Process(target=_worker, args=(k, world, port, name, d, r, steps, shard, ef, q)) for k in range(world)]
    for p in procs:
        p.start()
    got = dict((x[0], x[1:]) for x in (q.get(timeout=600) for _ in range(world)))
    for p in procs:
        p.join(timeout=120)
        assert p.exitcode == 0
    if shard is not None:
        assert got[0][2] == bool(shard)
    means, resids = _replay(name, d, r, steps, world, ef)
    for step in range(steps):
        assert np.array_equal(got[0][0][step], got[1][0][step]), "replicas diverged"
        assert np.array_equal(got[0][0][step], means[step]), f"step {step}: mean differs from the worker loop"
        if ef:
            for k in range(world):
                assert np.array_equal(got[k][1][step], resids[step][k]), f"rank {k} step {step}: residual differs"


def test_bloom_scan_range_slices(oracle):
    """gp_bloom_scan_range over arbitrary slices equals the full positive_scan
    (bloom.cpp:123-128) restricted to the slice; slices concatenate to it."""
    from paper_2102_03112_b200 import Codec
    d, r = 1_000_003, 10_000
    g = synthetic_gradient(d, rank=3)
    codec = Codec(max_d=d)
    try:
        for eps in (0.001, 0.05):
            filt = oracle.bloom_build(oracle.top_r(g, r), eps, 0xAB, 0xCD)
            full = oracle.positive_scan(filt, d)
            f = torch.from_numpy(np.frombuffer(filt, np.uint8).copy()).cuda()
            cuts = [0, 1, 31, 4097, 333_334, 666_667, d - 5, d]
            out = torch.empty(d, dtype=torch.int32, device="cuda")
            cnt = torch.zeros(1, dtype=torch.int64, device="cuda")
            parts = []
            for lo, hi in zip(cuts[:-1], cuts[1:]):
                codec.bloom_scan_range_into(f, d, lo, hi, out, cnt)
                codec.status()
                got = out[: int(cnt.item())].cpu().numpy().astype(np.uint32)
                assert np.array_equal(got, full[(full >= lo) & (full < hi)]), (eps, lo, hi)
                parts.append(got)
            codec.bloom_scan_range_into(f, d, 77, 77, out, cnt)  # empty slice
            assert int(cnt.item()) == 0
            assert np.array_equal(np.concatenate(parts), full)
    finally:
        codec.close()
