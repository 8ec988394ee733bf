"""The N > 1 exchange path on CPU: world_size-2 gloo process groups.

paper_2102_03112_b200.dp runs unchanged on CPU tensors with the gloo backend;
the codec is a CPU stand-in built on the oracle (this file), so the test
checks the exchange logic itself — sizes-first allgather, padding to the
largest container, rank-order decode with scale 1/N, the bucket seeding — and
that both replicas end with identical dense means (harness.cpp:287-288),
against a sequential replay of Simulation::step's worker loop.
"""
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from oracle.bindings import GpConfig, oracle, synthetic_gradient
from paper_2102_03112_b200 import IndexMethod, PipelineConfig, ValueMethod
from paper_2102_03112_b200._lib import lib


class OracleCodec:
    """CPU stand-in with Codec's exchange-facing interface (test infrastructure)."""

    @staticmethod
    def max_container_bytes(d, r, cfg):
        import ctypes
        c = cfg.to_c()
        return int(lib.gp_max_container_bytes(d, r, ctypes.byref(c)))

    @staticmethod
    def _c(cfg):
        return GpConfig.make(int(cfg.index_method), int(cfg.value_method), fpr=cfg.fpr, degree=cfg.degree,
                             max_segments=cfg.max_segments, seed=cfg.seed, pd_variant=cfg.pd_variant)

    def encode_into(self, grad, r, cfg, out, length, support=None, stream=None):
        b = oracle().encode_dense(grad.contiguous().numpy(), r, self._c(cfg))
        out[: len(b)] = torch.frombuffer(bytearray(b), dtype=torch.uint8)
        length[0] = len(b)

    def encode_ef_into(self, grad, residual, r, cfg, out, length, stream=None):
        from oracle.ef import ef_step
        b, res = ef_step(oracle(), grad.contiguous().numpy(), residual.numpy(), r, self._c(cfg))
        out[: len(b)] = torch.frombuffer(bytearray(b), dtype=torch.uint8)
        length[0] = len(b)
        residual.copy_(torch.from_numpy(res))

    def encode_ef64_into(self, grad, residual, r, cfg, out, length, stream=None):
        from oracle.bindings import reference
        res = residual.numpy()  # f64, updated in place by the reference's own loop
        b = reference().ef_step64(grad.contiguous().numpy(), res, r, self._c(cfg))
        out[: len(b)] = torch.frombuffer(bytearray(b), dtype=torch.uint8)
        length[0] = len(b)

    # the sharded decode (shard_scan): range scans, then the selection from the
    # assembled positive list — checked against the full scan here
    def bloom_scan_range_into(self, filt, d, lo, hi, out, count, stream=None):
        pos = oracle().positive_scan(filt.contiguous().numpy().tobytes(), d)
        sl = pos[(pos >= lo) & (pos < hi)]
        out[: sl.size] = torch.from_numpy(sl.astype(np.int32))
        count[0] = sl.size

    def decode_index_from_positions(self, filt, d, r, index_method, positions, count, stream=None):
        got = positions[: int(count.item())].numpy().astype(np.uint32)
        want = oracle().positive_scan(filt.contiguous().numpy().tobytes(), d)
        assert np.array_equal(got, want), "assembled positive list differs from the full scan"

    def set_decode_overwrite(self, on):
        self._overwrite = bool(on)

    def decode_accumulate_own(self, container, dense, length, hint, scale=1.0, stream=None):
        self.decode_accumulate(container, dense, scale=scale, length=length, overwrite=getattr(self, "_overwrite", False))

    def status(self, stream=None):
        pass  # the oracle raises at the call that fails

    def decode_accumulate(self, container, dense, scale=1.0, length=None, hint=None, stream=None, overwrite=False):
        if overwrite:
            dense.zero_()
        n = int(length.item()) if isinstance(length, torch.Tensor) else (container.numel() if length is None else length)
        _, sup, val = oracle().decode(container[:n].contiguous().numpy().tobytes())
        idx = torch.from_numpy(sup.astype(np.int64))
        # same arithmetic as the device scatter: fmaf(scale, (float)v, dense)
        dense[idx] = (np.float32(scale) * torch.from_numpy(val.astype(np.float32)) + dense[idx]).to(torch.float32)


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


CFGS = {
    "p2fit": dict(index_method=IndexMethod.BloomP2, value_method=ValueMethod.FitPoly, fpr=0.01),
    "bitmap": dict(index_method=IndexMethod.Bitmap, value_method=ValueMethod.None_),
    "rle": dict(index_method=IndexMethod.Rle, value_method=ValueMethod.None_),
}


def _worker(rank, world, port, name, d, r, steps, buckets, q, ef=False):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    from paper_2102_03112_b200.dp import BucketedSparseAllgather, SparseAllgather
    cfg = PipelineConfig(**CFGS[name])
    g = torch.from_numpy(synthetic_gradient(d, rank=rank))
    outs = []
    if buckets:
        ex = BucketedSparseAllgather(lambda dmax: OracleCodec(), d, r / d, cfg, buckets, streams=2,
                                     device="cpu", ef=ef)
    else:
        ex = SparseAllgather(OracleCodec(), d, r, cfg, device="cpu", ef=ef)
    for step in range(steps):
        outs.append(ex.step(g, step=step).clone().numpy())
    q.put((rank, outs))
    dist.destroy_process_group()


def _sequential(name, d, r, steps, world, buckets, ef=False):
    """Simulation::step's worker loop, one process: encode every worker, decode, mean
    (with compensation: input = g + residual, residual = input - decoded)."""
    from paper_2102_03112_b200.dp import hash64, pipeline_seed, ratio_r
    o = oracle()
    base = PipelineConfig(**CFGS[name])
    means = []
    if ef == "f64":  # the reference's own f64 loop (harness.cpp:230-271) through oracle/_ref
        from oracle.bindings import reference
        ref = reference()
        resid64 = [np.zeros(d, np.float64) for _ in range(world)]
        for step in range(steps):
            acc = np.zeros(d, np.float32)
            for w in range(world):
                g = synthetic_gradient(d, rank=w)
                c = ref.ef_step64(g, resid64[w], r, OracleCodec._c(PipelineConfig(
                    **{**base.__dict__, "seed": pipeline_seed(1, w, step)})))
                _, sup, val = o.decode(c)
                acc[sup] = np.float32(1.0 / world) * val.astype(np.float32) + acc[sup]
            means.append(acc)
        return means
    resid = [np.zeros(d, np.float32) for _ in range(world)]
    for step in range(steps):
        acc = np.zeros(d, np.float32)
        for w in range(world):  # rank order
            g = synthetic_gradient(d, rank=w)
            if ef:
                g = (g + resid[w]).astype(np.float32)
            parts = [(0, d, r, pipeline_seed(1, w, step))]
            if buckets:
                lo, parts = 0, []
                q, rem = divmod(d, buckets)
                for b in range(buckets):
                    n = q + (1 if b < rem else 0)
                    parts.append((lo, lo + n, ratio_r(n, r / d), hash64(b, pipeline_seed(1, w, step))))
                    lo += n
            for lo, hi, rb, seed in parts:
                c = o.encode_dense(g[lo:hi], rb, OracleCodec._c(PipelineConfig(**{**base.__dict__, "seed": seed})))
                _, sup, val = o.decode(c)
                if ef:
                    res = g[lo:hi].copy()
                    res[sup] = (g[lo:hi][sup] - val.astype(np.float32)).astype(np.float32)
                    resid[w][lo:hi] = res
                a = acc[lo:hi]
                a[sup] = np.float32(1.0 / world) * val.astype(np.float32) + a[sup]
        means.append(acc)
    return means


@pytest.mark.parametrize("name,d,r,buckets,ef", [("p2fit", 20_000, 200, 0, False), ("bitmap", 5_000, 50, 0, False),
                                                 ("rle", 7_000, 70, 0, False), ("p2fit", 40_000, 40, 4, False),
                                                 ("p2fit", 20_000, 200, 0, "f32"), ("bitmap", 40_000, 40, 4, "f32"),
                                                 ("p2fit", 20_000, 200, 0, "f64"), ("rle", 20_000, 200, 0, True)])
def test_gloo_world2_matches_sequential_harness(name, d, r, buckets, ef):
    if ef in ("f64", True):
        from oracle.bindings import reference
        if reference() is None:
            pytest.skip("oracle/_ref not built")
        ef = "f64"
    world, steps = 2, 3 if ef else 2
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(k, world, port, name, d, r, steps, buckets, q, ef))
             for k in range(world)]
    for p in procs:
        p.start()
    res = dict(q.get(timeout=300) for _ in range(world))
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    want = _sequential(name, d, r, steps, world, buckets, ef)
    for step in range(steps):
        assert np.array_equal(res[0][step], res[1][step]), "replicas diverged"
        assert np.array_equal(res[0][step], want[step])
