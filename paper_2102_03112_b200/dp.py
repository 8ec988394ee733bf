"""Data-parallel sparse-gradient exchange: encode → allgather → decode.

The real-process form of the reference's simulated worker loop
(Simulation::step, harness.cpp:219-293): every rank is one worker with its
own full d-element gradient; it runs top_r + compress_gradient + pack
(pipeline seed = Simulation::pipeline_seed(seed, rank, step),
harness.cpp:201-203); the variable-length containers are exchanged with an
allgather — sizes first, then the payloads padded to the largest size (NCCL
has no allgatherv) — and every rank decodes all N containers in rank order
into the dense mean.  The reference sums the N decoded f64 vectors in a
fixed pairwise tree and then divides by N (harness.cpp:274-284); this path
accumulates in f32, sequentially in rank order, dense = fmaf(1/N, v, dense)
— per coordinate at most N f32 roundings, i.e. within N ulp(f32) of the
largest term of the reference's f64 mean (tests/test_gpu_parity.py bounds it
at 4 ulp for the single-worker case).

torch.distributed is plumbing only (process group, NCCL communicator); every
payload byte is produced and consumed by the codec.  The codec is duck-typed
(encode_into / decode_accumulate / max_container_bytes) so the same exchange
runs on CUDA tensors with NCCL and on CPU tensors with gloo, where the tests
plug in a CPU stand-in codec (tests/test_dp_gloo.py).

BucketedSparseAllgather splits very large gradients (BERT-large, 340M) into
independent per-bucket containers — a convention of this framework with no
reference equivalent: bucket b of a rank's step uses seed
hash64(b, pipeline_seed(seed, rank, step)) and r_b = max(1, llround(ratio*d_b)).
Buckets are spread over several codec contexts on their own CUDA streams, so
encode, exchange and decode of different buckets overlap.
"""
from __future__ import annotations

from dataclasses import replace

import torch
import torch.distributed as dist

from .seeds import bucket_bounds, hash64, pipeline_seed, ratio_r  # noqa: F401  (re-exported)


def _world(group):
    if dist.is_available() and dist.is_initialized():
        return dist.get_world_size(group), dist.get_rank(group)
    return 1, 0


def _ef_mode(ef) -> str | None:
    """ef: False/None (off), "f64" or True (the reference's precision: the
    residual is a VectorXd, gradient.hpp:29), "f32" (an f32 residual)."""
    if ef is True:
        return "f64"
    if not ef:
        return None
    if ef not in ("f32", "f64"):
        raise ValueError(f"ef must be False, True, 'f32' or 'f64', not {ef!r}")
    return ef


class SparseAllgather:
    """One DP worker's encode → exchange → decode step.  ef adds the
    reference's memory compensation (TrainConfig::compensation,
    harness.cpp:230, :269-271): the rank encodes g + residual and keeps
    input - decode(own container) as the next step's residual — in f64 as the
    reference does (ef=True / "f64"), or in f32 (ef="f32")."""

    def __init__(self, codec, d: int, r: int, cfg, group=None, device=None, ef: bool = False,
                 graph: bool = False, decode_codecs=None, early_codec=None, shard_scan: bool | None = None):
        self.codec = codec
        self.d, self.r, self.cfg = d, r, cfg
        self.group = group
        self.world, self.rank = _world(group)
        dev = device if device is not None else torch.device("cuda", torch.cuda.current_device())
        self.cap = type(codec).max_container_bytes(d, r, cfg)
        self.out = torch.empty(self.cap, dtype=torch.uint8, device=dev)
        self.length = torch.zeros(1, dtype=torch.int64, device=dev)
        self.sizes = torch.zeros(self.world, dtype=torch.int64, device=dev)
        self.recv = torch.empty(self.world * self.cap, dtype=torch.uint8, device=dev) if self.world > 1 else None
        self.dense = torch.zeros(d, dtype=torch.float32, device=dev)
        self.ef = _ef_mode(ef)
        self.residual = (torch.zeros(d, dtype=torch.float64 if self.ef == "f64" else torch.float32, device=dev)
                         if self.ef else None)
        # decode_codecs (N > 1, CUDA): extra contexts that decode peers concurrently,
        # each on its own stream, up to the final scatter; the scatters then run
        # in rank order on the step's stream (gp_decode_prepare / gp_decode_finish),
        # so the accumulation order — and the result — is the sequential one.
        self.dec = [codec] + list(decode_codecs or [])
        # early_codec (N = 1, Bloom P0/P1/P2/Pd, CUDA): the own container's index
        # stage (positive scan + selection) runs on this second context and stream
        # as soon as the encode has built the filter, overlapping the rest of the
        # encode; the decode then finishes with that prepared index stage.
        im = int(cfg.index_method)
        self.early = (early_codec if early_codec is not None and self.world == 1 and 4 <= im <= 7
                      and torch.device(dev).type == "cuda" else None)
        if self.early is not None:
            from .api import bloom_params
            m, _ = bloom_params(cfg.fpr, r)
            self.filter_len = 26 + (m + 7) // 8 + (1 if im == 7 else 0)
            self.early_stream = torch.cuda.Stream(dev)
            self.ev_index = torch.cuda.Event()
            self.ev_index.record()  # materialise the CUDA event handle
            self.ev_early = torch.cuda.Event()
        # shard_scan (N > 1, Bloom P0/P1/P2/Pd): the positive scans of the N
        # received filters are split by coordinate range — rank i scans every
        # filter over [i d / N, (i + 1) d / N) and the slices are allgathered —
        # so a rank scans d keys per step instead of N d; each container's
        # selection then runs from its assembled positive list.
        bloom_sel = 4 <= im <= 7
        self.shard = bool(self.world > 1 and bloom_sel and (shard_scan if shard_scan is not None else True))
        if self.shard:
            from .api import bloom_params
            m, _ = bloom_params(cfg.fpr, r)
            self.filter_len = 26 + (m + 7) // 8 + (1 if im == 7 else 0)
            n = self.world
            self.lo, self.hi = self.rank * d // n, (self.rank + 1) * d // n
            self.slice_cap = max(1, max((k + 1) * d // n - k * d // n for k in range(n)))
            self.pslice = torch.empty((n, self.slice_cap), dtype=torch.int32, device=dev)
            self.pcount = torch.zeros(n, dtype=torch.int64, device=dev)
            self.pcount_all = torch.zeros(n * n, dtype=torch.int64, device=dev)
            self.precv = None
            self.pfull = torch.empty(d, dtype=torch.int32, device=dev)
            self.pfull_n = torch.zeros(1, dtype=torch.int64, device=dev)
        self.dec_streams = ([torch.cuda.Stream(dev) for _ in self.dec]
                            if len(self.dec) > 1 and torch.device(dev).type == "cuda" else None)
        # graph=True (one rank, CUDA): the whole step — pipeline seed from a device
        # step counter, encode, zero, decode — is captured once per (input,
        # output, base seed) and replayed; the step number is the only host input
        # (one fill of the counter before each replay).
        self.graph = bool(graph) and self.world == 1 and torch.device(dev).type == "cuda"
        self.graphs = {}
        self.kernels_per_step = None
        if self.graph:
            self.step_dev = torch.zeros(1, dtype=torch.int64, device=dev)
            self.seed_dev = torch.zeros(1, dtype=torch.int64, device=dev)

    def _captured(self, grad, out_dense, seed):
        from .api import pipeline_seed_device
        key = (grad.data_ptr(), out_dense.data_ptr(), seed)
        g = self.graphs.get(key)
        if g is None:
            if len(self.graphs) >= 8:  # callers should reuse buffers; bound the cache anyway
                self.graphs.pop(next(iter(self.graphs)))
            torch.cuda.synchronize()
            self.codec.set_seed_source(self.seed_dev)
            try:
                # one warm step outside the capture (one-time kernel attributes, tables);
                # the error-feedback residual is restored so the warm step leaves no trace
                keep = self.residual.clone() if self.residual is not None else None
                self.step_seeded(grad, self.cfg, dense=out_dense)
                if keep is not None:
                    self.residual.copy_(keep)
                torch.cuda.synchronize()
                users = [self.codec] + ([self.early] if self.early is not None else [])
                n0 = sum(c.launches for c in users)
                g = torch.cuda.CUDAGraph()
                with torch.cuda.graph(g):
                    s = torch.cuda.current_stream()
                    pipeline_seed_device(self.seed_dev, self.step_dev, seed, self.rank, stream=s)
                    self.step_seeded(grad, self.cfg, dense=out_dense, stream=s)
                self.kernels_per_step = sum(c.launches for c in users) - n0 + 1
            finally:
                self.codec.set_seed_source(None)
            self.graphs[key] = g
        return g

    def step(self, grad: torch.Tensor, step: int, seed: int = 1, dense: torch.Tensor | None = None,
             stream=None) -> torch.Tensor:
        """Dense mean of every rank's decoded container (accumulated into `dense`
        or the exchanger's own buffer)."""
        if self.graph and stream is None:
            out_dense = self.dense if dense is None else dense
            g = self._captured(grad, out_dense, seed)
            self.step_dev.fill_(step)
            g.replay()
            return out_dense
        cfg = replace(self.cfg, seed=pipeline_seed(seed, self.rank, step))
        return self.step_seeded(grad, cfg, dense=dense, stream=stream)

    def step_seeded(self, grad, cfg, dense=None, stream=None):
        out_dense = self.dense if dense is None else dense
        if self.early is not None:
            return self._step_early(grad, cfg, out_dense, stream)
        self._encode(grad, cfg, stream)
        n = self.world
        # the first container of the mean overwrites the output (zero + accumulate in one pass)
        if n == 1:  # no exchange: the device-side length drives the decode (no host sync)
            self.codec.decode_accumulate(self.out, out_dense, scale=1.0, length=self.length, hint=self.cfg,
                                         stream=stream, overwrite=True)
            return out_dense
        # the step's one host sync: a latched encode error (or a previous step's
        # decode error) raises here instead of shipping a stale container
        self.codec.status(stream)
        dist.all_gather_into_tensor(self.sizes, self.length, group=self.group)
        sizes = self.sizes.tolist()
        mx = max(sizes)
        dist.all_gather_into_tensor(self.recv[: n * mx], self.out[:mx], group=self.group)
        if self.shard:
            self._decode_sharded(n, mx, sizes, out_dense, stream)
            return out_dense
        if self.dec_streams is None:
            for j in range(n):  # fixed rank order, as the harness's worker order
                self.codec.decode_accumulate(self.recv[j * mx: j * mx + sizes[j]], out_dense, scale=1.0 / n,
                                             hint=self.cfg, stream=stream, overwrite=(j == 0))
            return out_dense
        main = stream if stream is not None else torch.cuda.current_stream()
        self._decode_concurrent(n, mx, out_dense, main)
        return out_dense

    def _encode(self, grad, cfg, stream):
        if self.ef == "f64":
            self.codec.encode_ef64_into(grad, self.residual, self.r, cfg, self.out, self.length, stream=stream)
        elif self.ef == "f32":
            self.codec.encode_ef_into(grad, self.residual, self.r, cfg, self.out, self.length, stream=stream)
        else:
            self.codec.encode_into(grad, self.r, cfg, self.out, self.length, stream=stream)

    def _decode_sharded(self, n, mx, sizes, out_dense, stream):
        """The decode of all N containers with the Bloom positive scans split by
        coordinate range across the ranks (shard_scan)."""
        if stream is not None:  # the buffer copies below must order with the codec calls
            with torch.cuda.stream(stream):
                return self._decode_sharded(n, mx, sizes, out_dense, None)
        fl = self.filter_len
        for j in range(n):  # this rank's slice of every container's positive set
            filt = self.recv[j * mx + 49: j * mx + 49 + fl]
            self.codec.bloom_scan_range_into(filt, self.d, self.lo, self.hi, self.pslice[j], self.pcount[j:j + 1],
                                             stream=stream)
        dist.all_gather_into_tensor(self.pcount_all, self.pcount, group=self.group)
        cnt = self.pcount_all.tolist()  # cnt[i * n + j]: rank i's slice of container j (second host sync)
        mxp = max(1, max(cnt))
        if self.precv is None or self.precv.numel() < n * n * mxp:
            self.precv = torch.empty(n * n * mxp, dtype=torch.int32, device=self.pslice.device)
        send = self.pslice[:, :mxp].contiguous().view(-1)
        dist.all_gather_into_tensor(self.precv[: n * n * mxp], send, group=self.group)
        parts = self.precv[: n * n * mxp].view(n, n, mxp)  # [rank i][container j][:]
        for j in range(n):  # rank order (harness.cpp:274-284)
            total = 0
            for i in range(n):  # slices in coordinate order: the ascending positive set
                c = cnt[i * n + j]
                if c:
                    self.pfull[total: total + c].copy_(parts[i, j, :c])
                total += c
            self.pfull_n.fill_(total)
            filt = self.recv[j * mx + 49: j * mx + 49 + fl]
            self.codec.decode_index_from_positions(filt, self.d, self.r, int(self.cfg.index_method), self.pfull,
                                                   self.pfull_n, stream=stream)
            self.codec.set_decode_overwrite(j == 0)
            try:
                self.codec.decode_accumulate_own(self.recv[j * mx: (j + 1) * mx], out_dense,
                                                 self.sizes[j:j + 1], self.cfg, scale=1.0 / n, stream=stream)
            finally:
                self.codec.set_decode_overwrite(False)

    def check(self, stream=None) -> None:
        """Synchronise and raise the first device error latched by any of this
        exchanger's contexts (checksum / payload / capacity errors of a decode,
        fit errors of an encode).  The status latch is sticky until read and
        every kernel of a latched context returns early, so callers of the
        host-sync-free paths (N = 1, CUDA graphs) poll this once per step, or
        as often as they can afford; N > 1 steps poll the encoding context at
        their sizes exchange."""
        seen = []
        for c in [self.codec] + list(self.dec[1:]) + ([self.early] if self.early is not None else []):
            if all(c is not x for x in seen):
                seen.append(c)
                c.status(stream)

    def _step_early(self, grad, cfg, out_dense, stream):
        main = stream if stream is not None else torch.cuda.current_stream()
        self.codec.set_index_event(self.ev_index)
        try:
            self._encode(grad, cfg, main)
        finally:
            self.codec.set_index_event(None)
        side = self.early_stream
        side.wait_event(self.ev_index)
        self.early.decode_index_prepare(self.out[49:49 + self.filter_len], self.d, self.r,
                                        int(self.cfg.index_method), stream=side)
        self.ev_early.record(side)
        out_dense.zero_()
        main.wait_event(self.ev_early)
        self.early.decode_accumulate_own(self.out, out_dense, self.length, self.cfg, scale=1.0, stream=main)
        return out_dense

    def _decode_concurrent(self, n, mx, out_dense, main):
        D = len(self.dec)
        gathered = torch.cuda.Event()
        gathered.record(main)
        finished = [None] * n
        for k in range(min(D, n)):
            self.dec_streams[k].wait_event(gathered)
        for j in range(n):
            k = j % D
            st = self.dec_streams[k]
            if j >= D:  # the context is free once its previous container's scatter ran
                st.wait_event(finished[j - D])
            part = self.recv[j * mx: (j + 1) * mx]
            self.dec[k].decode_prepare(part, self.sizes[j:j + 1], self.cfg, stream=st)
            ready = torch.cuda.Event()
            ready.record(st)
            main.wait_event(ready)
            self.dec[k].decode_finish(part, out_dense, 1.0 / n, stream=main, overwrite=(j == 0))  # rank order
            finished[j] = torch.cuda.Event()
            finished[j].record(main)


class BucketedSparseAllgather:
    """Bucketed DP step for gradients too large for one container (C5)."""

    def __init__(self, codec_factory, d: int, ratio: float, cfg, buckets: int, streams: int = 3, group=None,
                 device=None, ef: bool = False, graph: bool = False):
        self.d, self.cfg, self.buckets = d, cfg, buckets
        self.world, self.rank = _world(group)
        self.bounds = bucket_bounds(d, buckets)
        dmax = max(e - s for s, e in self.bounds)
        self.rs = [ratio_r(e - s, ratio) for s, e in self.bounds]
        self.nstreams = min(streams, buckets)
        self.codecs = [codec_factory(dmax) for _ in range(self.nstreams)]
        cuda = device is None or torch.device(device).type == "cuda"
        self.streams = [torch.cuda.Stream() for _ in range(self.nstreams)] if cuda else [None] * self.nstreams
        self.ex = [SparseAllgather(self.codecs[i % self.nstreams], e - s, self.rs[i], cfg, group=group,
                                   device=device, ef=ef) for i, (s, e) in enumerate(self.bounds)]
        dev = device if device is not None else torch.device("cuda", torch.cuda.current_device())
        self.dense = torch.zeros(d, dtype=torch.float32, device=dev)
        # graph=True (one rank): the whole multi-stream step is one CUDA graph;
        # per-bucket seeds come from the device (gp_pipeline_seed_device)
        self.graph = bool(graph) and self.world == 1 and cuda
        self.graphs = {}
        self.kernels_per_step = None
        if self.graph:
            self.step_dev = torch.zeros(1, dtype=torch.int64, device=dev)
            self.seeds_dev = torch.zeros(buckets, dtype=torch.int64, device=dev)

    def check(self) -> None:
        """Raise the first latched device error of any bucket context (see SparseAllgather.check)."""
        for c in self.codecs:
            c.status()

    def bucket_seed(self, seed: int, step: int, b: int) -> int:
        return hash64(b, pipeline_seed(seed, self.rank, step))

    def _captured(self, grad, out_dense, seed):
        from .api import pipeline_seed_device
        key = (grad.data_ptr(), out_dense.data_ptr(), seed)
        g = self.graphs.get(key)
        if g is not None:
            return g
        if len(self.graphs) >= 8:
            self.graphs.pop(next(iter(self.graphs)))
        torch.cuda.synchronize()
        keep = [e.residual.clone() if e.residual is not None else None for e in self.ex]
        self._run(grad, out_dense, lambda b: self.cfg)  # warm outside the capture
        for e, k in zip(self.ex, keep):
            if k is not None:
                e.residual.copy_(k)
        torch.cuda.synchronize()
        n0 = sum(c.launches for c in self.codecs)
        g = torch.cuda.CUDAGraph()
        try:
            with torch.cuda.graph(g):
                pipeline_seed_device(self.seeds_dev, self.step_dev, seed, self.rank, buckets=self.buckets)

                def seeded(b):  # the captured init_plan of bucket b reads seeds_dev[b]
                    self.ex[b].codec.set_seed_source(self.seeds_dev[b:b + 1])
                    return self.cfg
                self._run(grad, out_dense, seeded)
        finally:
            for c in self.codecs:
                c.set_seed_source(None)
        self.kernels_per_step = sum(c.launches for c in self.codecs) - n0 + 1
        self.graphs[key] = g
        return g

    def step(self, grad: torch.Tensor, step: int, seed: int = 1, dense: torch.Tensor | None = None) -> torch.Tensor:
        out_dense = self.dense if dense is None else dense
        if self.graph:
            g = self._captured(grad, out_dense, seed)
            self.step_dev.fill_(step)
            g.replay()
            return out_dense
        return self._run(grad, out_dense, lambda b: replace(self.cfg, seed=self.bucket_seed(seed, step, b)))

    def _run(self, grad, out_dense, cfg_of):
        cur = torch.cuda.current_stream() if self.streams[0] is not None else None
        if cur is not None:
            for s in self.streams:
                s.wait_stream(cur)
        for b, (lo, hi) in enumerate(self.bounds):
            si = b % self.nstreams
            s = self.streams[si]
            if s is not None:
                with torch.cuda.stream(s):
                    self.ex[b].step_seeded(grad[lo:hi], cfg_of(b), dense=out_dense[lo:hi], stream=s)
            else:
                self.ex[b].step_seeded(grad[lo:hi], cfg_of(b), dense=out_dense[lo:hi])
        if cur is not None:
            for s in self.streams:
                cur.wait_stream(s)
        return out_dense


class HostPipeline:
    """DP steps on HOST buffers with the copies overlapped across steps.

    The harness's step (harness.cpp:219-293) takes host gradients and produces
    the host dense mean.  Here step i's gradient is copied in on its own stream
    while step i-1 computes, and step i-1's mean is copied out on a third stream
    while step i computes (PCIe is full duplex), through double-buffered device
    input/output.  submit() only enqueues; drain() waits for the last copy-out.
    The caller must not overwrite a host output buffer before its step drained
    (alternate at least two)."""

    def __init__(self, ex, d: int, device=None):
        dev = device if device is not None else torch.device("cuda", torch.cuda.current_device())
        self.ex = ex
        self.gin = [torch.empty(d, dtype=torch.float32, device=dev) for _ in range(2)]
        self.dout = [torch.zeros(d, dtype=torch.float32, device=dev) for _ in range(2)]
        self.s_in = torch.cuda.Stream(dev)
        self.s_out = torch.cuda.Stream(dev)
        self.in_ready = [torch.cuda.Event() for _ in range(2)]
        self.in_free = [torch.cuda.Event() for _ in range(2)]
        self.out_ready = [torch.cuda.Event() for _ in range(2)]
        self.out_free = [torch.cuda.Event() for _ in range(2)]
        self.used = [False, False]
        self.i = 0

    def submit(self, host_in: torch.Tensor, host_out: torch.Tensor, step: int, seed: int = 1,
               between=None) -> None:
        b = self.i & 1
        compute = torch.cuda.current_stream()
        if self.used[b]:
            self.s_in.wait_event(self.in_free[b])    # step i-2 finished reading gin[b]
            compute.wait_event(self.out_free[b])     # step i-2's copy-out of dout[b] finished
        with torch.cuda.stream(self.s_in):
            self.gin[b].copy_(host_in, non_blocking=True)
            self.in_ready[b].record(self.s_in)
        if between is not None:
            between()                                # e.g. the benchmark's L2 flush, on the compute stream
        compute.wait_event(self.in_ready[b])
        self.ex.step(self.gin[b], step=step, seed=seed, dense=self.dout[b])
        self.in_free[b].record(compute)
        self.out_ready[b].record(compute)
        self.s_out.wait_event(self.out_ready[b])
        with torch.cuda.stream(self.s_out):
            host_out.copy_(self.dout[b], non_blocking=True)
            self.out_free[b].record(self.s_out)
        self.used[b] = True
        self.i += 1

    def drain(self) -> None:
        self.s_out.synchronize()
