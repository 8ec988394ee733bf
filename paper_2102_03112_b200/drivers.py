"""Reporting drivers of the reference CLI on the device path
(tools/gradpack_main.cpp).

  python -m paper_2102_03112_b200.drivers sweep [--dim D] [--topr R] [--seeds S] [--seed X]
  python -m paper_2102_03112_b200.drivers bench [--dim D] [--topr R] [--reps K] [--fpr E] [--seed X]

sweep : cmd_sweep (gradpack_main.cpp:216-267) — for every sparsifier (top-r,
        random-r), Bloom policy (P0/P1/P2) and FPR of the paper's grid, the
        mean relative volume (volume().ratio_dense, container.cpp:148-243) and
        reconstruction error ||decoded - target|| / ||target|| against the
        sparse gradient at wire precision, over `seeds` draws.  Same CSV.
bench : cmd_bench (gradpack_main.cpp:269-353) — per method row: total bits and
        the median encode / decode time, measured on the device with CUDA
        events (the reference times its CPU calls with steady_clock).  The
        deflate-slot row runs with the Store codec (the Deflate codec is not on
        the device path; a row the device cannot run is reported "unsupported").  The
        rle-clustered row gathers its values from g at the clustered support
        (the CLI reuses the uniform row's values); with raw f32 values the
        container size and work are the same.

Data follow the CLI exactly: g_j = CounterRng(seed_s).normal() in f64
(rng.hpp:65-69, one normal per element), stored as f32 for the device path —
the values travel as f32 on the wire either way.  compress_gradient is
called without a dense vector (values off the support are 0, pipeline.cpp:38-54):
the device gathers from to_dense(sg).
"""
from __future__ import annotations

import argparse
import math
import sys

import numpy as np
import torch

from .api import Codec, PipelineConfig, UnsupportedMethodError, volume
from .inputs import normal_f32
from .seeds import GAMMA, MASK, hash64, mix64, ratio_r

GRID = (0.2, 0.1, 0.05, 0.02, 0.01, 0.005, 0.002, 0.001)
POLICIES = ((4, "p0"), (5, "p1"), (6, "p2"))


def below_seq(seed: int, bounds, start: int = 0) -> list[int]:
    """CounterRng(seed).below(n) for successive n (rng.hpp:52-59), rejection exact,
    from draw position `start` of the stream."""
    out, pos = [], start
    for n in bounds:
        rem = ((2 ** 64 - 1) % n + 1) % n
        bound = 2 ** 64 - 1 - rem
        while True:
            v = mix64((seed + (pos + 1) * GAMMA) & MASK)
            pos += 1
            if v <= bound:
                break
        out.append(v % n)
    return out


def random_r(d: int, r: int, seed: int) -> np.ndarray:
    """random_r (sparsify.cpp:48-58): Floyd's sampling with CounterRng(seed).below, sorted."""
    chosen: set[int] = set()
    draws = below_seq(seed, [j + 1 for j in range(d - r, d)])
    for j, t in zip(range(d - r, d), draws):
        chosen.add(j if t in chosen else t)
    return np.array(sorted(chosen), dtype=np.uint32)


def _encode_decode(codec: Codec, dense_f32: torch.Tensor, support: torch.Tensor, cfg: PipelineConfig):
    c = codec.compress(dense_f32, support.numel(), cfg, support=support)
    d, sup, val = codec.decompress(c)
    return c, sup, val


def sweep(dim: int = 100_000, top_ratio: float = 0.01, seeds: int = 3, seed: int = 1, codec: Codec | None = None,
          grid=GRID, policies=POLICIES, sparsifiers=("topr", "randomr")) -> str:
    own = codec is None
    codec = codec or Codec(max_d=dim)
    r = ratio_r(dim, top_ratio)
    csv = ["sparsifier,policy,fpr,relative_volume,reconstruction_error"]
    data = {}
    for sp in sparsifiers:
        for s in range(seeds):  # the data draw depends only on (sparsifier, s)
            g = normal_f32(hash64(s, hash64(0x5EED, seed)), dim)
            if sp == "topr":
                sup, _ = codec.top_r(torch.from_numpy(g).cuda(), r)
                sup = sup.cpu().numpy().astype(np.uint32)
            else:
                sup = random_r(dim, r, hash64(s, hash64(0x9AA9, seed)))
            target = np.zeros(dim, np.float32)
            target[sup] = g[sup]
            data[sp, s] = (sup, target)
    for sp in sparsifiers:
        for im, pname in policies:
            for eps in grid:
                vol, err = 0.0, 0.0
                for s in range(seeds):
                    sup, target = data[sp, s]
                    cfg = PipelineConfig(index_method=im, value_method=0, fpr=eps,
                                         seed=hash64(s, hash64(0xC4A0, seed)))
                    c, dsup, dval = _encode_decode(codec, torch.from_numpy(target).cuda(),
                                                   torch.from_numpy(sup.astype(np.int32)).cuda(), cfg)
                    vol += volume(c.cpu().numpy().tobytes())["ratio_dense"]
                    dec = np.zeros(dim, np.float64)
                    dec[dsup.cpu().numpy().astype(np.int64)] = dval.cpu().numpy()
                    t64 = target.astype(np.float64)
                    err += float(np.linalg.norm(dec - t64) / np.linalg.norm(t64))
                csv.append(f"{sp},{pname},{eps!r},{vol / seeds!r},{err / seeds!r}")
    if own:
        codec.close()
    return "\n".join(csv) + "\n"


BENCH_ROWS = [("identity", 0, 5, False), ("bitmap", 1, 0, False), ("rle", 2, 0, False), ("rle-clustered", 2, 0, True),
              ("huffman", 3, 0, False), ("bloom-p0", 4, 0, False), ("bloom-p1", 5, 0, False),
              ("bloom-p2", 6, 0, False), ("bloom-pd", 7, 0, False), ("fit-poly", 1, 1, False),
              ("fit-dexp", 1, 2, False), ("quant", 1, 3, False), ("deflate-slot", 1, 4, False)]


def method_bench(dim: int = 1_000_000, top_ratio: float = 0.01, reps: int = 10, fpr: float = 0.01, seed: int = 1,
                 codec: Codec | None = None) -> str:
    own = codec is None
    codec = codec or Codec(max_d=dim)
    g = normal_f32(hash64(0xBE7C, seed), dim)  # the CLI draws g from CounterRng(hash64(0xBE7C, seed))
    gt = torch.from_numpy(g).cuda()
    r = ratio_r(dim, top_ratio)
    sup, _ = codec.top_r(gt, r)
    # the same stream continues after the dim normals (two draws each): gradpack_main.cpp:285-287
    start = below_seq(hash64(0xBE7C, seed), [dim - r + 1], start=2 * dim)[0]
    clustered = torch.arange(start, start + r, dtype=torch.int32, device="cuda")
    csv = ["method,bits_total,t_encode_ns,t_decode_ns"]
    for name, im, vm, clus in BENCH_ROWS:
        cfg = PipelineConfig(index_method=im, value_method=vm, fpr=fpr, seed=hash64(0xB0B, seed),
                             slot_codec=0 if vm == 4 else 1)
        s = clustered if clus else sup
        try:
            enc, dec = [], []
            out = torch.empty(Codec.max_container_bytes(dim, r, cfg), dtype=torch.uint8, device="cuda")
            length = torch.zeros(1, dtype=torch.int64, device="cuda")
            dense = torch.zeros(dim, dtype=torch.float32, device="cuda")
            for it in range(reps + 2):  # two warmup repetitions are dropped
                e0, e1, e2 = (torch.cuda.Event(enable_timing=True) for _ in range(3))
                e0.record()
                codec.encode_into(gt, r, cfg, out, length, support=s)
                e1.record()
                codec.decode_accumulate(out, dense, length=length, hint=cfg)
                e2.record()
                e2.synchronize()
                codec.status()
                if it >= 2:
                    enc.append(e0.elapsed_time(e1) * 1e6)
                    dec.append(e1.elapsed_time(e2) * 1e6)
            n = int(length.item())
            bits = volume(out[:n].cpu().numpy().tobytes())["total_bits"]
            csv.append(f"{name},{bits},{int(np.median(enc))},{int(np.median(dec))}")
        except UnsupportedMethodError:
            csv.append(f"{name},unsupported,,")
    if own:
        codec.close()
    return "\n".join(csv) + "\n"


def main(argv=None) -> int:
    ap = argparse.ArgumentParser(prog="python -m paper_2102_03112_b200.drivers")
    sub = ap.add_subparsers(dest="cmd", required=True)
    sw = sub.add_parser("sweep")
    sw.add_argument("--dim", type=int, default=100_000)
    sw.add_argument("--topr", type=float, default=0.01)
    sw.add_argument("--seeds", type=int, default=3)
    sw.add_argument("--seed", type=int, default=1)
    be = sub.add_parser("bench")
    be.add_argument("--dim", type=int, default=1_000_000)
    be.add_argument("--topr", type=float, default=0.01)
    be.add_argument("--reps", type=int, default=10)
    be.add_argument("--fpr", type=float, default=0.01)
    be.add_argument("--seed", type=int, default=1)
    a = ap.parse_args(argv)
    if a.cmd == "sweep":
        sys.stdout.write(sweep(a.dim, a.topr, a.seeds, a.seed))
    else:
        sys.stdout.write(method_bench(a.dim, a.topr, a.reps, a.fpr, a.seed))
    return 0


if __name__ == "__main__":
    raise SystemExit(main())
