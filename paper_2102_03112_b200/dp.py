"""Data-parallel sparse-gradient exchange: encode → allgather → decode.

The real-process form of the reference's simulated worker loop
(Simulation::step, harness.cpp:219-293): every rank is one worker with its
own full d-element gradient; it runs top_r + compress_gradient + pack on its
device (pipeline seed = Simulation::pipeline_seed(seed, rank, step),
harness.cpp:201-203), the variable-length containers are exchanged with an
NCCL allgather — sizes first, then the payloads padded to the largest size
(NCCL has no allgatherv) — and every rank decodes all N containers in rank
order into the dense mean (harness.cpp:274-284, f32 accumulate of x/N).

torch.distributed is plumbing only (process group, NCCL communicator); the
payload bytes are produced and consumed by libgradpack_b200.so.  The same
code runs on CPU tensors with the gloo backend (tests/test_dp_gloo.py), where
a host-side codec stands in for the device codec.
"""
from __future__ import annotations

import torch
import torch.distributed as dist

from .api import Codec, PipelineConfig

GAMMA = 0x9E3779B97F4A7C15
MASK = (1 << 64) - 1


def _mix64(z: int) -> int:
    z &= MASK
    z ^= z >> 30
    z = (z * 0xBF58476D1CE4E5B9) & MASK
    z ^= z >> 27
    z = (z * 0x94D049BB133111EB) & MASK
    return z ^ (z >> 31)


def hash64(x: int, seed: int) -> int:
    """rng.hpp:35-37"""
    return _mix64((x ^ ((seed + GAMMA) & MASK)) & MASK)


def pipeline_seed(seed: int, worker: int, step: int) -> int:
    """Simulation::pipeline_seed (harness.cpp:201-203) over Problem::batch_seed (:47-51)."""
    key = ((worker & 0xFFFFFFFF) << 32) | (step & 0xFFFFFFFF)
    return hash64(0xC0DEC, hash64(key, hash64(0xDA7A, seed)))


def ratio_r(d: int, ratio: float) -> int:
    """r = max(1, llround(ratio * d)) (harness.cpp:212)."""
    import math
    x = ratio * d
    return max(1, int(math.floor(x + 0.5)) if x >= 0 else int(math.ceil(x - 0.5)))


class SparseAllgather:
    """One DP worker's encode → exchange → decode step on its CUDA device."""

    def __init__(self, codec: Codec, d: int, r: int, cfg: PipelineConfig, group=None):
        self.codec = codec
        self.d, self.r, self.cfg = d, r, cfg
        self.group = group
        self.world = dist.get_world_size(group) if dist.is_available() and dist.is_initialized() else 1
        self.rank = dist.get_rank(group) if self.world > 1 else 0
        dev = torch.device("cuda", torch.cuda.current_device())
        self.cap = Codec.max_container_bytes(d, r, cfg)
        self.out = torch.empty(self.cap, dtype=torch.uint8, device=dev)
        self.length = torch.zeros(1, dtype=torch.int64, device=dev)
        self.sizes = torch.zeros(self.world, dtype=torch.int64, device=dev)
        self.recv = torch.empty(self.world * self.cap, dtype=torch.uint8, device=dev) if self.world > 1 else None
        self.dense = torch.zeros(d, dtype=torch.float32, device=dev)

    def step(self, grad: torch.Tensor, step: int, seed: int = 1) -> torch.Tensor:
        """Returns the dense mean of every rank's decoded container (device f32[d])."""
        cfg = PipelineConfig(**{**self.cfg.__dict__, "seed": pipeline_seed(seed, self.rank, step)})
        self.codec.encode_into(grad, self.r, cfg, self.out, self.length)
        self.dense.zero_()
        n = self.world
        if n == 1:
            self.codec.decode_accumulate(self.out, self.dense, scale=1.0, length=self.length, hint=self.cfg)
            return self.dense
        # sizes first (one D2H of N words), then the payloads padded to the largest
        dist.all_gather_into_tensor(self.sizes, self.length, group=self.group)
        sizes = self.sizes.tolist()
        mx = max(sizes)
        dist.all_gather_into_tensor(self.recv[: n * mx], self.out[:mx], group=self.group)
        for j in range(n):  # fixed rank order, like the harness's worker order
            self.codec.decode_accumulate(self.recv[j * mx: j * mx + sizes[j]], self.dense, scale=1.0 / n,
                                         hint=self.cfg)
        return self.dense
