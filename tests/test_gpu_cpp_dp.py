"""The C-ABI data-parallel step (gp_dp_*, csrc/dp_exchange.cpp) driven from C++
(tests/cpp/dp_test.cpp), one host thread per rank.

`local`: an in-process group of N contexts on one GPU — the full step (encode,
lengths allgather, the one host sync, padded payload allgather, rank-order
decode into the mean) with device copies as the transport.  `nccl`: a
single-rank NCCL communicator (one GPU), the NCCL allgather path.  Every
rank's mean (and, with compensation, its f64 residual) must equal, bit for
bit, the same worker loop run through the Python API of the codec — encode
with Simulation::pipeline_seed(1, rank, step) (harness.cpp:201-203), decode in
rank order with scale 1/N — whose pieces the parity suites check against the
reference; and every rank must hold the same mean (harness.cpp:287-288).
"""
import os
import subprocess

import numpy as np
import pytest
import torch

from oracle.bindings import synthetic_gradient

pytestmark = pytest.mark.gpu

HERE = os.path.dirname(os.path.abspath(__file__))
BIN = os.path.join(HERE, "cpp", "dp_test")


def _replay(n, d, r, im, vm, fpr, steps, ef):
    from paper_2102_03112_b200 import Codec, PipelineConfig
    from paper_2102_03112_b200.seeds import pipeline_seed
    codec = Codec(max_d=d)
    grads = [torch.from_numpy(synthetic_gradient(d, rank=k)).cuda() for k in range(n)]
    res = [torch.zeros(d, dtype=torch.float64, device="cuda") for _ in range(n)]
    means, resids = [], []
    try:
        for step in range(steps):
            cs = []
            for k in range(n):
                cfg = PipelineConfig(index_method=im, value_method=vm, fpr=fpr, seed=pipeline_seed(1, k, step))
                cs.append(codec.compress_ef64(grads[k], res[k], r, cfg) if ef else codec.compress(grads[k], r, cfg))
            mean = torch.zeros(d, dtype=torch.float32, device="cuda")
            for k in range(n):
                codec.decode_accumulate(cs[k], mean, scale=1.0 / n)
            codec.status()
            means.append(mean.cpu().numpy())
            resids.append([x.cpu().numpy().copy() for x in res])
    finally:
        codec.close()
    return means, resids


@pytest.mark.parametrize("mode,n,im,vm,fpr,ef", [
    ("local", 2, 6, 1, 0.001, 0),   # P2 + fit (the C4 pipeline)
    ("local", 3, 1, 0, 0.01, 0),    # bitmap + raw
    ("local", 2, 4, 1, 0.01, 1),    # P0 + fit with f64 compensation
    ("local", 4, 2, 0, 0.01, 1),    # RLE + raw with f64 compensation
    ("nccl", 1, 6, 1, 0.001, 0),
    ("nccl", 1, 1, 0, 0.01, 1),
])
def test_cpp_dp_step(tmp_path, mode, n, im, vm, fpr, ef):
    if mode == "nccl":
        try:
            import ctypes
            ctypes.CDLL("libnccl.so.2")
        except OSError:
            pytest.skip("libnccl.so.2 not loadable")
    d, r, steps = 300_007, 3_000, 3
    for k in range(n):
        synthetic_gradient(d, rank=k).astype(np.float32).tofile(tmp_path / f"g_{k}.bin")
    out = subprocess.run([BIN, mode, str(n), str(d), str(r), str(im), str(vm), str(fpr), str(steps), str(ef),
                          str(tmp_path), str(tmp_path)], capture_output=True, text=True, timeout=600)
    assert out.returncode == 0, out.stderr
    means, resids = _replay(n, d, r, im, vm, fpr, steps, ef)
    for step in range(steps):
        for k in range(n):
            got = np.fromfile(tmp_path / f"mean_{k}_{step}.bin", dtype=np.float32)
            assert np.array_equal(got, means[step]), f"rank {k} step {step}: mean differs"
            if ef:
                e = np.fromfile(tmp_path / f"res_{k}_{step}.bin", dtype=np.float64)
                assert np.array_equal(e, resids[step][k]), f"rank {k} step {step}: residual differs"
