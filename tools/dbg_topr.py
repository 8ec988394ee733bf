import sys, os
sys.path.insert(0, '/root/repo'); sys.path.insert(0, '/root/repo/tests')
import numpy as np, torch
from oracle.bindings import synthetic_gradient
from paper_2102_03112_b200 import Codec, PipelineConfig
codec = Codec(max_d=1 << 22)
rng = np.random.default_rng(0)
sizes = [1, 2, 3, 7, 64, 1000, 4097, 65536 + 3, 269722, 1_000_000]
for d in sizes:
    g = synthetic_gradient(d, rank=d % 5)
    for r in sorted({1, max(1, d // 100), max(1, d // 3), d}):
        print("d", d, "r", r, flush=True)
        c = codec.compress(torch.from_numpy(g).cuda(), r, PipelineConfig(index_method=1, value_method=0, seed=r))
