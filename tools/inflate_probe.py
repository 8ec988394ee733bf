"""Time the device decode of a reference-written Deflate-slot container (correctness path)."""
import time
import numpy as np
import torch
from oracle.bindings import GpConfig, reference, synthetic_gradient
from paper_2102_03112_b200 import Codec

ref = reference()
codec = Codec(max_d=1 << 22)
import sys
sizes = [(1_000_000, 10_000)] if "--small" in sys.argv else [(1_000_000, 10_000), (4_000_000, 400_000)]
for d, r in sizes:
    g = synthetic_gradient(d, rank=1)
    for slot in (0, 1):
        c = ref.encode_dense(g, r, GpConfig.make(1, 4, seed=3, slot_codec=slot))
        t = torch.from_numpy(np.frombuffer(c, np.uint8).copy()).cuda()
        dense = torch.zeros(d, dtype=torch.float32, device="cuda")
        codec.decode_accumulate(t, dense); codec.status()
        torch.cuda.synchronize(); t0 = time.perf_counter()
        for _ in range(3):
            codec.decode_accumulate(t, dense)
        codec.status(); torch.cuda.synchronize()
        ms = (time.perf_counter() - t0) / 3 * 1e3
        print(f"d={d} r={r} codec={'deflate' if slot else 'store'} bytes={len(c)} decode {ms:.2f} ms "
              f"({4 * r / ms / 1e6:.3f} GB/s of raw values)")
