import os, sys, time
import numpy as np, torch
sys.path.insert(0, ".")
from paper_2102_03112_b200 import Codec, PipelineConfig
from paper_2102_03112_b200.synth import gradient_torch
d = int(sys.argv[1]) if len(sys.argv) > 1 else 25557032
r = d // 100
codec = Codec(max_d=d)
g = gradient_torch(d, 0)
cfg = PipelineConfig(index_method=3, value_method=0, seed=1)
c = codec.compress(g, r, cfg)
dense = torch.zeros(d, dtype=torch.float32, device="cuda")
for rounds in ["24"]:
    os.environ["GP_HUFF_FIX_ROUNDS"] = rounds
    codec.decode_accumulate(c, dense, hint=cfg)
    codec.status()
    torch.cuda.synchronize()
    t = time.perf_counter()
    codec.decode_accumulate(c, dense, hint=cfg)
    codec.status()
    torch.cuda.synchronize()
    print(d, "rounds", rounds, round((time.perf_counter() - t) * 1e3, 3), "ms", flush=True)
