"""Device time of one encode (gp_encode_topr) of a config's rank-0 input, CUDA events, median of N.
   python tools/time_encode.py c3 [N]   (GP_EXPERIMENT selects kernel experiments)"""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_2102_03112_b200 import Codec, PipelineConfig
from paper_2102_03112_b200.configs import CONFIGS, case_input

cfg = CONFIGS[sys.argv[1]]
n = int(sys.argv[2]) if len(sys.argv) > 2 else 20
g, r, _ = case_input(cfg)
gd = torch.from_numpy(g).cuda()
codec = Codec(max_d=g.size)
pc = PipelineConfig(index_method=cfg["index"], value_method=cfg["value"], fpr=cfg["fpr"], degree=cfg["degree"],
                    max_segments=cfg["max_segments"], seed=7)
out = torch.empty(codec.max_container_bytes(g.size, r, pc), dtype=torch.uint8, device="cuda")
ln = torch.zeros(1, dtype=torch.int64, device="cuda")
flush = torch.empty(256 << 20, dtype=torch.uint8, device="cuda")
ts = []
for i in range(n + 3):
    flush.fill_(i & 255)
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record()
    codec.encode_into(gd, r, pc, out, ln)
    b.record()
    torch.cuda.synchronize()
    if i >= 3:
        ts.append(a.elapsed_time(b))
ts.sort()
print(sys.argv[1], "encode ms median", ts[len(ts) // 2], "min", ts[0])
codec.profile(True)
for i in range(5):
    codec.encode_into(gd, r, pc, out, ln)
torch.cuda.synchronize()
print(codec.stage_times())
