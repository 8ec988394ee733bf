"""Timing probe: the N=1 DP step eager vs captured in a CUDA graph (fixed seed;
measurement only, not a bench number)."""
import sys, time
import torch
sys.path.insert(0, ".")
from bench import CONFIGS
from paper_2102_03112_b200 import Codec, PipelineConfig, synth
from paper_2102_03112_b200.dp import SparseAllgather, ratio_r

for name in sys.argv[1:] or ["c4", "c1", "c2"]:
    cfg = CONFIGS[name]
    d = cfg["d"]
    grad = synth.gradient_torch(d, 0, device="cuda")
    r = ratio_r(d, cfg["ratio"])
    pcfg = PipelineConfig(index_method=cfg["index"], value_method=cfg["value"], fpr=cfg["fpr"], degree=cfg["degree"],
                          max_segments=cfg["max_segments"])
    codec = Codec(max_d=d)
    ex = SparseAllgather(codec, d, r, pcfg)
    s = torch.cuda.Stream()
    with torch.cuda.stream(s):
        for _ in range(3):
            ex.step(grad, step=0)
        torch.cuda.synchronize()
        g = torch.cuda.CUDAGraph()
        with torch.cuda.graph(g, stream=s):
            ex.step(grad, step=0)
        torch.cuda.synchronize()
        flush = torch.empty(64 << 20, dtype=torch.float32, device="cuda")
        for mode in ["eager", "graph"]:
            ts = []
            for i in range(10):
                flush.fill_(float(i))
                a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                a.record(s)
                if mode == "eager":
                    ex.step(grad, step=0)
                else:
                    g.replay()
                b.record(s)
                b.synchronize()
                ts.append(a.elapsed_time(b))
            print(name, mode, round(sum(ts) / len(ts), 4), "ms", flush=True)
    codec.status()
