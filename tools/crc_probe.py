"""Times gp_crc32c alone over several sizes (CUDA events, warm) — probe."""
import torch
from paper_2102_03112_b200 import Codec
from paper_2102_03112_b200._lib import lib
from paper_2102_03112_b200.api import _ptr, _stream

codec = Codec(max_d=1 << 20)
buf = torch.randint(0, 256, (90_000_000,), dtype=torch.uint8, device="cuda")
out = torch.zeros(1, dtype=torch.int64, device="cuda")
for n in [0, 64, 4096, 1_260_000, 10_000_000, 80_000_000]:
    for _ in range(5):
        lib.gp_crc32c(codec._ctx, _ptr(buf), n, _ptr(out), _stream())
    torch.cuda.synchronize()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record()
    for _ in range(50):
        lib.gp_crc32c(codec._ctx, _ptr(buf), n, _ptr(out), _stream())
    b.record()
    torch.cuda.synchronize()
    print(n, "us/launch", round(a.elapsed_time(b) * 1000 / 50, 2))
