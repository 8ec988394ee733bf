import torch
from paper_2102_03112_b200 import Codec
c = Codec(max_d=1 << 16)
t = torch.randint(0, 256, (1000,), dtype=torch.uint8, device="cuda")
print(c.crc32c(t[:64]))
