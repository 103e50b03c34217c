"""ncu target: write 32 MB (fill_), then read it (sum), twice; ncu reports the
DRAM bytes the read kernel fetched (L2 retention across kernel boundaries).
BIG=1: a 600 MB device allocation exists (like config 2's X) and is written
once first."""
import os

import torch

if os.environ.get("BIG") == "1":
    big = torch.empty(600 << 20, dtype=torch.uint8, device="cuda")
    big.zero_()
buf = torch.empty((32 << 20) // 8, dtype=torch.float64, device="cuda")
for _ in range(2):
    buf.fill_(1.0)
    s = buf.sum()
torch.cuda.synchronize()
print(float(s))
