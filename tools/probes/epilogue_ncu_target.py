"""ncu target: the plain bf16 forward epilogue with a one-k-block main loop
(8192 x 4096 x 64: 67 MB of output, 6.9 waves of 256 x 256 tiles), three launches."""
import os
import sys

sys.path.insert(0, os.getcwd())
import torch

from paper_2406_17145_b200.runtime import lib

dev = torch.device("cuda", 0)
x = torch.randn(8192, 64, device=dev).bfloat16()
w = (torch.randn(4096, 64, device=dev) / 8).bfloat16()
y = torch.empty(8192, 4096, device=dev, dtype=torch.bfloat16)
for _ in range(3):
    lib.linear_fwd(y, x, w, bias=None, act="none")
torch.cuda.synchronize()
