"""Phase timeline of the attention backward's dK/dV role (CTA 0, first 64 query blocks).

Needs a library built with -DGPP_ATTN_TRACE (on the GPU box:
  sed -i '1i #define GPP_ATTN_TRACE' paper_2406_17145_b200/csrc/attn_flash_sm100.cu
then build()).  Events per block g (SM clock): 0 stage landed (MMA warp), 1 S/dP issued,
2 softmax sees S/dP, 3 softmax done, 4 MMA warp sees P/dS (dV/dK issue), 5 TMA stage issued.
"""
import ctypes
import json
import os
import sys

sys.path.insert(0, os.path.join(os.path.dirname(os.path.abspath(__file__)), "..", ".."))

import torch

from paper_2406_17145_b200.runtime import lib

B, S, H, d = 16, 512, 16, 1024
dev = "cuda"
g = torch.Generator(device=dev).manual_seed(0)
qkv = (torch.randn(B * S, 3 * d, device=dev, generator=g) * 0.5).bfloat16()
o = torch.empty(B * S, d, device=dev, dtype=torch.bfloat16)
lse2 = torch.empty(B * H, S, device=dev, dtype=torch.float32)
dout = torch.randn(B * S, d, device=dev, generator=g).bfloat16()
dvec = torch.empty(B * H, S, device=dev, dtype=torch.float32)
dqkv = torch.empty_like(qkv)
sc = 1.0 / 8.0
h = lib.load()
lib.flash_attn_fwd(qkv, lse2, o, B, S, d, H, sc)
for _ in range(5):
    lib.flash_attn_bwd(qkv, lse2, o, dout, dvec, dqkv, B, S, d, H, sc)
torch.cuda.synchronize()
buf = (ctypes.c_longlong * (6 * 64))()
h.gpp_attn_trace_read(buf)
t = [[buf[e * 64 + i] for i in range(64)] for e in range(6)]
t0 = min(x for row in t for x in row if x)
rows = []
for i in range(64):
    rows.append([t[e][i] - t0 if t[e][i] else None for e in range(6)])
names = ["landed", "sp_issued", "sm_start", "sm_done", "p_seen", "tma_issued"]
print(json.dumps({"events": names, "rows": rows}))
for i, r in enumerate(rows[:40]):
    print(i, r, file=sys.stderr)
