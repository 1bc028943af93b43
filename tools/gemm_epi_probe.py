"""The two GELU-epilogue MMT GEMMs alone (FFN1 forward with bias + GELU + pre-activation
store, 8192 x 4096 x 1024; FFN2 dgrad with the GELU' mask, 8192 x 4096 x 1024), three
launches each -- an ncu target (`-k regex:gemm_tc_pair --launch-skip 2 -c 1` = the FFN1
forward, `--launch-skip 5 -c 1` = the dgrad).

    python tools/gemm_epi_probe.py
"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch

from paper_2406_17145_b200.runtime import lib


def qkv():
    """--qkv: the QKV projection forward (8192 x 3072 x 1024, bias epilogue), three launches."""
    dev = torch.device("cuda", 0)
    x = torch.randn(8192, 1024, device=dev).bfloat16()
    w = (torch.randn(3072, 1024, device=dev) / 32).bfloat16()
    b = torch.zeros(3072, device=dev)
    y = torch.empty(8192, 3072, device=dev, dtype=torch.bfloat16)
    for _ in range(3):
        lib.linear_fwd(y, x, w, bias=b, act="none")
    torch.cuda.synchronize()


def main():
    if "--qkv" in sys.argv:
        return qkv()
    dev = torch.device("cuda", 0)
    T, N, K = 8192, 4096, 1024
    x = torch.randn(T, K, device=dev).bfloat16()
    w = (torch.randn(N, K, device=dev) / 32).bfloat16()
    b = torch.zeros(N, device=dev)
    y = torch.empty(T, N, device=dev, dtype=torch.bfloat16)
    pre = torch.empty_like(y)
    dy = torch.randn(T, K, device=dev).bfloat16()
    w2 = (torch.randn(K, N, device=dev) / 32).bfloat16()
    dx = torch.empty(T, N, device=dev, dtype=torch.bfloat16)
    for _ in range(3):
        lib.linear_fwd(y, x, w, bias=b, act="gelu", pre=pre)
    for _ in range(3):
        lib.linear_dgrad(dx, dy, w2, saved=pre, act="gelu")
    torch.cuda.synchronize()


if __name__ == "__main__":
    main()
