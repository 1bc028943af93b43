"""MMT projection GEMMs (T = 8192 tokens, d = 1024, FFN 4096) with each epilogue option,
vs cuBLAS as a yardstick: isolates what the fused epilogues (bias / GELU / pre-activation
store / residual / GELU' mask) cost on top of the tcgen05 main loop.

    python tools/bench_mmt_gemm.py [--reps 30]
"""
import argparse
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch

from paper_2406_17145_b200.runtime import lib
from tools.bench_gemm import timeit


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--reps", type=int, default=30)
    args = ap.parse_args()
    dev = torch.device("cuda", 0)
    T = 8192
    rows = []
    for (N, K) in [(3072, 1024), (1024, 1024), (4096, 1024), (1024, 4096)]:
        x = torch.randn(T, K, device=dev).bfloat16()
        w = (torch.randn(N, K, device=dev) / 32).bfloat16()
        b = torch.zeros(N, device=dev)
        y = torch.empty(T, N, device=dev, dtype=torch.bfloat16)
        pre = torch.empty_like(y)
        res = torch.randn(T, N, device=dev).bfloat16()
        dy = torch.randn(T, N, device=dev).bfloat16()
        dx = torch.empty(T, K, device=dev, dtype=torch.bfloat16)
        sv = torch.randn(T, K, device=dev).bfloat16()
        fl = 2.0 * T * N * K
        r = {"shape": [T, N, K]}
        r["fwd_plain"] = timeit(lambda: lib.linear_fwd(y, x, w, bias=None, act="none"), args.reps)
        r["fwd_bias"] = timeit(lambda: lib.linear_fwd(y, x, w, bias=b, act="none"), args.reps)
        r["fwd_gelu_pre"] = timeit(lambda: lib.linear_fwd(y, x, w, bias=b, act="gelu", pre=pre), args.reps)
        r["fwd_gelu"] = timeit(lambda: lib.linear_fwd(y, x, w, bias=b, act="gelu"), args.reps)
        r["fwd_residual"] = timeit(lambda: lib.linear_fwd(y, x, w, bias=b, act="none", residual=res), args.reps)
        r["dgrad_plain"] = timeit(lambda: lib.linear_dgrad(dx, dy, w, saved=None, act="none"), args.reps)
        r["dgrad_gelu"] = timeit(lambda: lib.linear_dgrad(dx, dy, w, saved=sv, act="gelu"), args.reps)
        r["cublas_fwd"] = timeit(lambda: torch.matmul(x, w.t()), args.reps)
        r["cublas_dgrad"] = timeit(lambda: torch.matmul(dy, w), args.reps)
        for k in list(r):
            if k != "shape":
                r[k] = f"{r[k]:.1f}us {fl / (r[k] * 1e-6) / 1e12:.0f}TF"
        rows.append(r)
        print(json.dumps(r), flush=True)


if __name__ == "__main__":
    main()
