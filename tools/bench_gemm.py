"""GEMM microbenchmark: libgpp_b200 dense-operator GEMMs vs cuBLAS (yardstick) on B200.

    python tools/bench_gemm.py [--reps 50]

Shapes are the CANDLE-Uno training-step GEMMs at b = 1024 (fw / dgrad / wgrad of
Linear(4096,4096) and of the Linear(28672,1024) tail).  Times are CUDA events
around `reps` back-to-back launches after warm-up (L2-warm for weights that fit).
"""
import argparse
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch

from paper_2406_17145_b200.runtime import lib


def timeit(fn, reps):
    for _ in range(3):
        fn()
    torch.cuda.synchronize()
    s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    s.record()
    for _ in range(reps):
        fn()
    e.record()
    torch.cuda.synchronize()
    return s.elapsed_time(e) / reps * 1e3  # us


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--reps", type=int, default=50)
    args = ap.parse_args()
    dev = torch.device("cuda", 0)
    out = []
    for (M, N, K) in [(1024, 4096, 4096), (1024, 1024, 28672), (2048, 4096, 4096), (4096, 4096, 4096)]:
        x = torch.randn(M, K, device=dev).bfloat16()
        w = (torch.randn(N, K, device=dev) / 64).bfloat16()
        y = torch.empty(M, N, device=dev, dtype=torch.bfloat16)
        dy = torch.randn(M, N, device=dev).bfloat16()
        dx = torch.empty(M, K, device=dev, dtype=torch.bfloat16)
        dw = torch.empty(N, K, device=dev)
        b = torch.zeros(N, device=dev)
        fl = 2.0 * M * N * K
        r = {"shape": [M, N, K]}
        r["fwd_us"] = timeit(lambda: lib.linear_fwd(y, x, w, bias=b, act="relu"), args.reps)
        r["dgrad_us"] = timeit(lambda: lib.linear_dgrad(dx, dy, w, saved=x, act="relu"), args.reps)
        r["wgrad_us"] = timeit(lambda: lib.linear_wgrad(dw, None, dy, x), args.reps)
        r["cublas_fwd_us"] = timeit(lambda: torch.matmul(x, w.t()), args.reps)
        r["cublas_dgrad_us"] = timeit(lambda: torch.matmul(dy, w), args.reps)
        r["cublas_wgrad_us"] = timeit(lambda: torch.matmul(dy.t(), x), args.reps)
        for k in list(r):
            if k.endswith("_us"):
                r[k.replace("_us", "_tflops")] = round(fl / (r[k] * 1e-6) / 1e12, 1)
                r[k] = round(r[k], 2)
        out.append(r)
        print(json.dumps(r), flush=True)


if __name__ == "__main__":
    main()
