"""Fused wgrad + SGD GEMM microbenchmark under in-step memory conditions.

    python tools/bench_wgrad_sgd.py [--layers 8] [--reps 10]

Rotates over `layers` distinct Linear(4096,4096) weight sets (fp32 master + bf16 shadow,
~96 MB each) so the masters are not L2-resident, as in a training step.  Reports the
fused wgrad+SGD time, the plain fp32 wgrad time and the bias colsum time per layer, plus
the algorithmic HBM bytes of the fused kernel (dy, x, master read+write, shadow write).
"""
import argparse
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch

from paper_2406_17145_b200.runtime import lib


def timeit(fn, n, reps):
    """Per-launch device time of n rotating launches, replayed from a CUDA graph so host
    launch overhead (ctypes) does not hide short kernels."""
    for i in range(2 * n):
        fn(i % n)
    torch.cuda.synchronize()
    side = torch.cuda.Stream()
    side.wait_stream(torch.cuda.current_stream())
    g = torch.cuda.CUDAGraph()
    with torch.cuda.stream(side):
        with torch.cuda.graph(g, stream=side):
            for i in range(n):
                fn(i)
    torch.cuda.synchronize()
    g.replay()
    torch.cuda.synchronize()
    s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    s.record()
    for r in range(reps):
        g.replay()
    e.record()
    torch.cuda.synchronize()
    return s.elapsed_time(e) / (reps * n) * 1e3  # us per launch


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--layers", type=int, default=8)
    ap.add_argument("--reps", type=int, default=10)
    ap.add_argument("--batch", type=int, default=1024)
    ap.add_argument("--width", type=int, default=4096, help="in features (and out unless --out-width)")
    ap.add_argument("--out-width", type=int, default=None)
    args = ap.parse_args()
    dev = torch.device("cuda", 0)
    B, W, L = args.batch, args.width, args.layers
    O = args.out_width or W
    master = [torch.randn(O, W, device=dev) / 64 for _ in range(L)]
    shadow = [m.bfloat16() for m in master]
    grad = [torch.zeros(O, W, device=dev) for _ in range(L)]
    dy = [torch.randn(B, O, device=dev).bfloat16() for _ in range(L)]
    x = [torch.randn(B, W, device=dev).bfloat16() for _ in range(L)]
    db = torch.zeros(O, device=dev)
    r = {"shape": [O, W, B], "layers": L, "timing": "CUDA-graph replay"}
    r["wgrad_sgd_us"] = timeit(lambda i: lib.linear_wgrad_sgd(master[i], shadow[i], grad[i], dy[i], x[i], 1e-6), L, args.reps)
    r["wgrad_sgd_acc_us"] = timeit(
        lambda i: lib.linear_wgrad_sgd(master[i], shadow[i], grad[i], dy[i], x[i], 1e-6, accumulate=True), L, args.reps)
    r["wgrad_sgd_bias_us"] = timeit(
        lambda i: lib.linear_wgrad_sgd(master[i], shadow[i], grad[i], dy[i], x[i], 1e-6, dbias=db), L, args.reps)
    r["wgrad_f32_us"] = timeit(lambda i: lib.linear_wgrad(grad[i], None, dy[i], x[i]), L, args.reps)
    r["colsum_us"] = timeit(lambda i: lib.colsum(db, dy[i]), L, args.reps)
    flops = 2.0 * O * W * B
    hbm = B * (O + W) * 2 + O * W * (4 + 4 + 2)
    r["wgrad_sgd_tflops"] = round(flops / r["wgrad_sgd_us"] / 1e6, 1)
    r["wgrad_sgd_algo_GBs"] = round(hbm / r["wgrad_sgd_us"] / 1e3, 1)
    r["floor_us"] = {"tensor@1.5PF": round(flops / 1.5e9, 1), "hbm@7.0TB/s": round(hbm / 7.0e6, 1)}
    for k in list(r):
        if k.endswith("_us") and isinstance(r[k], float):
            r[k] = round(r[k], 2)
    print(json.dumps(r), flush=True)


if __name__ == "__main__":
    main()
