"""MMT glue kernels at the MMT step's shapes (T = 8192 tokens, d = 1024, FFN 4096), timed by
CUDA-graph replay of 20 launches each (true per-launch time, no event nodes):
LayerNorm fwd / bwd (+ its dgamma/dbeta reduction), the bias-gradient column sums, mean-pool.
Reports achieved GB/s against the measured HBM copy bandwidth.

    python tools/bench_glue.py
"""
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch

from paper_2406_17145_b200.runtime import lib
from paper_2406_17145_b200.runtime.profiler import _time_us


def main():
    dev = torch.device("cuda", 0)
    torch.cuda.set_device(dev)
    T, D, F = 8192, 1024, 4096
    bw = json.load(open(os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "MEASURED_PEAKS.json"))).get("hbm_gbs", 6446.0) \
        if os.path.exists("MEASURED_PEAKS.json") else 6446.0
    x = torch.randn(T, D, device=dev).bfloat16()
    y = torch.empty_like(x)
    g = 1 + 0.1 * torch.randn(D, device=dev)
    b = 0.1 * torch.randn(D, device=dev)
    mean, rstd = torch.empty(T, device=dev), torch.empty(T, device=dev)
    dy, dres, dx = torch.randn_like(x.float()).bfloat16(), torch.randn_like(x.float()).bfloat16(), torch.empty_like(x)
    dg, db = torch.zeros(D, device=dev), torch.zeros(D, device=dev)
    rows = []

    def rec(name, us, nbytes):
        rows.append({"kernel": name, "us": round(us, 2), "MB": round(nbytes / 1e6, 1),
                     "GBs": round(nbytes / (us * 1e-6) / 1e9, 1), "frac_hbm": round(nbytes / (us * 1e-6) / 1e9 / bw, 3)})

    rec("layernorm_fwd T=8192 D=1024", _time_us(lambda: lib.layernorm_fwd(y, mean, rstd, x, g, b), 20), 2 * T * D * 2 + 8 * T)
    rec("layernorm_bwd (+dres, + dgamma/dbeta reduce)", _time_us(
        lambda: lib.layernorm_bwd(dx, dg, db, dy, x, mean, rstd, g, dres, True), 20), 4 * T * D * 2 + 8 * T)
    for n in (1024, 3072, 4096):
        z = torch.randn(T, n, device=dev).bfloat16()
        out = torch.zeros(n, device=dev)
        rec(f"colsum T=8192 N={n}", _time_us(lambda: lib.colsum(out, z, True), 20), T * n * 2)
    print(json.dumps(rows, indent=1))


if __name__ == "__main__":
    main()
