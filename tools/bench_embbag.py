"""DLRM sparse SGD at the bench shape (26 tables x 1M rows x 64, B = 8192 bags of 100):
the fp32-atomic per-table scatter vs the deterministic multi-table kernel, CUDA-graph replay.

    python tools/bench_embbag.py
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
    T, R, M, bag = 26, 1_000_000, 8192, 100
    g = torch.Generator(device=dev).manual_seed(0)
    tables = [torch.randn(R, 64, device=dev, generator=g) * 0.05 for _ in range(T)]
    idxs = [torch.randint(0, R, (M, bag), device=dev, generator=g) for _ in range(T)]
    dps = [torch.randn(M, 64, device=dev, generator=g).bfloat16() for _ in range(T)]

    def atomic():
        for t, d, i in zip(tables, dps, idxs):
            lib.embbag_sgd(t, d, i, 1e-6)

    r = {"atomic_us": _time_us(atomic, 3), "deterministic_us": _time_us(lambda: lib.embbag_sgd_multi(tables, dps, idxs, 1e-6), 3)}
    r["rmw_bytes"] = T * M * bag * 64 * 4 * 2
    r["atomic_GBs"] = round(r["rmw_bytes"] / (r["atomic_us"] * 1e-6) / 1e9, 1)
    print(json.dumps({k: (round(v, 1) if isinstance(v, float) else v) for k, v in r.items()}))


if __name__ == "__main__":
    main()
