"""Per-kernel-family time of one graph-replayed training iteration of a bench workload at
N = 1, measured in the step itself (CUDA-event nodes around every kernel-launching call,
runtime.profiler.TimedBackend): GEMMs by (kind, m, n, k) with TF/s, every other call by
name.  Event nodes cost a little per kernel; compare shares, not the absolute step time.

    python tools/step_breakdown.py [--workload mmt|candle|dlrm]
"""
import argparse
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--workload", default="mmt")
    a = ap.parse_args()
    from bench import _workload
    from paper_2406_17145_b200.runtime.api import build, execute, plan_cached
    from paper_2406_17145_b200.runtime.data import make_batch
    from paper_2406_17145_b200.workloads import b200_cluster

    torch.cuda.set_device(0)
    wl = _workload(a.workload, 1, None)
    sg, _ = plan_cached(wl, 1, "gpp")
    ex = build(wl, sg, 0, 1, 0, timed=True)
    fulls = [make_batch(wl, s + 1) for s in range(2)]
    execute(sg, b200_cluster(1), wl, batch_source=lambda i: fulls[i % 2], iters=3, ex=ex)
    ex.be.reset()
    rep = execute(sg, b200_cluster(1), wl, batch_source=lambda i: fulls[i % 2], iters=2, trace=True, ex=ex)
    s = ex.be.summary()
    out = {"workload": a.workload, "iteration_ms_traced": round(rep.iteration_times_ms[-1], 3),
           "busy_ms": round(s["busy_ms"], 3), "gemm_ms": round(s["ms"], 3), "gemm_tflops": round(s["tflops"], 1),
           "gemm_by_shape": {k: {kk: round(vv, 2) for kk, vv in v.items()} for k, v in s["by_shape"].items()},
           "other_ms": {k: {"launches": v["launches"], "ms": round(v["ms"], 3)} for k, v in s["other_ms"].items()}}
    print(json.dumps(out, indent=1))


if __name__ == "__main__":
    main()
