"""One training iteration of a bench workload at N = 1 (its frozen single-stage plan) inside a
cudaProfilerStart/Stop range, after two warm-up iterations -- the target of

    ncu --profile-from-start off --metrics gpu__time_duration.sum --csv --log-file L.csv \\
        python tools/ncu_step.py --workload candle

(the step's launch list; `tools/launch_summary.py L.csv` summarises it).
"""
import argparse
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--workload", default="candle")
    a = ap.parse_args()
    from bench import _workload
    from paper_2406_17145_b200.runtime.api import build, plan_cached
    from paper_2406_17145_b200.runtime.data import make_batch, to_device_rows

    torch.cuda.set_device(0)
    wl = _workload(a.workload, 1, None)
    sg, _ = plan_cached(wl, 1, "gpp")
    ex = build(wl, sg, 0, 1, 0)
    dev = torch.device("cuda", 0)
    batch = to_device_rows(ex, make_batch(wl, 0), ex.dtype, dev)
    for _ in range(2):
        ex.run_iteration(batch)
    torch.cuda.synchronize()
    torch.cuda.profiler.start()
    ex.run_iteration(batch)
    torch.cuda.synchronize()
    torch.cuda.profiler.stop()


if __name__ == "__main__":
    main()
