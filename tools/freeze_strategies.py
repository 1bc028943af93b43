"""Plan and freeze the benchmark strategies as StrategyFiles (profiles/strategies/).

    python tools/freeze_strategies.py [--gpus 1 2 4 8] [--jobs 6]

bench.py loads these through ``runtime.api.plan_cached`` (used only when the embedded
cost-annotated graph equals the current one), so an 8-GPU bench run does not spend
minutes in the partitioner.  Workloads follow bench.py's weak scaling: MMT B = 16 N
(4 branches; the BASELINE configs[4] branch sweep 2 / 8 at N >= 2), CANDLE-Uno
B = 1024 N, DLRM B = 8192 N; GPP and SPP arms each.
"""

from __future__ import annotations

import argparse
import os
import sys
import time
from concurrent.futures import ProcessPoolExecutor

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def jobs_for(gpus):
    out = []
    for n in gpus:
        for mode in ("gpp", "spp"):
            if n == 1 and mode == "spp":
                continue
            out += [("mmt", n, mode, 4), ("candle", n, mode, None), ("dlrm", n, mode, None)]
            if n > 1:
                out += [("mmt", n, mode, 2), ("mmt", n, mode, 8)]
    return out


def run(job):
    name, n, mode, br = job
    sys.path.insert(0, ROOT)
    from bench import _workload
    from paper_2406_17145_b200.runtime.api import plan_cached

    wl = _workload(name, n, None, br)
    t0 = time.perf_counter()
    sg, meta = plan_cached(wl, n, mode, write=True)
    return job, meta["source"], round(time.perf_counter() - t0, 1), [(len(s.op_ids), s.micro_batch, s.dp_degree) for s in sg.stages]


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, nargs="+", default=[1, 2, 4, 8])
    ap.add_argument("--jobs", type=int, default=max(1, (os.cpu_count() or 2) - 1))
    a = ap.parse_args()
    js = sorted(jobs_for(a.gpus), key=lambda j: -j[1])  # the slow 8-GPU plans first
    with ProcessPoolExecutor(a.jobs) as pool:
        for job, src, dt, stages in pool.map(run, js):
            print(job, src, f"{dt}s", stages, flush=True)


if __name__ == "__main__":
    main()
