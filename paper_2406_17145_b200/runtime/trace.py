"""Measured task trace of an executed iteration, in the simulator's Chrome-trace schema.

``sim.emit_trace`` writes one ``X`` event per task — name
``fw3``/``bw3``, cat = direction, ts/dur in µs, one row (tid) per stage.  The
executor's measured counterpart comes from CUDA events around every kernel of
the iteration (``profiler.TimedBackend`` tags each launch with the task being
executed): a task spans its first kernel's start to its last kernel's end,
relative to the rank's iteration-start event, and its ``busy`` time is the sum
of its kernel durations (stream waits for peers excluded).  ``trace_diff``
compares a measured iteration with the simulated twin task by task.
"""

from __future__ import annotations

import json
from typing import Mapping

__all__ = ["emit_measured_trace", "trace_diff", "stage_summary"]


def emit_measured_trace(task_times_by_rank: Mapping[int, dict], stage_names: Mapping[int, str] | None = None) -> str:
    """Chrome trace JSON: ``task_times_by_rank[rank][(stage, dir, j)] = (t0_ms, t1_ms, busy_ms)``.
    Same keys as ``sim.emit_trace`` (name/cat/ph/ts/dur/pid/tid); pid = rank (a DP stage's
    replicas are separate rows), args.busy_us = the task's kernel time."""
    rows = []
    for rank, times in sorted(task_times_by_rank.items()):
        for (sid, d, j), (t0, t1, busy) in sorted(times.items(), key=lambda kv: (kv[1][0], kv[0][0], kv[0][1], kv[0][2])):
            rows.append({
                "name": f"{d}{j}" if d in ("fw", "bw") else d,
                "cat": d,
                "ph": "X",
                "ts": round(t0 * 1000.0, 3),
                "dur": round((t1 - t0) * 1000.0, 3),
                "pid": rank,
                "tid": (stage_names or {}).get(sid, f"stage{sid}"),
                "args": {"busy_us": round(busy * 1000.0, 3)},
            })
    return json.dumps({"traceEvents": rows, "displayTimeUnit": "ms"}, sort_keys=True)


def stage_summary(task_times_by_rank: Mapping[int, dict], stage_of_rank: Mapping[int, int],
                  iteration_ms: float) -> dict:
    """Per stage: busy (kernel ms per iteration, mean over the stage's replicas; optimizer
    epilogue included) and idle = iteration - busy — the SimReport busy/idle fields."""
    per: dict[int, list[float]] = {}
    for rank, times in task_times_by_rank.items():
        sid = stage_of_rank.get(rank)
        if sid is None:
            continue
        per.setdefault(sid, []).append(sum(v[2] for v in times.values()))
    busy = {sid: sum(v) / len(v) for sid, v in per.items()}
    return {"busy_ms": busy, "idle_ms": {sid: max(0.0, iteration_ms - b) for sid, b in busy.items()}}


def trace_diff(task_times_by_rank: Mapping[int, dict], sim_report) -> dict:
    """Measured vs simulated iteration, task by task (fw/bw tasks of every stage).

    ``order_equal``: every rank ran its stage's tasks in the simulated order (Π is never
    reordered); ``start_rank_corr``: Spearman correlation of measured vs
    simulated task start times over all tasks (the pipeline shape); per-stage measured vs
    simulated busy time; measured vs simulated iteration length."""
    sim_t = sim_report.task_times
    order_equal = True
    pairs = []
    seen = set()
    meas_busy: dict[int, float] = {}
    meas_end = 0.0
    for rank, times in task_times_by_rank.items():
        tasks = {k: v for k, v in times.items() if k[1] in ("fw", "bw")}
        if not tasks:
            continue
        sid = next(iter(tasks))[0]
        mine = sorted(tasks, key=lambda k: tasks[k][0])
        sims = sorted((k for k in sim_t if k[0] == sid), key=lambda k: sim_t[k][0])
        if [k[1:] for k in mine] != [k[1:] for k in sims]:
            order_equal = False
        meas_busy[sid] = sum(v[2] for v in tasks.values())
        meas_end = max(meas_end, max(v[1] for v in times.values()))
        for k in mine:
            if k in sim_t and k not in seen:
                seen.add(k)
                pairs.append((tasks[k][0], sim_t[k][0]))

    def ranks(xs):
        order = sorted(range(len(xs)), key=lambda i: xs[i])
        r = [0.0] * len(xs)
        for pos, i in enumerate(order):
            r[i] = float(pos)
        return r

    corr = None
    if len(pairs) > 2:
        a, b = ranks([p[0] for p in pairs]), ranks([p[1] for p in pairs])
        n = len(a)
        ma, mb = sum(a) / n, sum(b) / n
        cov = sum((x - ma) * (y - mb) for x, y in zip(a, b))
        va = sum((x - ma) ** 2 for x in a) ** 0.5
        vb = sum((y - mb) ** 2 for y in b) ** 0.5
        corr = cov / (va * vb) if va > 0 and vb > 0 else None
    return {
        "tasks_compared": len(pairs),
        "order_equal": order_equal,
        "start_rank_corr": corr,
        "iteration_ms": {"measured": meas_end, "simulated": sim_report.iteration_ms},
        "busy_ms": {sid: {"measured": meas_busy[sid], "simulated": sim_report.busy_ms.get(sid)} for sid in sorted(meas_busy)},
    }
