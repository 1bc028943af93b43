"""Deterministic discrete-event simulator of one synchronous training iteration.

SPEC.md:417-479 (the reference ships no code for it).  It is the semantic
contract the B200 executor honours:

* each stage runs its task list Pi_i strictly in order on one logical executor
  (a DP stage is one executor with d-scaled durations);
* fw(y, j) is eligible when every predecessor's forward outputs covering
  samples [j*b_y, (j+1)*b_y) have arrived; bw(x, j) when every successor's
  gradients covering [j*b_x, (j+1)*b_x) have arrived;
* communication is a post-compute edge delay occupying no compute slot
  (SPEC.md:468); durations come from the cost module;
* no eligible task while work remains -> ``Deadlock``.

Because every stage executes a fixed order, start times are the longest paths
of the task-dependency DAG; the trace is ordered by (time, stage id, fw before
bw, index) — the SPEC's determinism tie-break.
"""

from __future__ import annotations

import json
from dataclasses import dataclass, field
from typing import Callable, Mapping

from .cost import DEFAULT_WEIGHT_MULTIPLIER, comm_time, stage_memory
from .model import ComputationGraph, DeviceCluster, StageGraph, pipeline_depth
from .spgraph import NormalizedGraph

__all__ = [
    "Deadlock",
    "SimEvent",
    "SimReport",
    "stage_edge_bytes",
    "covering_tasks",
    "simulate",
    "measure_min_inflight",
    "emit_trace",
]


class Deadlock(RuntimeError):
    def __init__(self, blocked: list):
        self.blocked = blocked
        super().__init__(f"deadlock: blocked tasks {blocked}")


@dataclass(frozen=True)
class SimEvent:
    time: float
    stage: int
    direction: str
    index: int
    kind: str  # "start" | "end"


@dataclass
class SimReport:
    iteration_ms: float
    peak_inflight_samples: dict[int, int]
    busy_ms: dict[int, float]
    idle_ms: dict[int, float]
    peak_mem_bytes: dict[int, float]
    warm_up_microbatches: int
    warm_up_per_stage: dict[int, int]
    depth: int
    task_times: dict[tuple[int, str, int], tuple[float, float]] = field(repr=False, default_factory=dict)
    trace: list[SimEvent] = field(repr=False, default_factory=list)

    @property
    def bubble_fraction(self) -> float:
        tot = sum(self.busy_ms.values()) + sum(self.idle_ms.values())
        return 0.0 if tot == 0 else sum(self.idle_ms.values()) / tot

    def bottleneck_tps(self, mini_batch: int) -> float:
        return max(self.busy_ms.values()) / mini_batch


def _graph_of(g):
    return g.graph if isinstance(g, NormalizedGraph) else g


def stage_edge_bytes(g, s: StageGraph) -> dict[tuple[int, int], float]:
    """Per-sample bytes on each stage edge: one tensor per distinct producer op crossing it."""
    cg = _graph_of(g)
    owner = {op: st.id for st in s.stages for op in st.op_ids}
    producers: dict[tuple[int, int], set[int]] = {e: set() for e in s.edges}
    for u, v in cg.edges:
        su, sv = owner.get(u), owner.get(v)
        if su is None or sv is None or su == sv:
            continue
        producers.setdefault((su, sv), set()).add(u)
    out: dict[tuple[int, int], float] = {}
    for e, us in producers.items():
        if isinstance(g, NormalizedGraph):
            out[e] = sum(g.effective_out_bytes[u] for u in us)
        else:
            out[e] = sum(cg.by_id[u].out_bytes_per_sample for u in us)
    return out


def covering_tasks(j: int, b_cons: int, b_prod: int) -> range:
    """Producer micro-batch indices overlapping consumer micro-batch j's sample range."""
    lo = j * b_cons
    hi = (j + 1) * b_cons
    return range(lo // b_prod, (hi - 1) // b_prod + 1)


def simulate(
    s: StageGraph,
    cluster: DeviceCluster | None,
    g: ComputationGraph | NormalizedGraph | None = None,
    durations: Callable[[int, str], float] | None = None,
    weight_multiplier: float = DEFAULT_WEIGHT_MULTIPLIER,
    sync_epilogue: bool = False,
    op_granular: bool = False,
    optimizer_bytes_per_param_byte: float = 0.0,
    hbm_bytes_per_ms: float = 6.5395e9,
) -> SimReport:
    """Simulate one iteration of a configured StageGraph.

    Task durations: ``durations(stage_id, direction)`` if given, else the sum of
    the stage ops' fwd/bwd cost curves at b/d.  Edge delays use ``comm_time``
    over the cluster's inter-stage bandwidth (zero-byte edges are free).

    ``op_granular`` (runtime twin, off for the SPEC semantics): a task runs its ops in
    the executor's order (topological for fw, reversed for bw) and each op waits only for
    its own remote inputs -- a producer's output leaves when the producing op finishes,
    not when its whole task does (the B200 executor posts receives up front, waits at the
    consuming op and ships pieces as soon as they are final, runtime/executor.py).
    ``optimizer_bytes_per_param_byte`` adds, with ``sync_epilogue``, the unfused optimizer
    pass a DP stage runs after its all-reduce (HBM-bound, ``hbm_bytes_per_ms``).
    """
    cg = _graph_of(g) if g is not None else None
    B = s.mini_batch
    for st in s.stages:
        if st.schedule is None:
            raise ValueError(f"stage {st.id} has no schedule")

    def dur(sid: int, direction: str) -> float:
        if durations is not None:
            return durations(sid, direction)
        st = s.by_id[sid]
        per = st.micro_batch // st.dp_degree
        tot = 0.0
        for op in sorted(st.op_ids):
            if cg is None or op not in cg.by_id:
                continue
            c = cg.by_id[op].fwd_cost if direction == "fw" else cg.by_id[op].bwd_cost
            tot += c.evaluate(per)
        return tot

    ebytes = stage_edge_bytes(g, s) if g is not None else {e: 0.0 for e in s.edges}

    def delay(e: tuple[int, int], samples: int) -> float:
        nb = ebytes.get(e, 0.0)
        if cluster is None or nb <= 0:
            return 0.0
        return comm_time(nb, samples, cluster.inter_bw, cluster.link_latency)

    preds = {st.id: s.predecessors(st.id) for st in s.stages}
    succs = {st.id: s.successors(st.id) for st in s.stages}
    dcache = {(st.id, d): dur(st.id, d) for st in s.stages for d in ("fw", "bw")}
    pos = {st.id: 0 for st in s.stages}
    free_at = {st.id: 0.0 for st in s.stages}
    times: dict[tuple[int, str, int], tuple[float, float]] = {}
    remaining = sum(len(st.schedule) for st in s.stages)

    # op-granular twin: per-op order / costs and the op-level finish times of every task
    op_fin: dict[tuple[int, str, int], dict[int, float]] = {}
    if op_granular:
        if cg is None:
            raise ValueError("op_granular simulation needs the computation graph")
        owner = {o: st.id for st in s.stages for o in st.op_ids}
        # stage edges without operator data still order whole tasks (token messages)
        data_pairs = {(owner[u], owner[v]) for u, v in cg.edges
                      if u in owner and v in owner and owner[u] != owner[v]}
        order = {}
        costs = {}
        for st in s.stages:
            ops = [o for o in cg.topo_order if o in st.op_ids]
            order[(st.id, "fw")] = ops
            order[(st.id, "bw")] = ops[::-1]
            per = st.micro_batch // st.dp_degree
            for d in ("fw", "bw"):
                costs[(st.id, d)] = {o: (cg.by_id[o].fwd_cost if d == "fw" else cg.by_id[o].bwd_cost).evaluate(per)
                                     for o in ops}

    def ready_time(sid: int, direction: str, j: int):
        st = s.by_id[sid]
        t = free_at[sid]
        if direction == "fw":
            for x in preds[sid]:
                bx = s.by_id[x].micro_batch
                for i in covering_tasks(j, st.micro_batch, bx):
                    key = (x, "fw", i)
                    if key not in times:
                        return None
                    t = max(t, times[key][1] + delay((x, sid), bx))
        else:
            for y in succs[sid]:
                by = s.by_id[y].micro_batch
                for i in covering_tasks(j, st.micro_batch, by):
                    key = (y, "bw", i)
                    if key not in times:
                        return None
                    t = max(t, times[key][1] + delay((sid, y), by))
        return t

    def op_timeline(sid: int, direction: str, j: int):
        """(start, end, per-op finish) of a task whose producers are all simulated."""
        st = s.by_id[sid]
        for nb in (preds[sid] if direction == "fw" else succs[sid]):
            bn = s.by_id[nb].micro_batch
            for i in covering_tasks(j, st.micro_batch, bn):
                if (nb, direction, i) not in times:
                    return None
        t = free_at[sid]
        t0 = None
        for nb in (preds[sid] if direction == "fw" else succs[sid]):
            if ((nb, sid) if direction == "fw" else (sid, nb)) in data_pairs:
                continue
            for i in covering_tasks(j, st.micro_batch, s.by_id[nb].micro_batch):
                t = max(t, times[(nb, direction, i)][1])
        fin = {}
        for o in order[(sid, direction)]:
            remote = ([u for u in cg.predecessors(o) if owner.get(u, sid) != sid] if direction == "fw"
                      else [v for v in cg.successors(o) if owner.get(v, sid) != sid])
            for u in remote:
                nb = owner[u]
                bn = s.by_id[nb].micro_batch
                e = (nb, sid) if direction == "fw" else (sid, nb)
                for i in covering_tasks(j, st.micro_batch, bn):
                    t = max(t, op_fin[(nb, direction, i)][u] + delay(e, bn))
            if t0 is None:
                t0 = t  # the task starts with its first op
            t += costs[(sid, direction)][o]
            fin[o] = t
        return (t if t0 is None else t0), t, fin

    while remaining:
        progressed = False
        for st in s.stages:  # ascending stage id
            sid = st.id
            while pos[sid] < len(st.schedule):
                task = st.schedule[pos[sid]]
                if op_granular:
                    tl = op_timeline(sid, task.direction, task.index)
                    if tl is None:
                        break
                    t0, t1, fin = tl
                    op_fin[(sid, task.direction, task.index)] = fin
                else:
                    t0 = ready_time(sid, task.direction, task.index)
                    if t0 is None:
                        break
                    t1 = t0 + dcache[(sid, task.direction)]
                times[(sid, task.direction, task.index)] = (t0, t1)
                free_at[sid] = t1
                pos[sid] += 1
                remaining -= 1
                progressed = True
        if not progressed:
            blocked = [(st.id, st.schedule[pos[st.id]].direction, st.schedule[pos[st.id]].index)
                       for st in s.stages if pos[st.id] < len(st.schedule)]
            raise Deadlock(blocked)

    iteration = max((t1 for _, t1 in times.values()), default=0.0)
    if sync_epilogue and cluster is not None and cg is not None:
        # weight-update epilogue: a DP stage all-reduces its gradients once per iteration
        # after its last task (SPEC.md:469 makes this configurable; default 0)
        from .cost import dp_sync_time
        for st in s.stages:
            if st.dp_degree > 1:
                last = max(t1 for (sid, _, _), (_, t1) in times.items() if sid == st.id)
                params = sum(cg.by_id[o].param_bytes for o in st.op_ids if o in cg.by_id)
                opt = optimizer_bytes_per_param_byte * params / hbm_bytes_per_ms
                iteration = max(iteration, last + dp_sync_time(params, st.dp_degree, cluster.intra_bw) + opt)
    busy = {st.id: sum(dcache[(st.id, t.direction)] for t in st.schedule) for st in s.stages}
    idle = {sid: iteration - b for sid, b in busy.items()}
    peak: dict[int, int] = {}
    warm: dict[int, int] = {}
    for st in s.stages:
        live = hi = 0
        first_bw = None
        for n, t in enumerate(st.schedule):
            live += 1 if t.direction == "fw" else -1
            hi = max(hi, live)
            if first_bw is None and t.direction == "bw":
                first_bw = n
        peak[st.id] = hi * st.micro_batch
        warm[st.id] = first_bw if first_bw is not None else len(st.schedule)
    mem: dict[int, float] = {}
    for st in s.stages:
        ops = [cg.by_id[o] for o in st.op_ids if cg is not None and o in cg.by_id]
        m = stage_memory(ops, st.dp_degree, peak[st.id], weight_multiplier).total
        for dev in st.devices:
            mem[dev] = max(mem.get(dev, 0.0), m)
    sources = s.source_stage_ids()
    events: list[SimEvent] = []
    for (sid, d, j), (t0, t1) in times.items():
        events.append(SimEvent(t0, sid, d, j, "start"))
        events.append(SimEvent(t1, sid, d, j, "end"))
    events.sort(key=lambda e: (e.time, e.stage, 0 if e.direction == "fw" else 1, e.index, e.kind != "end"))
    return SimReport(
        iteration_ms=iteration,
        peak_inflight_samples=peak,
        busy_ms=busy,
        idle_ms=idle,
        peak_mem_bytes=mem,
        warm_up_microbatches=max((warm[x] for x in sources), default=0),
        warm_up_per_stage=warm,
        depth=pipeline_depth(s),
        task_times=times,
        trace=events,
    )


def measure_min_inflight(
    b_x: int, k_x: int, b_y: int, k_y: int, i_y: int, mini_batch: int,
    fw_ms_per_sample: float = 1.0, bw_ms_per_sample: float = 1.0,
) -> int:
    """Smallest in-flight cap (samples, multiple of b_x) of the upstream stage of a
    two-stage chain that neither deadlocks nor lengthens the iteration versus an
    all-forwards-first upstream.  Oracle for Appendix A."""
    from .model import ScheduleConfig, Stage  # local: avoid a cycle at import time
    from .sched import schedule_tasks

    y_cfg = ScheduleConfig(i_y, b_y, k_y)
    y_sched = schedule_tasks(y_cfg, mini_batch)

    def run(i_x: int):
        x_cfg = ScheduleConfig(i_x, b_x, k_x)
        sg = StageGraph(
            [
                Stage(0, frozenset({0}), b_x, frozenset({0}), x_cfg, schedule_tasks(x_cfg, mini_batch)),
                Stage(1, frozenset({1}), b_y, frozenset({1}), y_cfg, y_sched),
            ],
            [(0, 1)],
            mini_batch,
        )
        per = {0: b_x, 1: b_y}
        try:
            return simulate(
                sg, None, None,
                durations=lambda sid, d: per[sid] * (fw_ms_per_sample if d == "fw" else bw_ms_per_sample),
            ).iteration_ms
        except Deadlock:
            return None

    ref = run(mini_batch)
    for i_x in range(b_x, mini_batch + 1, b_x):
        t = run(i_x)
        if t is not None and t <= ref + 1e-9:
            return i_x
    return mini_batch


def emit_trace(report: SimReport, stage_names: Mapping[int, str] | None = None) -> str:
    """Chrome trace-event JSON (name/cat/ph/ts/dur/pid/tid), one row per stage, µs units."""
    rows = []
    for (sid, d, j), (t0, t1) in sorted(report.task_times.items(), key=lambda kv: (kv[1][0], kv[0][0], kv[0][1] != "fw", kv[0][2])):
        rows.append({
            "name": f"{d}{j}",
            "cat": d,
            "ph": "X",
            "ts": round(t0 * 1000.0, 3),
            "dur": round((t1 - t0) * 1000.0, 3),
            "pid": 0,
            "tid": (stage_names or {}).get(sid, f"stage{sid}"),
        })
    return json.dumps({"traceEvents": rows, "displayTimeUnit": "ms"}, sort_keys=True)
