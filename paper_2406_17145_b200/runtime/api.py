"""Public runtime API: plan a strategy, build the executor, run training steps.

``execute(s, cluster, model, batch_source, iters)`` is the real counterpart of
``sim.simulate(s, cluster)``: it runs a configured
StageGraph on B200s and returns a ``RunReport`` with the SimReport fields that
are measurable plus throughput.
"""

from __future__ import annotations

import os
from dataclasses import dataclass, field

import torch
import torch.distributed as dist

from .. import partition as P
from ..model import StageGraph, validate_strategy
from ..workloads import Workload, b200_cluster
from .backend import CudaBackend
from .data import make_batch, to_device_rows
from .executor import Executor

__all__ = ["plan", "twin", "build", "RunReport", "execute", "dist_env"]


def dist_env() -> tuple[int, int, int]:
    """(rank, world, local_rank) from torchrun's environment (1 process per GPU)."""
    return (int(os.environ.get("RANK", 0)), int(os.environ.get("WORLD_SIZE", 1)),
            int(os.environ.get("LOCAL_RANK", 0)))


def twin(sg: StageGraph, cluster, graph):
    """The executor's simulated twin: op-granular sends/receives (what runtime.executor
    does) and, for DP stages, the once-per-iteration all-reduce plus the unfused SGD pass
    (14 B per parameter = 3.5 x the fp32 param_bytes) after the last task."""
    from ..sim import simulate

    return simulate(sg, cluster, graph, sync_epilogue=True, op_granular=True, optimizer_bytes_per_param_byte=3.5)


def refine_per_stage(sg: StageGraph, cluster, graph, mem_bytes: float | None = None, passes: int = 3,
                     time_budget_s: float = 45.0) -> tuple[StageGraph, dict]:
    """Per-stage (b, k) for a fixed partition: the runtime planner's kFkB mode (SPEC.md:320,
    PAPER.md:747-749).

    The exact per-stage search inside the SP-DP (``PartitionOptions.per_stage_schedules``)
    enumerates every (b, k) pair at every stage boundary -- 464 s on MMT-4 at 4 GPUs.  Here
    the partition, devices and edges of the uniform-b plan are kept and each stage's
    micro-batch b (powers of two within 4x of its current b that divide B and the stage's DP
    degree) and k (1, 2, 4) are improved by coordinate descent, every candidate rescheduled
    with the Appendix-A in-flight calculus (``schedule_stage_graph`` with the ks pinned) and
    scored by the executor's twin.  Returns (stage graph, info)."""
    import time

    from ..model import Stage
    from ..sched import schedule_stage_graph

    t0 = time.perf_counter()
    B = sg.mini_batch
    mem = mem_bytes if mem_bytes is not None else cluster.mem_per_device

    def build_sg(bs: dict, ks: dict):
        raw = StageGraph([Stage(st.id, st.op_ids, bs[st.id], st.devices) for st in sg.stages], sg.edges, B)
        return schedule_stage_graph(raw, mem_limit=mem, g=graph, fixed_k=ks)

    from ..sim import Deadlock

    def score(cand):
        if cand is None:
            return None
        try:
            return twin(cand, cluster, graph).iteration_ms
        except Deadlock:  # e.g. a k-block larger than a neighbour's in-flight window
            return None

    bs = {st.id: st.micro_batch for st in sg.stages}
    ks = {st.id: (st.sched_cfg.k if st.sched_cfg else 1) for st in sg.stages}
    best_sg = build_sg(bs, ks)
    best = score(best_sg)
    if best is None:
        return sg, {"refined": False, "reason": "base plan infeasible under the memory cap"}
    start, evals = best, 1
    for _ in range(passes):
        improved = False
        for st in sg.stages:
            d = st.dp_degree
            b0 = bs[st.id]
            cands_b = [b for b in (b0 // 4, b0 // 2, b0, 2 * b0, 4 * b0)
                       if b >= d and b % d == 0 and B % b == 0 and b & (b - 1) == 0]
            for b in cands_b:
                for k in (1, 2, 4):
                    if k > B // b or (b == bs[st.id] and k == ks[st.id]):
                        continue
                    if time.perf_counter() - t0 > time_budget_s:
                        break
                    tb, tk = dict(bs), dict(ks)
                    tb[st.id], tk[st.id] = b, k
                    cand = build_sg(tb, tk)
                    t = score(cand)
                    evals += 1
                    if t is not None and t < best - 1e-9:
                        best, best_sg, bs, ks, improved = t, cand, tb, tk, True
        if not improved:
            break
    return best_sg, {"refined": True, "twin_ms_before": start, "twin_ms_after": best, "evals": evals,
                     "seconds": round(time.perf_counter() - t0, 2),
                     "b": {sid: bs[sid] for sid in sorted(bs)}, "k": {sid: ks[sid] for sid in sorted(ks)}}


def _plan_candidate(job):
    """One sweep candidate: (strategy, twin iteration ms) or None if infeasible."""
    fname, graph, cluster, B, o = job
    f = getattr(P, fname)
    try:
        cand = f(graph, cluster, B, o)
    except P.NoFeasibleStrategy:
        return None
    return cand, twin(cand.stage_graph, cluster, graph).iteration_ms


def _map_candidates(jobs):
    workers = min(len(jobs), int(os.environ.get("GPP_PLAN_WORKERS", os.cpu_count() or 1)))
    if workers <= 1 or len(jobs) <= 1:
        return [_plan_candidate(j) for j in jobs]
    import multiprocessing as mp
    import threading
    from concurrent.futures import ProcessPoolExecutor

    # fork: the candidates are pure Python (no CUDA in the children); serial otherwise
    if "fork" not in mp.get_all_start_methods() or threading.current_thread() is not threading.main_thread():
        return [_plan_candidate(j) for j in jobs]
    with ProcessPoolExecutor(workers, mp_context=mp.get_context("fork")) as pool:
        return list(pool.map(_plan_candidate, jobs))


def plan(wl: Workload, n_gpus: int, mode: str = "gpp", opts: P.PartitionOptions | None = None,
         mem_bytes: float = 180e9, sweep: bool | None = None, min_microbatches: int = 1,
         max_microbatches: int = 32, costs: str = "measured", include_spp: bool | None = None,
         info: dict | None = None, per_stage: bool = False) -> P.Strategy:
    """Run the GPP (or SPP baseline) partitioner + scheduler for ``n_gpus`` B200s.

    The TPS objective (Eq. 1) is a steady-state measure: with launch overheads in the
    cost curves it always prefers one giant micro-batch, i.e. no pipelining at all.
    Like the paper's evaluation ("We sweep over all possible micro-batch sizes ...
    to maximize training throughput"), ``sweep`` runs the optimizer
    once per uniform micro-batch size b (B/b in [min_microbatches, max_microbatches])
    and keeps the strategy with the shortest simulated iteration (sim.simulate),
    which does see warm-up / cool-down bubbles.  Single-GPU plans skip the sweep.

    A sequential pipeline is itself a graph pipeline (a chain of stages), but the SP-DP
    only cuts at series/parallel boundaries, so it can miss a balanced chain cut through
    the middle of a parallel region (DLRM at 2 GPUs: 30/5 ops, twin 8.63 ms, vs the
    sequential 18/17-op cut, 7.46 ms).  With ``include_spp`` (default for GPP sweeps) the
    SPP candidates join the GPP sweep and the twin picks; ``optimize`` itself is unchanged.
    ``info`` (a dict) receives the twin's iteration time of the pick, which arm produced
    it, and the best pure-``optimize`` (GraphPipe partitioner) candidate on its own.
    ``per_stage``: then refine each stage's (b, k) on the picked partition
    (``refine_per_stage``; GPP mode, N > 1).
    """
    from ..sim import simulate
    from ..workloads import with_measured_curves

    if costs == "measured":  # frozen B200 tables where profiled (falls back to analytic curves)
        wl = with_measured_curves(wl)[0]
    cluster = b200_cluster(n_gpus, mem_bytes)
    fn = P.optimize if mode == "gpp" else P.spp_optimize
    opts = opts or P.PartitionOptions(sync_per_iteration=True)
    if sweep is None:
        sweep = n_gpus > 1 and opts.micro_batches is None
    if not sweep:
        st = fn(wl.graph, cluster, wl.mini_batch, opts)
    else:
        B = wl.mini_batch
        best, best_t, best_arm = None, None, None
        gbest, gbest_t = None, None
        # GPP also tries join-merging stages (PartitionOptions.merge_join); SPP stays the
        # paper's sequential baseline
        merges = (False, True) if mode == "gpp" and P.merge_join_applicable(wl.graph, opts) else (False,)
        if include_spp is None:
            include_spp = mode == "gpp"
        jobs = []
        for b, _ in P.candidate_configs(B):
            if not (min_microbatches <= B // b <= max_microbatches):
                continue
            arms = [(fn, mj) for mj in merges] + ([(P.spp_optimize, False)] if include_spp and mode == "gpp" else [])
            for f, mj in arms:
                o = P.PartitionOptions(**{**opts.__dict__, "micro_batches": (b,), "merge_join": mj,
                                          "rich_splits": f is P.optimize})
                jobs.append((f.__name__, wl.graph, cluster, B, o))
        # the sweep's candidates are independent: one process each (results consumed in the
        # serial order, so the pick is identical to a serial sweep)
        results = _map_candidates(jobs)
        for (fname, *_), res in zip(jobs, results):
            if res is None:
                continue
            cand, t = res
            if best_t is None or t < best_t:
                best, best_t = cand, t
                best_arm = fname
            if fname != "spp_optimize" and (gbest_t is None or t < gbest_t):
                gbest, gbest_t = cand, t
        if best is None:
            st = fn(wl.graph, cluster, wl.mini_batch, opts)
        else:
            st = best
        if info is not None:
            info.update({"twin_ms": best_t, "picked_by": best_arm,
                         "gpp_partitioner": None if gbest is None else {"strategy": gbest, "twin_ms": gbest_t}})
    if per_stage and mode == "gpp" and n_gpus > 1:
        import dataclasses

        refined, rinfo = refine_per_stage(st.stage_graph, cluster, wl.graph, mem_bytes)
        if info is not None:
            info["per_stage"] = rinfo
        if rinfo.get("refined") and rinfo["twin_ms_after"] < rinfo["twin_ms_before"]:
            st = dataclasses.replace(st, stage_graph=refined)
    rep = validate_strategy(wl.graph, cluster, st.stage_graph)
    if rep:
        raise RuntimeError(f"partitioner produced an invalid strategy: {rep}")
    return st


STRATEGY_DIR = os.path.join(os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))),
                            "profiles", "strategies")


def _planning_graph(wl: Workload, costs: str):
    from ..workloads import with_measured_curves

    return with_measured_curves(wl)[0].graph if costs == "measured" else wl.graph


def strategy_path(wl: Workload, n_gpus: int, mode: str, costs: str = "measured", cache_dir: str | None = None) -> str:
    g = wl.graph
    return os.path.join(cache_dir or STRATEGY_DIR,
                        f"{wl.name}-{len(g.op_ids)}ops_{mode}_n{n_gpus}_B{wl.mini_batch}_{costs}.json")


def plan_cached(wl: Workload, n_gpus: int, mode: str = "gpp", costs: str = "measured",
                cache_dir: str | None = None, write: bool = False) -> tuple[StageGraph, dict]:
    """``plan`` through a frozen StrategyFile (cli.py format).

    The file embeds the cost-annotated graph it was planned on; it is used only if that
    graph equals the current one exactly (same ops, edges, curves), so a stale plan can
    never run.  Otherwise the strategy is planned now (and written when ``write``).
    Returns (configured StageGraph, meta) — meta: source ("frozen" | "planned"),
    plan_s, the twin's iteration time, which arm won, and the pure GraphPipe partitioner
    (``optimize``) candidate's stages / twin time."""
    import json
    import time

    from ..cli import FORMAT_VERSION, graph_to_json, strategy_from_json, strategy_to_json

    path = strategy_path(wl, n_gpus, mode, costs, cache_dir)
    g = _planning_graph(wl, costs)
    want = graph_to_json(g)
    if os.path.exists(path):
        with open(path) as f:
            doc = json.load(f)
        if doc.get("format_version") == FORMAT_VERSION and doc.get("strategy", {}).get("graph") == want:
            sg, _, _ = strategy_from_json(doc["strategy"])
            return sg, {**doc.get("meta", {}), "source": "frozen", "path": os.path.relpath(path)}
    info: dict = {}
    t0 = time.perf_counter()
    st = plan(wl, n_gpus, mode, costs=costs, info=info)
    dt = time.perf_counter() - t0
    gp = info.get("gpp_partitioner")
    meta = {"plan_s": round(dt, 3), "twin_ms": info.get("twin_ms"), "picked_by": info.get("picked_by"),
            "gpp_partitioner": None if gp is None else {
                "twin_ms": gp["twin_ms"],
                "stages": [{"ops": sorted(x.op_ids), "b": x.micro_batch, "devices": sorted(x.devices),
                            "k": x.sched_cfg.k if x.sched_cfg else None} for x in gp["strategy"].stage_graph.stages]}}
    if write:
        os.makedirs(os.path.dirname(path), exist_ok=True)
        doc = {"format_version": FORMAT_VERSION, "kind": "frozen_strategy", "workload": wl.name,
               "n_gpus": n_gpus, "mode": mode, "costs": costs, "meta": meta,
               "strategy": strategy_to_json(st.stage_graph, g)}
        with open(path, "w") as f:
            json.dump(doc, f, sort_keys=True, separators=(",", ":"))
    return st.stage_graph, {**meta, "source": "planned"}


def build(wl: Workload, sg: StageGraph, rank: int, world: int, device=None, lr: float = 1e-3,
          seed: int = 0, timed: bool = False) -> Executor:
    dev = torch.device("cuda", device if device is not None else torch.cuda.current_device())
    torch.cuda.set_device(dev)
    if timed:
        from .profiler import TimedBackend

        be = TimedBackend(dev)
        be.enabled = False
    else:
        be = CudaBackend(dev)
    return Executor(wl, sg, rank, world, be, lr=lr, seed=seed)


@dataclass
class RunReport:
    """What ``execute`` measured — the SimReport fields plus throughput.

    Stage- and device-keyed fields cover every rank (gathered to all ranks).  ``busy_ms``
    is the stage's kernel time per iteration (mean over its DP replicas), ``idle_ms`` =
    iteration - busy; both need ``trace=True`` (CUDA events around every kernel of the
    last iteration), otherwise they are empty and ``trace`` is None."""

    iteration_ms: float
    peak_inflight_samples: dict[int, int]
    busy_ms: dict[int, float]
    idle_ms: dict[int, float]
    peak_mem_bytes: dict[int, float]
    warm_up_microbatches: int
    warm_up_per_stage: dict[int, int]
    depth: int
    trace: str | None
    losses: list[float]
    iteration_times_ms: list[float]
    samples_per_s: float
    stage_id: int | None
    h2d_bytes_per_step: int = 0
    d2h_bytes_per_step: int = 0
    task_times: dict = field(default_factory=dict, repr=False)
    extra: dict = field(default_factory=dict)

    @property
    def bubble_fraction(self) -> float | None:
        tot = sum(self.busy_ms.values()) + sum(self.idle_ms.values())
        return None if not self.busy_ms or tot == 0 else sum(self.idle_ms.values()) / tot


def _schedule_fields(s: StageGraph) -> tuple[dict, dict, int]:
    """Peak in-flight samples and warm-up micro-batches of the task lists as executed
    (each rank runs its stage's Pi verbatim; the executor's ring depth is this peak)."""
    peak, warm = {}, {}
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
    srcs = s.source_stage_ids()
    return peak, warm, max((warm[x] for x in srcs), default=0)


def host_batch(ex: Executor, full: dict[str, torch.Tensor]) -> dict[str, torch.Tensor]:
    """This rank's rows of a full CPU batch, cast for the compute dtype, in pinned memory."""
    out = {}
    for k in ex.data_keys() if ex.stage else []:
        t = ex.local_rows(full[k])
        if t.is_floating_point():
            t = t.to(ex.dtype) if t.dim() > 1 else t.float()
        out[k] = t.pin_memory()
    return out


def execute(s: StageGraph, cluster, wl: Workload, batch_source=None, iters: int = 1, lr: float = 1e-3,
            seed: int = 0, graph: bool = True, trace: bool = False, ex: Executor | None = None) -> RunReport:
    """Run ``iters`` synchronous training iterations of the configured StageGraph ``s`` on
    this rank's B200 (one process per GPU, torchrun env) — the executed counterpart of
    ``sim.simulate(s, cluster)``.

    Every step copies that step's input rows from pinned host memory to the device and
    reads the loss back: ``batch_source(step) -> {key: full [B, ...] CPU tensor}``
    (default: the seeded synthetic batches of ``runtime.data.make_batch``).  With
    ``graph`` the iteration is captured once (warm-up effects undone, so training is
    identical to eager) and replayed, the next step's H2D overlapping the current
    replay.  With ``trace`` every kernel is bracketed by CUDA-event nodes and the last
    iteration's task times become the Chrome trace (``runtime.trace``) and the
    busy / idle fields.  ``cluster`` is validated against the strategy (C1-C4)."""
    from ..model import pipeline_depth
    from .data import make_batch
    from .graph import GraphedIteration
    from .trace import emit_measured_trace, stage_summary

    rep = validate_strategy(wl.graph, cluster, s)
    if rep:
        raise ValueError(f"invalid strategy: {rep}")
    rank, world, local = dist_env()
    if world > 1 and not dist.is_initialized():
        dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    ex = ex or build(wl, s, rank, world, local, lr, seed, timed=trace)
    if trace and not hasattr(ex.be, "task_times"):
        raise ValueError("trace=True needs an executor built on profiler.TimedBackend")
    dev = ex.dev
    src = batch_source or (lambda step: make_batch(wl, step, seed, keys=set(ex.data_keys()) if ex.stage else set()))
    fulls = [src(i) for i in range(min(2, iters))]
    hosts = [host_batch(ex, f) for f in fulls]
    h2d = sum(t.numel() * t.element_size() for t in hosts[0].values()) if hosts else 0
    torch.cuda.reset_peak_memory_stats(dev)
    dev_bufs = None
    graphed = None
    if graph and iters > 0:
        tmpl = {k: v.to(dev) for k, v in hosts[0].items()}

        def arm_trace():
            if trace:
                ex.be.reset()
                ex.be.enabled = True
                ex.be.external = True

        graphed = GraphedIteration(ex, tmpl, n_buffers=1 if trace else 2, preserve_state=True,
                                   before_capture=arm_trace)
        if trace:
            ex.be.enabled = False
        dev_bufs = graphed.bufs
    else:
        dev_bufs = [{k: torch.empty_like(v, device=dev) for k, v in hosts[0].items()} for _ in range(2)] if hosts else []
        if trace:
            ex.be.enabled = False
    copy_stream = torch.cuda.Stream(dev)
    nb = len(dev_bufs)
    ready = [torch.cuda.Event() for _ in range(nb)]
    consumed = [torch.cuda.Event() for _ in range(nb)]
    for e in consumed:
        e.record()
    loss_host = torch.zeros(max(1, iters), dtype=torch.float32).pin_memory()
    has_loss = False

    pinned: dict[int, dict] = {id(f): h for f, h in zip(fulls, hosts)}

    def stage_h2d(i):
        if not hosts:
            return
        full = fulls[i] if i < len(fulls) else src(i)
        hb = pinned.get(id(full))
        if hb is None:  # a new batch: stage it (sources that cycle a few batches are pinned once)
            hb = host_batch(ex, full)
            if len(pinned) < 4:
                pinned[id(full)] = hb
        with torch.cuda.stream(copy_stream):
            copy_stream.wait_event(consumed[i % nb])
            for k, v in hb.items():
                dev_bufs[i % nb][k].copy_(v, non_blocking=True)
            ready[i % nb].record(copy_stream)

    if world > 1:
        dist.barrier()
    torch.cuda.synchronize(dev)
    stage_h2d(0)
    ev = []
    for i in range(iters):
        t0, t1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        t0.record()
        if hosts:
            torch.cuda.current_stream().wait_event(ready[i % nb])
        if graphed is not None:
            loss = graphed.replay(i % nb)
        else:
            if trace and i == iters - 1:
                ex.be.reset()
                ex.be.enabled = True
            loss = ex.run_iteration(dev_bufs[i % nb] if dev_bufs else {})
            if trace:
                ex.be.enabled = False
        consumed[i % nb].record()
        if i + 1 < iters:
            stage_h2d(i + 1)  # on the copy stream: overlaps this step (double-buffered)
        if loss is not None and ex.is_head:
            has_loss = True
            loss_host[i:i + 1].copy_(loss, non_blocking=True)
        t1.record()
        ev.append((t0, t1))
    torch.cuda.synchronize(dev)
    times = [a.elapsed_time(b) for a, b in ev]
    # max over ranks per iteration (the slowest rank bounds the synchronous step)
    tt = torch.tensor(times or [0.0], dtype=torch.float64, device=dev)
    if world > 1:
        dist.all_reduce(tt, op=dist.ReduceOp.MAX)
    times = tt.tolist() if times else []
    losses = []
    if has_loss:
        l = loss_host[:iters].to(dev)
        if ex.d > 1:
            ex.tp.allreduce(l)  # a DP head stage: sum of the replicas' shares
        losses = l.tolist()
    ms = sum(times) / len(times) if times else 0.0
    from .lib import embbag_check_indices

    if ex.stage is not None and ex.tables:
        embbag_check_indices()
    my = {"rank": rank, "stage": ex.stage.id if ex.stage else None, "losses": losses,
          "peak_mem": float(torch.cuda.max_memory_allocated(dev)),
          "tasks": ex.be.task_times() if trace else {}}
    allr = [my]
    if world > 1:
        allr = [None] * world
        dist.all_gather_object(allr, my)
    peak, warm_per, warm = _schedule_fields(s)
    tt_by_rank = {r["rank"]: r["tasks"] for r in allr}
    summ = stage_summary(tt_by_rank, {r["rank"]: r["stage"] for r in allr}, ms) if trace else {"busy_ms": {}, "idle_ms": {}}
    head_losses = next((r["losses"] for r in allr if r["losses"]), [])
    return RunReport(
        iteration_ms=ms, peak_inflight_samples=peak, busy_ms=summ["busy_ms"], idle_ms=summ["idle_ms"],
        peak_mem_bytes={r["rank"]: r["peak_mem"] for r in allr}, warm_up_microbatches=warm,
        warm_up_per_stage=warm_per, depth=pipeline_depth(s),
        trace=emit_measured_trace(tt_by_rank) if trace else None, losses=head_losses,
        iteration_times_ms=times, samples_per_s=wl.mini_batch / (ms / 1e3) if ms > 0 else 0.0,
        stage_id=ex.stage.id if ex.stage else None, h2d_bytes_per_step=int(h2d),
        d2h_bytes_per_step=4 if has_loss else 0, task_times=tt_by_rank,
        extra={"graph": graphed is not None, "executor": ex})
