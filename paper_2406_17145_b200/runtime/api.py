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


def plan(wl: Workload, n_gpus: int, mode: str = "gpp", opts: P.PartitionOptions | None = None,
         mem_bytes: float = 180e9, sweep: bool | None = None, min_microbatches: int = 1,
         max_microbatches: int = 32, costs: str = "measured", include_spp: bool | None = None) -> P.Strategy:
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
        best, best_t = None, None
        # GPP also tries join-merging stages (PartitionOptions.merge_join); SPP stays the
        # paper's sequential baseline
        merges = (False, True) if mode == "gpp" and P.merge_join_applicable(wl.graph, opts) else (False,)
        for b, _ in P.candidate_configs(B):
            if not (min_microbatches <= B // b <= max_microbatches):
                continue
            if include_spp is None:
                include_spp = mode == "gpp"
            arms = [(fn, mj) for mj in merges] + ([(P.spp_optimize, False)] if include_spp and mode == "gpp" else [])
            for f, mj in arms:
                o = P.PartitionOptions(**{**opts.__dict__, "micro_batches": (b,), "merge_join": mj,
                                          "rich_splits": f is P.optimize})
                try:
                    cand = f(wl.graph, cluster, B, o)
                except P.NoFeasibleStrategy:
                    continue
                t = twin(cand.stage_graph, cluster, wl.graph).iteration_ms
                if best_t is None or t < best_t:
                    best, best_t = cand, t
        if best is None:
            st = fn(wl.graph, cluster, wl.mini_batch, opts)
        else:
            st = best
    rep = validate_strategy(wl.graph, cluster, st.stage_graph)
    if rep:
        raise RuntimeError(f"partitioner produced an invalid strategy: {rep}")
    return st


def build(wl: Workload, sg: StageGraph, rank: int, world: int, device=None, lr: float = 1e-3,
          seed: int = 0) -> Executor:
    dev = torch.device("cuda", device if device is not None else torch.cuda.current_device())
    torch.cuda.set_device(dev)
    return Executor(wl, sg, rank, world, CudaBackend(dev), lr=lr, seed=seed)


@dataclass
class RunReport:
    losses: list[float]
    iteration_ms: list[float]
    samples_per_s: float
    stage_id: int | None
    extra: dict = field(default_factory=dict)


def execute(wl: Workload, sg: StageGraph, iters: int = 1, lr: float = 1e-3, seed: int = 0,
            ex: Executor | None = None) -> RunReport:
    """Train ``iters`` steps on this rank's share of ``sg`` (host batches -> device)."""
    rank, world, local = dist_env()
    ex = ex or build(wl, sg, rank, world, local, lr, seed)
    losses, times = [], []
    for step in range(iters):
        full = make_batch(wl, step, seed, keys=set(ex.data_keys()) if ex.stage else set())
        if world > 1:
            dist.barrier()
        torch.cuda.synchronize()
        t0 = torch.cuda.Event(enable_timing=True)
        t1 = torch.cuda.Event(enable_timing=True)
        t0.record()
        batch = to_device_rows(ex, full, ex.dtype, ex.dev) if ex.stage else {}
        loss = ex.run_iteration(batch)
        t1.record()
        torch.cuda.synchronize()
        times.append(t0.elapsed_time(t1))
        if loss is not None and ex.is_head:
            losses.append(ex.stage_loss(loss))
    ms = sum(times) / max(1, len(times))
    return RunReport(losses, times, wl.mini_batch / (ms / 1e3) if ms > 0 else 0.0,
                     ex.stage.id if ex.stage else None)
