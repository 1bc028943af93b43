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

__all__ = ["plan", "build", "RunReport", "execute", "dist_env"]


def dist_env() -> tuple[int, int, int]:
    """(rank, world, local_rank) from torchrun's environment (1 process per GPU)."""
    return (int(os.environ.get("RANK", 0)), int(os.environ.get("WORLD_SIZE", 1)),
            int(os.environ.get("LOCAL_RANK", 0)))


def plan(wl: Workload, n_gpus: int, mode: str = "gpp", opts: P.PartitionOptions | None = None,
         mem_bytes: float = 180e9) -> P.Strategy:
    """Run the GPP (or SPP baseline) partitioner + scheduler for ``n_gpus`` B200s."""
    cluster = b200_cluster(n_gpus, mem_bytes)
    fn = P.optimize if mode == "gpp" else P.spp_optimize
    st = fn(wl.graph, cluster, wl.mini_batch, opts)
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
            l = loss.clone()
            if ex.d > 1:
                dist.all_reduce(l, group=ex.dp_group)
            losses.append(float(l.item()))
    ms = sum(times) / max(1, len(times))
    return RunReport(losses, times, wl.mini_batch / (ms / 1e3) if ms > 0 else 0.0,
                     ex.stage.id if ex.stage else None)
