"""CUDA-graph replay of one rank's whole training iteration.

The per-iteration program of a rank is static — the same kernels, shapes,
buffers and order every step — so it is captured once and replayed, removing
the per-launch host cost of ~150 C-ABI calls per step.  Two graphs read two
static input buffer sets so the next step's host->device copy can overlap the
current replay (bench.py e2e, runtime.api.execute).  Multi-rank programs
capture their NCCL P2P and DP all-reduce too (NCCL supports stream capture);
every rank must capture.

Capture needs one or two eager iterations first (kernel attributes, split-K /
LayerNorm scratch are sized outside capture).  With ``preserve_state`` those
warm-up iterations are undone: master / shadow / gradient buffers and the
embedding tables are snapshotted before and restored after, so a captured run
trains exactly like an eager one from the same state.
"""

from __future__ import annotations

import torch

from .executor import Executor


def _state(ex: Executor) -> list[torch.Tensor]:
    ts = [ex.master, ex.grad] + ([ex.shadow] if ex.shadow is not None else [])
    return ts + list(ex.tables.values())


class GraphedIteration:
    def __init__(self, ex: Executor, batch_template: dict[str, torch.Tensor], n_buffers: int = 2,
                 warmup: int = 2, preserve_state: bool = False, before_capture=None):
        self.ex = ex
        self.bufs = [{k: v.clone() for k, v in batch_template.items()} for _ in range(n_buffers)]
        saved = [t.clone() for t in _state(ex)] if (preserve_state and ex.stage is not None) else None
        side = torch.cuda.Stream(ex.dev)
        side.wait_stream(torch.cuda.current_stream(ex.dev))
        with torch.cuda.stream(side):
            for _ in range(warmup):  # first launches set kernel attributes / scratch outside capture
                ex.run_iteration(self.bufs[0])
        torch.cuda.current_stream(ex.dev).wait_stream(side)
        torch.cuda.synchronize(ex.dev)
        if saved is not None:
            for dst, src in zip(_state(ex), saved):
                dst.copy_(src)
            del saved
            torch.cuda.synchronize(ex.dev)
        if before_capture is not None:
            before_capture()
        self.graphs, self.losses = [], []
        for b in self.bufs:
            g = torch.cuda.CUDAGraph()
            if ex.world > 1:
                import torch.distributed as dist
                dist.barrier()
            with torch.cuda.graph(g):
                loss = ex.run_iteration(b)
            self.graphs.append(g)
            self.losses.append(loss)

    def replay(self, i: int = 0):
        self.graphs[i % len(self.graphs)].replay()
        return self.losses[i % len(self.losses)]
