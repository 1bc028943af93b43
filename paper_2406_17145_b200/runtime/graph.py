"""CUDA-graph replay of one rank's whole training iteration.

The per-iteration program of a rank is static — the same kernels, shapes,
buffers and order every step — so it is captured once and replayed, removing
the per-launch host cost of ~150 C-ABI calls per step.  Two graphs read two
static input buffer sets so the next step's host->device copy can overlap the
current replay (bench.py e2e).  Multi-rank programs capture their NCCL P2P and
DP all-reduce too (NCCL supports stream capture); every rank must capture.
"""

from __future__ import annotations

import torch

from .executor import Executor


class GraphedIteration:
    def __init__(self, ex: Executor, batch_template: dict[str, torch.Tensor], n_buffers: int = 2,
                 warmup: int = 2):
        self.ex = ex
        self.bufs = [{k: v.clone() for k, v in batch_template.items()} for _ in range(n_buffers)]
        side = torch.cuda.Stream(ex.dev)
        side.wait_stream(torch.cuda.current_stream(ex.dev))
        with torch.cuda.stream(side):
            for _ in range(warmup):  # first launches set kernel attributes / scratch outside capture
                ex.run_iteration(self.bufs[0])
        torch.cuda.current_stream(ex.dev).wait_stream(side)
        torch.cuda.synchronize(ex.dev)
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
