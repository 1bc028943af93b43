"""Multi-GPU executor (NCCL P2P over NVLink + DP all-reduce) vs the CPU oracle.

Needs >= 2 (or 4) visible GPUs; skipped otherwise.  One process per GPU, like
bench.py under torchrun.  fp32 toy (rtol 1e-4) in a 2-stage GPP layout and a
4-rank layout with unequal micro-batch sizes and a DP-2 stage.
"""

import os
import socket
import tempfile

import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

pytestmark = pytest.mark.gpu

LR = 0.05
STEPS = 2
TOWER_A, TOWER_B, TAIL = [0, 1, 2, 3], [4, 5, 6, 7], [8, 9, 10]


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, layout, B, outdir, graphed=False, extra_edges=()):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    torch.cuda.set_device(rank)
    dist.init_process_group("nccl", rank=rank, world_size=world, device_id=torch.device("cuda", rank))
    try:
        from paper_2406_17145_b200 import model as M
        from paper_2406_17145_b200 import sched as S
        from paper_2406_17145_b200 import workloads as W
        from paper_2406_17145_b200.runtime.backend import CudaBackend
        from paper_2406_17145_b200.runtime.data import make_batch, to_device_rows
        from paper_2406_17145_b200.runtime.executor import Executor

        wl = W.toy(B=B)
        stages = [M.Stage(i, frozenset(ops), b, frozenset(devs)) for i, (ops, b, devs) in enumerate(layout)]
        edges = set(M.induced_stage_edges(wl.graph, [s.op_ids for s in stages])) | set(extra_edges)
        sg = S.schedule_stage_graph(M.StageGraph(stages, edges, B))
        dev = torch.device("cuda", rank)
        ex = Executor(wl, sg, rank, world, CudaBackend(dev), lr=LR, keep_grads=True)
        res = {"loss": [], "grads": []}
        g = None
        for step in range(STEPS):
            full = make_batch(wl, step)
            batch = to_device_rows(ex, full, ex.dtype, dev)
            if graphed:
                from paper_2406_17145_b200.runtime.graph import GraphedIteration
                if g is None:
                    # capture AFTER computing nothing: warm-up inside would advance the weights,
                    # so capture on a throwaway executor state and re-sync the params after
                    snap = ex.master.clone()
                    g = GraphedIteration(ex, batch, n_buffers=1, warmup=1)
                    ex.master.copy_(snap)
                    if ex.shadow is not None:
                        ex.shadow.copy_(ex.master.to(ex.shadow.dtype))
                for k in g.bufs[0]:
                    g.bufs[0][k].copy_(batch[k])
                loss = g.replay(0)
            else:
                loss = ex.run_iteration(batch)
            torch.cuda.synchronize()
            if ex.is_head:
                res["loss"].append(ex.stage_loss(loss))
            res["grads"].append({k: v.detach().cpu().clone() for k, v in ex.G.items()})
        torch.save(res, os.path.join(outdir, f"rank{rank}.pt"))
        dist.barrier()
    finally:
        dist.destroy_process_group()


def _run(layout, B, world, graphed=False, extra_edges=()):
    if torch.cuda.device_count() < world:
        pytest.skip(f"needs {world} GPUs")
    from oracle.reference_model import ReferenceModel
    from paper_2406_17145_b200 import workloads as W
    from paper_2406_17145_b200.runtime.data import make_batch

    with tempfile.TemporaryDirectory() as d:
        mp.spawn(_worker, args=(world, _free_port(), layout, B, d, graphed, extra_edges), nprocs=world, join=True)
        outs = [torch.load(os.path.join(d, f"rank{r}.pt")) for r in range(world)]
    wl = W.toy(B=B)
    ref = ReferenceModel(wl)
    for step in range(STEPS):
        rl, rg = ref.step(make_batch(wl, step), LR)
        losses = [o["loss"][step] for o in outs if o["loss"]]
        assert losses
        for l in losses:
            assert abs(l - rl.item()) <= 1e-4 * abs(rl.item())
        for o in outs:
            for k, g in o["grads"][step].items():
                err = ((g - rg[k]).abs().max() / (rg[k].abs().max() + 1e-12)).item()
                assert err < 1e-4, (k, err)


def test_two_stage_gpp_nccl():
    _run([(TOWER_A, 16, [0]), (TOWER_B + TAIL, 16, [1])], 64, 2)


def test_four_rank_unequal_b_and_dp_nccl():
    _run([(TOWER_A, 16, [0]), (TOWER_B, 32, [1, 2]), (TAIL, 8, [3])], 64, 4)


def test_two_stage_gpp_nccl_cuda_graph():
    """The whole rank iteration (kernels + NCCL P2P pieces) captured into a CUDA graph."""
    _run([(TOWER_A, 16, [0]), (TOWER_B + TAIL, 16, [1])], 64, 2, graphed=True)


def test_four_rank_dp_nccl_cuda_graph():
    _run([(TOWER_A, 16, [0]), (TOWER_B, 32, [1, 2]), (TAIL, 8, [3])], 64, 4, graphed=True)


def test_sequential_chain_tokens_nccl_cuda_graph():
    """SPP-shaped chain tower A -> tower B -> tail on 3 GPUs: the data-less chain edge
    A -> B is realised with NCCL token messages, inside the captured graph too."""
    _run([(TOWER_A, 16, [0]), (TOWER_B, 16, [1]), (TAIL, 16, [2])], 64, 3, graphed=True, extra_edges=[(0, 1)])
