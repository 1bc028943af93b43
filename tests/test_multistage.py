"""Multi-stage GPP executor parity with the CUDA kernels on ONE GPU (bf16, rtol 2e-2).

(``backend="cuda"``, marked gpu.  The same layouts also run on CPU with the oracle's
torch kernel backend, ``backend="torch-cpu"``, to check the host logic in the CPU suite.)

Several executor ranks share cuda:0 (one process each, like torchrun ranks) and
move their stage-edge pieces through a host-staged gloo transport
(tests/_hoststaged.py); all compute runs through libgpp_b200.so.  This exercises
what the 1-GPU driver box can't reach with NCCL: pieces covering sample ranges
with unequal micro-batch sizes, the re-shard into and out of a DP-2 stage, the
DP all-reduce / all-gather, data-less token edges, cuts
inside an MMT branch ([b, S*d] activations on the edge) — checked per rank,
per step against the monolithic CPU oracle with the device's ReLU masks.
"""

import os
import socket
import tempfile

import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from oracle.reference_model import ReferenceModel
from paper_2406_17145_b200 import model as M
from paper_2406_17145_b200 import sched as S
from paper_2406_17145_b200 import workloads as W
from paper_2406_17145_b200.runtime.data import make_batch

from _parity import assert_close, masks_from_taps

BACKENDS = [pytest.param("cuda", marks=pytest.mark.gpu), "torch-cpu"]

LR = 1e-2
STEPS = 2


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _sg(wl, layout, extra_edges=()):
    stages = [M.Stage(i, frozenset(ops), b, frozenset(devs)) for i, (ops, b, devs) in enumerate(layout)]
    edges = set(M.induced_stage_edges(wl.graph, [s.op_ids for s in stages])) | set(extra_edges)
    sg = S.schedule_stage_graph(M.StageGraph(stages, edges, wl.mini_batch))
    assert M.validate_strategy(wl.graph, M.DeviceCluster(8, 1e12, 1, 1), sg) == []
    return sg


def _worker(rank, world, port, make_wl, layout, extra_edges, outdir, backend):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        from paper_2406_17145_b200.runtime.data import to_device_rows
        from paper_2406_17145_b200.runtime.executor import Executor
        from _hoststaged import HostStagedTransport

        wl = make_wl()
        sg = _sg(wl, layout, extra_edges)
        if backend == "cuda":
            from paper_2406_17145_b200.runtime.backend import CudaBackend

            dev = torch.device("cuda", 0)  # every rank on the same GPU
            torch.cuda.set_device(dev)
            be = CudaBackend(dev)
        else:
            from oracle.torch_backend import TorchBackend

            dev = torch.device("cpu")
            be = TorchBackend()
        ex = Executor(wl, sg, rank, world, be, lr=LR, keep_grads=True, transport=HostStagedTransport)
        res = []
        for step in range(STEPS):
            full = make_batch(wl, step)
            before = {k: v.detach().cpu().clone() for k, v in ex.P.items()}
            ex.tap = {}
            loss = ex.run_iteration(to_device_rows(ex, full, ex.dtype, dev) if ex.stage else {})
            if backend == "cuda":
                torch.cuda.synchronize()
            rec = {"before": before, "after": {k: v.detach().cpu().clone() for k, v in ex.P.items()},
                   "grads": {k: v.detach().cpu().clone() for k, v in ex.G.items()},
                   "taps": {k: v.cpu() for k, v in ex.tap.items()},
                   "loss": ex.stage_loss(loss) if (loss is not None and ex.is_head) else None}
            ex.tap = None
            res.append(rec)
        dist.barrier()
        torch.save(res, os.path.join(outdir, f"rank{rank}.pt"))
    finally:
        dist.destroy_process_group()


def _run(backend, make_wl, layout, extra_edges=()):
    world = max(max(devs) for _, _, devs in layout) + 1
    if backend == "cuda" and not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    with tempfile.TemporaryDirectory() as d:
        mp.spawn(_worker, args=(world, _free_port(), make_wl, layout, tuple(extra_edges), d, backend),
                 nprocs=world, join=True)
        outs = [torch.load(os.path.join(d, f"rank{r}.pt")) for r in range(world)]
    wl = make_wl()
    sg = _sg(wl, layout, extra_edges)
    ref = ReferenceModel(wl)
    for step in range(STEPS):
        params = {}
        for o in outs:
            params.update(o[step]["before"])
        ref.load_params(params)
        masks = masks_from_taps([(r, o[step]["taps"]) for r, o in enumerate(outs)], sg, wl)
        full = make_batch(wl, step)
        rl, rg = ref.step(full, LR, masks)
        losses = [o[step]["loss"] for o in outs if o[step]["loss"] is not None]
        assert losses, "no head rank reported a loss"
        for l in losses:
            assert abs(l - rl.item()) <= 2e-2 * abs(rl.item()), (step, l, rl.item())
        checked = set()
        for r, o in enumerate(outs):
            rec = o[step]
            for k, g in rg.items():
                if k not in rec["before"]:
                    continue
                if k[1] == "table":
                    rows = full[wl.layers[k[0]].data_key].reshape(-1).unique()
                    got = (rec["before"][k][rows] - rec["after"][k][rows]) / LR
                    assert_close(got, g[rows], 2e-2, (r, step, k))
                else:
                    assert_close(rec["grads"][k], g, 2e-2, (r, step, k))
                checked.add(k)
        assert checked == set(rg), ("parameters owned by no rank", set(rg) - checked)


def _towers():
    # ops: tower 0 = 0,1,2; tower 1 = 3,4,5; concat 6; tail 7; MSE head 8
    return W.multi_tower("ms-relu", towers=2, layers=3, width=1024, in_dim=512, tail_hidden=512, B=64)


def _mmt():
    # ops: branch 0 = 0,1; branch 1 = 2,3; concat 4; CE head 5
    return W.mmt(B=8, branches=2, layers=2, S=128, d=128, H=2, ffn=256, classes=64)


def _dlrm():
    # ops: bottom MLP 0..3, tables 4..7, interaction 8, top MLP 9..11, BCE head 12
    return W.dlrm(B=64, tables=4, rows=500, bag=8, hidden=256)


@pytest.mark.parametrize("backend", BACKENDS)
def test_towers_gpp_unequal_b_and_dp2_tail(backend):
    """Towers on their own ranks with b = 16 / 32, the tail a DP-2 stage (b = 16, 8 rows
    per replica): pieces split and merge micro-batches, the DP stage all-reduces."""
    _run(backend, _towers, [([0, 1, 2], 16, [0]), ([3, 4, 5], 32, [1]), ([6, 7, 8], 16, [2, 3])])


@pytest.mark.parametrize("backend", BACKENDS)
def test_towers_sequential_chain_token_edge(backend):
    """SPP-shaped chain tower 0 -> tower 1 -> tail: the 0 -> 1 edge carries no operator
    data and is realised as ordering tokens."""
    _run(backend, _towers, [([0, 1, 2], 16, [0]), ([3, 4, 5], 16, [1]), ([6, 7, 8], 16, [2])], extra_edges=[(0, 1)])


@pytest.mark.parametrize("backend", BACKENDS)
def test_mmt_branch_stages_and_mid_branch_cut(backend):
    """MMT: branch 0 cut between its layers (the edge carries [b, S*d] activations and
    their gradients), branch 1 whole on one rank, concat + CE head on a fourth."""
    _run(backend, _mmt, [([0], 2, [0]), ([1], 2, [1]), ([2, 3], 4, [2]), ([4, 5], 2, [3])])


@pytest.mark.parametrize("backend", BACKENDS)
def test_dlrm_dp2_embedding_stage(backend):
    """DLRM: the embedding tables as a DP-2 stage (replicas all-gather indices and pooled
    gradients and apply every replica's sparse update), MLPs on their own ranks."""
    _run(backend, _dlrm, [([0, 1, 2, 3], 16, [0]), ([4, 5, 6, 7], 32, [1, 2]), ([8, 9, 10, 11, 12], 16, [3])])


def _mmt4():
    # ops: branches 0..3 (one layer each), concat 4, CE head 5
    return W.mmt(B=8, branches=4, layers=1, S=128, d=128, H=2, ffn=256, classes=64)


@pytest.mark.parametrize("backend", BACKENDS)
def test_mmt_eight_rank_branch_dp2_layout(backend):
    """The shape of the frozen MMT plan at 8 GPUs (profiles/strategies/mmt-*_gpp_n8_*): one
    stage per branch, each a DP-2 stage over two ranks, the last also holding concat + CE
    head -- eight executor ranks (sharing one GPU with the cuda backend), per-rank gradients
    vs the oracle.  The 8-GPU box itself is the driver's SCALE run."""
    _run(backend, _mmt4, [([0], 8, [0, 1]), ([1], 8, [2, 3]), ([2], 8, [4, 5]), ([3, 4, 5], 8, [6, 7])])


@pytest.mark.parametrize("backend", BACKENDS)
def test_dlrm_eight_rank_plan_layout(backend):
    """The shape of the frozen DLRM plan at 8 GPUs (profiles/strategies/dlrm-*_gpp_n8_*): the
    bottom MLP a DP-2 stage, the embedding tables split over four single-rank stages, the
    interaction + top MLP + BCE head a DP-2 stage; four micro-batches."""
    _run(backend, _dlrm, [([0, 1, 2, 3], 16, [0, 1]), ([4], 16, [2]), ([5], 16, [3]), ([6], 16, [4]), ([7], 16, [5]),
                          ([8, 9, 10, 11, 12], 16, [6, 7])])
