"""Executor host logic on CPU: ring slots, piece routing, DP re-shard, all-reduce.

The executor runs with the torch-CPU kernel backend (oracle/torch_backend.py)
over gloo with world_size 2 and 4, and every rank's gradients plus the loss are
compared with the monolithic reference model (oracle/reference_model.py).
fp32 toy workload (BASELINE configs[0]) -> rtol 1e-4 (north_star).
"""

import os
import socket
import tempfile

import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from paper_2406_17145_b200 import model as M
from paper_2406_17145_b200 import sched as S
from paper_2406_17145_b200 import workloads as W
from paper_2406_17145_b200.runtime.data import make_batch, to_device_rows
from paper_2406_17145_b200.runtime.executor import Executor, build_pieces

from oracle.reference_model import ReferenceModel
from oracle.torch_backend import TorchBackend

LR = 0.05
STEPS = 2


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _stage_graph(layout, B):
    """layout: list of (op ids, micro_batch, devices)."""
    wl = W.toy(B=B)
    stages = [M.Stage(i, frozenset(ops), b, frozenset(devs)) for i, (ops, b, devs) in enumerate(layout)]
    part = [st.op_ids for st in stages]
    edges = M.induced_stage_edges(wl.graph, part)
    sg = S.schedule_stage_graph(M.StageGraph(stages, edges, B))
    assert M.validate_strategy(wl.graph, M.DeviceCluster(8, 1e12, 1, 1), sg) == []
    return wl, sg


def _worker(rank, world, port, layout, B, outdir):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        wl, sg = _stage_graph(layout, B)
        ex = Executor(wl, sg, rank, world, TorchBackend(), lr=LR, keep_grads=True)
        res = {"loss": [], "grads": []}
        for step in range(STEPS):
            full = make_batch(wl, step)
            batch = to_device_rows(ex, full, torch.float32, "cpu")
            loss = ex.run_iteration(batch)
            if ex.is_head:
                res["loss"].append(ex.stage_loss(loss))
            res["grads"].append({k: v.clone() for k, v in ex.G.items()})
        torch.save(res, os.path.join(outdir, f"rank{rank}.pt"))
    finally:
        dist.destroy_process_group()


def _run(layout, B, world):
    with tempfile.TemporaryDirectory() as d:
        mp.spawn(_worker, args=(world, _free_port(), layout, B, d), nprocs=world, join=True)
        outs = [torch.load(os.path.join(d, f"rank{r}.pt")) for r in range(world)]
    wl = W.toy(B=B)
    ref = ReferenceModel(wl)
    for step in range(STEPS):
        rl, rg = ref.step(make_batch(wl, step), LR)
        losses = [o["loss"][step] for o in outs if o["loss"]]
        assert losses, "no head rank reported a loss"
        for l in losses:
            assert abs(l - rl.item()) <= 1e-4 * abs(rl.item())
        for o in outs:
            for k, g in o["grads"][step].items():
                err = ((g - rg[k]).abs().max() / (rg[k].abs().max() + 1e-12)).item()
                assert err < 1e-4, (k, err)


TOWER_A, TOWER_B, TAIL = [0, 1, 2, 3], [4, 5, 6, 7], [8, 9, 10]


def test_two_stage_gpp_gloo():
    _run([(TOWER_A, 16, [0]), (TOWER_B + TAIL, 16, [1])], 64, 2)


def test_unequal_microbatch_and_dp_gloo():
    # tower A b=16 on rank 0; tower B b=32 as a DP-2 stage; tail b=8 on rank 3
    _run([(TOWER_A, 16, [0]), (TOWER_B, 32, [1, 2]), (TAIL, 8, [3])], 64, 4)


def test_single_rank_matches_reference():
    wl, sg = _stage_graph([(TOWER_A + TOWER_B + TAIL, 16, [0])], 64)
    ex = Executor(wl, sg, 0, 1, TorchBackend(), lr=LR, keep_grads=True)
    ref = ReferenceModel(wl)
    for step in range(STEPS):
        full = make_batch(wl, step)
        loss = ex.run_iteration(to_device_rows(ex, full, torch.float32, "cpu"))
        rl, rg = ref.step(full, LR)
        assert abs(loss.item() - rl.item()) <= 1e-5 * abs(rl.item())
        for k, g in rg.items():
            assert ((ex.G[k] - g).abs().max() / (g.abs().max() + 1e-12)).item() < 1e-4


def test_pieces_cover_every_sample_once():
    p = M.Stage(0, frozenset({0}), 16, frozenset({0, 1}))
    c = M.Stage(1, frozenset({1}), 8, frozenset({2, 3, 4, 5}))
    pcs = build_pieces(p, c, [0], 64)
    covered = sorted((pc.start, pc.rows) for pc in pcs)
    pos = 0
    for s, r in covered:
        assert s == pos
        pos += r
    assert pos == 64
