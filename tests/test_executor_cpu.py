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


def _stage_graph(layout, B, wl=None, extra_edges=()):
    """layout: list of (op ids, micro_batch, devices); extra_edges: data-less stage edges."""
    wl = wl or W.toy(B=B)
    stages = [M.Stage(i, frozenset(ops), b, frozenset(devs)) for i, (ops, b, devs) in enumerate(layout)]
    part = [st.op_ids for st in stages]
    edges = set(M.induced_stage_edges(wl.graph, part)) | set(extra_edges)
    sg = S.schedule_stage_graph(M.StageGraph(stages, edges, B))
    assert M.validate_strategy(wl.graph, M.DeviceCluster(8, 1e12, 1, 1), sg) == []
    return wl, sg


def _worker(rank, world, port, layout, B, outdir, wl=None, extra_edges=()):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        wl, sg = _stage_graph(layout, B, wl, extra_edges)
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


def _run(layout, B, world, wl=None, extra_edges=()):
    with tempfile.TemporaryDirectory() as d:
        mp.spawn(_worker, args=(world, _free_port(), layout, B, d, wl, extra_edges), nprocs=world, join=True)
        outs = [torch.load(os.path.join(d, f"rank{r}.pt")) for r in range(world)]
    wl = wl or W.toy(B=B)
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


def test_sequential_chain_token_edges_gloo():
    """SPP-shaped layout: tower A -> tower B -> tail as a stage chain.  The chain edge
    A -> B carries no operator data (the towers are independent) but still orders the
    tasks, so the executor realises it with token messages; results
    still equal the reference."""
    layout = [(TOWER_A, 16, [0]), (TOWER_B, 16, [1]), (TAIL, 16, [2])]
    _run(layout, 64, 3, extra_edges=[(0, 1)])


def test_token_pieces_only_on_dataless_edges():
    wl, sg = _stage_graph([(TOWER_A, 16, [0]), (TOWER_B, 32, [1]), (TAIL, 16, [2])], 64, extra_edges=[(0, 1)])
    exs = [Executor(wl, sg, r, 3, TorchBackend(), use_dist=False) for r in range(3)]
    # stage 0 -> stage 1 (b 16 -> 32): two producer tasks feed each consumer task
    assert [len(exs[1].tok_in[j]) for j in range(2)] == [2, 2]
    assert [len(exs[0].tok_out[j]) for j in range(4)] == [1, 1, 1, 1]
    assert all(not v for v in exs[2].tok_in.values()) and all(not v for v in exs[1].tok_out.values())


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


def test_eight_rank_seven_towers_gloo():
    """The CANDLE-shaped N=8 layout: 7 tower stages + a tail stage, one rank
    each, 4 micro-batches, fp32 -> every rank's gradients and the loss vs the reference."""
    wl = W.multi_tower("towers7", 7, 2, 32, 32, 32, 64, dtype="fp32")
    layout = [(list(range(2 * t, 2 * t + 2)), 16, [t]) for t in range(7)] + [([14, 15, 16], 16, [7])]
    _run(layout, 64, 8, wl)


DLRM_LR = 1.0  # large steps on a tiny, collision-heavy table make early updates visible


def _dlrm_worker(rank, world, port, layout, B, outdir):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        wl = W.dlrm(B=B, tables=3, rows=8, bag=4, hidden=64)
        wl, sg = _stage_graph(layout, B, wl)
        ex = Executor(wl, sg, rank, world, TorchBackend(), lr=DLRM_LR)
        for step in range(STEPS):
            ex.run_iteration(to_device_rows(ex, make_batch(wl, step), torch.bfloat16, "cpu"))
        torch.save({o: t.clone() for o, t in ex.tables.items()}, os.path.join(outdir, f"rank{rank}.pt"))
    finally:
        dist.destroy_process_group()


def test_dlrm_sparse_updates_match_single_stage_gloo():
    """Two pipeline stages x 4 micro-batches apply each micro-batch's table scatter as soon
    as the stage's forwards are done; after 2 steps the tables equal a 1-stage,
    1-micro-batch run's (the same per-row contributions, exact SGD semantics)."""
    B = 32
    two = [(list(range(7)), 8, [0]), (list(range(7, 12)), 8, [1])]
    with tempfile.TemporaryDirectory() as d:
        mp.spawn(_dlrm_worker, args=(2, _free_port(), two, B, d), nprocs=2, join=True)
        multi = torch.load(os.path.join(d, "rank0.pt"))
    with tempfile.TemporaryDirectory() as d:
        mp.spawn(_dlrm_worker, args=(1, _free_port(), [(list(range(12)), 32, [0])], B, d), nprocs=1, join=True)
        single = torch.load(os.path.join(d, "rank0.pt"))
    assert sorted(multi) == sorted(single) == [4, 5, 6]
    for o in multi:
        err = ((multi[o] - single[o]).abs().max() / (single[o].abs().max() + 1e-12)).item()
        assert err < 1e-5, (o, err)  # exact in practice; an early scatter gives ~6e-3
