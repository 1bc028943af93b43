"""The executor's simulated twin (sim.simulate(op_granular=True), runtime.api.twin).

op_granular relaxes the SPEC task-level semantics exactly where the executor does
(receives waited at the consuming op, pieces shipped when final) and keeps task-level
ordering for stage edges that carry no operator data (the token messages of
runtime/executor.py).
"""

import pytest

from paper_2406_17145_b200 import model as M
from paper_2406_17145_b200 import sched as S
from paper_2406_17145_b200 import workloads as W
from paper_2406_17145_b200.runtime.api import plan, twin
from paper_2406_17145_b200.sim import simulate


def _sg(wl, layout, extra=()):
    stages = [M.Stage(i, frozenset(ops), b, frozenset(devs)) for i, (ops, b, devs) in enumerate(layout)]
    edges = set(M.induced_stage_edges(wl.graph, [s.op_ids for s in stages])) | set(extra)
    return S.schedule_stage_graph(M.StageGraph(stages, edges, wl.mini_batch))


@pytest.mark.parametrize("b", [8, 16, 32])
def test_op_granular_never_slower_than_task_granular(b):
    wl = W.toy(B=64)
    cl = W.b200_cluster(3)
    sg = _sg(wl, [([0, 1, 2, 3], b, [0]), ([4, 5, 6, 7, 8, 9, 10], b, [1])])
    t_task = simulate(sg, cl, wl.graph).iteration_ms
    t_op = simulate(sg, cl, wl.graph, op_granular=True).iteration_ms
    assert t_op <= t_task + 1e-9


def test_single_op_chain_equals_task_granular():
    g = W.chain(4)
    wl = W.Workload("chain", g, {}, {}, 8)
    sg = _sg(wl, [([i], 2, [i]) for i in range(4)])
    a = simulate(sg, W.b200_cluster(4), g)
    b = simulate(sg, W.b200_cluster(4), g, op_granular=True)
    assert a.iteration_ms == pytest.approx(b.iteration_ms)
    for k, (s0, s1) in a.task_times.items():
        assert b.task_times[k][0] == pytest.approx(s0) and b.task_times[k][1] == pytest.approx(s1)


def test_dataless_edge_orders_whole_tasks():
    """Tower B's stage follows tower A's in a chain without data: fw(B, j) may not start
    before fw(A, j) ends, bw(A, j) not before bw(B, j) ends."""
    wl = W.toy(B=64)
    sg = _sg(wl, [([0, 1, 2, 3], 16, [0]), ([4, 5, 6, 7], 16, [1]), ([8, 9, 10], 16, [2])], extra=[(0, 1)])
    rep = simulate(sg, W.b200_cluster(3), wl.graph, op_granular=True)
    tt = rep.task_times
    for j in range(4):
        assert tt[(1, "fw", j)][0] >= tt[(0, "fw", j)][1] - 1e-12
        assert tt[(0, "bw", j)][0] >= tt[(1, "bw", j)][1] - 1e-12
    free = simulate(_sg(wl, [([0, 1, 2, 3], 16, [0]), ([4, 5, 6, 7], 16, [1]), ([8, 9, 10], 16, [2])]),
                    W.b200_cluster(3), wl.graph, op_granular=True)
    assert free.iteration_ms < rep.iteration_ms


def test_mmt_gpp_beats_spp_in_twin_at_4_gpus():
    """MMT 4 branches at 4 GPUs (B = 64, measured B200 layer curves): the GPP plan runs the
    branches side by side; the sequential pipeline is chained through data-less edges."""
    wl = W.mmt(B=64)
    g = plan(wl, 4, "gpp")
    s = plan(wl, 4, "spp")
    cl = W.b200_cluster(4)
    mg = W.with_measured_curves(wl)[0].graph
    tg, ts = twin(g.stage_graph, cl, mg).iteration_ms, twin(s.stage_graph, cl, mg).iteration_ms
    assert tg < 0.8 * ts, (tg, ts)
    assert M.pipeline_depth(g.stage_graph) < M.pipeline_depth(s.stage_graph)


def test_runtime_planner_balances_candle_towers_at_4_gpus():
    """rich_splits (runtime planner only): 7 towers + tail on 4 GPUs -> 2/2/2 towers and
    1 tower + tail (the reference's one-vs-rest / halves cuts cannot form three 2-tower
    groups; the SPEC search keeps them, tests/test_spec_acceptance.py)."""
    wl = W.candle(B=4096)
    sg = plan(wl, 4, "gpp").stage_graph
    assert sorted(len(s.op_ids) for s in sg.stages) == [7, 8, 8, 8]
    mg = W.with_measured_curves(wl)[0].graph
    assert twin(sg, W.b200_cluster(4), mg).iteration_ms < 3.5


@pytest.mark.parametrize("preset", ["candle", "mmt"])
def test_rich_splits_never_worse(preset):
    from paper_2406_17145_b200 import partition as P

    wl = W.with_measured_curves(W.candle(B=2048) if preset == "candle" else W.mmt(B=32, layers=2))[0]
    cl = W.b200_cluster(4)
    base = dict(sync_per_iteration=True, micro_batches=(wl.mini_batch // 2,), merge_join=True)
    a = P.optimize(wl.graph, cl, wl.mini_batch, P.PartitionOptions(**base))
    b = P.optimize(wl.graph, cl, wl.mini_batch, P.PartitionOptions(**base, rich_splits=True))
    assert b.bottleneck_tps <= a.bottleneck_tps * (1 + 2e-3)
