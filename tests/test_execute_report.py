"""runtime.api.execute: the SimReport fields measured, the Chrome trace, and trace_diff.

The CPU tests exercise the trace utilities on a simulated report; the GPU test runs
execute(trace=True) on cuda:0 and checks the report against the simulator's twin."""

import json

import pytest
import torch

from paper_2406_17145_b200 import model as M
from paper_2406_17145_b200 import sched as S
from paper_2406_17145_b200 import sim as SIM
from paper_2406_17145_b200 import workloads as W
from paper_2406_17145_b200.runtime.trace import emit_measured_trace, stage_summary, trace_diff


def _two_stage():
    wl = W.multi_tower("t", towers=2, layers=2, width=256, in_dim=256, tail_hidden=128, B=64)
    stages = [M.Stage(0, frozenset({0, 1, 2, 3}), 16, frozenset({0})), M.Stage(1, frozenset({4, 5, 6}), 16, frozenset({1}))]
    sg = S.schedule_stage_graph(M.StageGraph(stages, M.induced_stage_edges(wl.graph, [s.op_ids for s in stages]), 64))
    return wl, sg


def test_trace_schema_matches_the_simulator_and_diff_is_exact_on_its_own_times():
    wl, sg = _two_stage()
    cl = W.b200_cluster(2)
    rep = SIM.simulate(sg, cl, wl.graph)
    # a "measurement" equal to the simulation: every task as simulated, busy = duration
    by_rank = {}
    for (sid, d, j), (t0, t1) in rep.task_times.items():
        by_rank.setdefault(sid, {})[(sid, d, j)] = (t0, t1, t1 - t0)
    doc = json.loads(emit_measured_trace(by_rank))
    sim_doc = json.loads(SIM.emit_trace(rep))
    keys = {"name", "cat", "ph", "ts", "dur", "pid", "tid"}
    assert all(keys <= set(e) for e in doc["traceEvents"]) and all(keys <= set(e) for e in sim_doc["traceEvents"])
    assert sorted((e["name"], e["tid"]) for e in doc["traceEvents"]) == sorted((e["name"], e["tid"]) for e in sim_doc["traceEvents"])
    diff = trace_diff(by_rank, rep)
    assert diff["order_equal"] and diff["tasks_compared"] == len(rep.task_times)
    assert diff["start_rank_corr"] == pytest.approx(1.0)
    summ = stage_summary(by_rank, {0: 0, 1: 1}, rep.iteration_ms)
    for sid in (0, 1):
        assert summ["busy_ms"][sid] == pytest.approx(rep.busy_ms[sid])


def test_trace_diff_flags_a_reordered_stage():
    wl, sg = _two_stage()
    rep = SIM.simulate(sg, W.b200_cluster(2), wl.graph)
    by_rank = {}
    for (sid, d, j), (t0, t1) in rep.task_times.items():
        by_rank.setdefault(sid, {})[(sid, d, j)] = (t0, t1, t1 - t0)
    k = sorted(by_rank[0], key=lambda t: by_rank[0][t][0])
    a, b = k[0], k[1]
    by_rank[0][a], by_rank[0][b] = by_rank[0][b], by_rank[0][a]
    assert not trace_diff(by_rank, rep)["order_equal"]


@pytest.mark.gpu
def test_execute_reports_simreport_fields_and_a_trace(cuda_lib):
    from paper_2406_17145_b200.runtime.api import execute, twin

    wl = W.multi_tower("t", towers=2, layers=2, width=256, in_dim=256, tail_hidden=128, B=64)
    sg = S.schedule_stage_graph(M.StageGraph([M.Stage(0, wl.graph.op_ids, 16, frozenset({0}))], [], 64))
    cl = W.b200_cluster(1)
    rep = execute(sg, cl, wl, iters=3, trace=True)
    sim = SIM.simulate(sg, cl, wl.graph)
    assert rep.peak_inflight_samples == sim.peak_inflight_samples
    assert rep.warm_up_microbatches == sim.warm_up_microbatches and rep.depth == sim.depth
    assert len(rep.losses) == 3 and all(l == l for l in rep.losses)
    assert rep.samples_per_s > 0 and rep.h2d_bytes_per_step > 0 and rep.d2h_bytes_per_step == 4
    assert 0 < rep.busy_ms[0] <= rep.iteration_ms * 1.05 and rep.bubble_fraction is not None
    doc = json.loads(rep.trace)
    names = {e["name"] for e in doc["traceEvents"]}
    assert {f"fw{j}" for j in range(4)} <= names and {f"bw{j}" for j in range(4)} <= names
    diff = trace_diff(rep.task_times, twin(sg, cl, wl.graph))
    assert diff["order_equal"] and diff["tasks_compared"] == 8
    # graph replay trains exactly like eager execution (warm-up iterations undone)
    eager = execute(sg, cl, wl, iters=3, graph=False)
    assert eager.losses == pytest.approx(rep.losses, rel=1e-6)
