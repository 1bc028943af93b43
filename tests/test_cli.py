"""CLI + file formats: round trips, strict parsing, exit codes,
byte-determinism, and the compare command on the SPEC's pinned workloads."""

import json

import pytest

from paper_2406_17145_b200 import cli
from paper_2406_17145_b200 import model as M
from paper_2406_17145_b200 import partition as P
from paper_2406_17145_b200 import sim as SIM
from paper_2406_17145_b200 import workloads as W


def _run(argv, capsys):
    rc = cli.main(argv)
    cap = capsys.readouterr()
    return rc, cap.out, cap.err


@pytest.mark.parametrize("preset", ["fig2", "case-study", "candle-uno", "toy", "chain"])
def test_graph_and_cluster_round_trip(preset, tmp_path, capsys):
    g, cl = cli._presets(preset, None)
    text = cli.dumps(cli.graph_to_json(g))
    g2 = cli.graph_from_json(json.loads(text))
    assert cli.dumps(cli.graph_to_json(g2)) == text
    assert sorted(g2.edges) == sorted(g.edges) and [o.id for o in g2.ops] == [o.id for o in g.ops]
    for n in (0, 1, 3, 64, 1024):
        for a, b in zip(sorted(g.ops, key=lambda o: o.id), sorted(g2.ops, key=lambda o: o.id)):
            assert a.fwd_cost.evaluate(n) == b.fwd_cost.evaluate(n)
    ctext = cli.dumps(cli.cluster_to_json(cl))
    assert cli.dumps(cli.cluster_to_json(cli.cluster_from_json(json.loads(ctext)))) == ctext


def test_strategy_round_trip_and_resimulation(tmp_path, capsys):
    g, cl = W.fig2(), M.DeviceCluster(4, 1e12, 1e3, 1e9)
    st = P.optimize(g, cl, 8)
    text = cli.dumps(cli.strategy_to_json(st.stage_graph, g))
    sg2, g2, simo = cli.strategy_from_json(json.loads(text))
    assert cli.dumps(cli.strategy_to_json(sg2, g2, **simo)) == text
    assert SIM.simulate(sg2, cl, g2).iteration_ms == SIM.simulate(st.stage_graph, cl, g).iteration_ms


def test_unknown_fields_and_versions_rejected():
    g = cli.graph_to_json(W.fig2())
    with pytest.raises(cli.FormatError):
        cli.graph_from_json({**g, "extra": 1})
    with pytest.raises(cli.FormatError):
        cli.graph_from_json({**g, "format_version": 2})
    with pytest.raises(cli.FormatError):
        cli.cluster_from_json(cli.graph_to_json(W.fig2()))  # wrong kind
    bad = json.loads(json.dumps(g))
    bad["ops"][0]["fwd_cost"]["c"] = 0
    with pytest.raises(cli.FormatError):
        cli.graph_from_json(bad)


def test_optimize_simulate_validate_end_to_end(tmp_path, capsys):
    gf, cf, sf = tmp_path / "g.json", tmp_path / "c.json", tmp_path / "s.json"
    assert _run(["gen", "--preset", "fig2", "--out", str(gf), "--cluster-out", str(cf)], capsys)[0] == 0
    rc, _, err = _run(["optimize", "--graph", str(gf), "--cluster", str(cf), "--mini-batch", "8", "--out", str(sf)], capsys)
    assert rc == 0
    summary = json.loads(err.strip().splitlines()[-1])
    assert summary["depth"] == 2 and summary["search"]["dp_states"] > 0 and summary["search"]["probes"] > 0
    first = sf.read_text()
    # re-simulates to the summary's numbers exactly and re-validates
    rc, out, _ = _run(["simulate", "--strategy", str(sf), "--cluster", str(cf), "--trace", str(tmp_path / "t.json"),
                       "--gantt", str(tmp_path / "t.svg")], capsys)
    assert rc == 0 and json.loads(out)["iteration_ms"] == summary["iteration_ms"]
    rc, out, _ = _run(["validate", "--strategy", str(sf), "--cluster", str(cf)], capsys)
    assert rc == 0 and json.loads(out) == {"violations": []}
    # byte-determinism of strategy, trace and gantt
    trace, svg = (tmp_path / "t.json").read_text(), (tmp_path / "t.svg").read_text()
    _run(["optimize", "--graph", str(gf), "--cluster", str(cf), "--mini-batch", "8", "--out", str(sf)], capsys)
    _run(["simulate", "--strategy", str(sf), "--cluster", str(cf), "--trace", str(tmp_path / "t.json"),
          "--gantt", str(tmp_path / "t.svg")], capsys)
    assert sf.read_text() == first
    assert (tmp_path / "t.json").read_text() == trace and (tmp_path / "t.svg").read_text() == svg
    assert svg.startswith("<svg") and svg.count("<rect") == len(json.loads(trace)["traceEvents"])


def test_compare_fig2_case_study_chain(tmp_path, capsys):
    for preset, B, check in [
        ("fig2", 8, lambda r: (r["gpp"]["depth"], r["spp"]["depth"], r["gpp"]["warm_up_microbatches"],
                               r["spp"]["warm_up_microbatches"]) == (2, 4, 2, 4) and r["iteration_ratio_gpp_over_spp"] < 1),
        ("case-study", W.CASE_STUDY_B, lambda r: 0.78 <= r["iteration_ratio_gpp_over_spp"] <= 0.88
         and (r["gpp"]["depth"], r["spp"]["depth"]) == (4, 8)),
        ("chain", 8, lambda r: abs(r["iteration_ratio_gpp_over_spp"] - 1.0) < 1e-9),
    ]:
        gf, cf = tmp_path / f"{preset}.json", tmp_path / f"{preset}_c.json"
        _run(["gen", "--preset", preset, "--out", str(gf), "--cluster-out", str(cf)], capsys)
        rc, out, _ = _run(["compare", "--graph", str(gf), "--cluster", str(cf), "--mini-batch", str(B)], capsys)
        assert rc == 0 and check(json.loads(out)), (preset, out)


def test_exit_codes(tmp_path, capsys):
    cf = tmp_path / "c.json"
    cf.write_text(cli.dumps(cli.cluster_to_json(M.DeviceCluster(2, 1e12, 1e3, 1e9))))
    # 2: parse error
    (tmp_path / "bad.json").write_text("{not json")
    assert _run(["optimize", "--graph", str(tmp_path / "bad.json"), "--cluster", str(cf), "--mini-batch", "4"], capsys)[0] == 2
    # 3: not series-parallel (Wheatstone bridge), witness printed
    unit = lambda i: M.Operator(i, f"u{i}", 1.0, 1.0, 1.0, M.CostCurve.affine(0, 1), M.CostCurve.affine(0, 1))
    ws = M.ComputationGraph([unit(i) for i in range(4)], [(0, 1), (0, 2), (1, 2), (1, 3), (2, 3)])
    (tmp_path / "ws.json").write_text(cli.dumps(cli.graph_to_json(ws)))
    rc, _, err = _run(["optimize", "--graph", str(tmp_path / "ws.json"), "--cluster", str(cf), "--mini-batch", "4"], capsys)
    assert rc == 3 and "witness" in err
    # 4: no feasible strategy (weights do not fit any device)
    big = M.ComputationGraph([M.Operator(0, "w", 1e9, 1.0, 1.0, M.CostCurve.affine(0, 1), M.CostCurve.affine(0, 1))], [])
    (tmp_path / "big.json").write_text(cli.dumps(cli.graph_to_json(big)))
    small = tmp_path / "small.json"
    small.write_text(cli.dumps(cli.cluster_to_json(M.DeviceCluster(2, 1e6, 1e3, 1e9))))
    assert _run(["optimize", "--graph", str(tmp_path / "big.json"), "--cluster", str(small), "--mini-batch", "4"], capsys)[0] == 4
    # 5: deadlock (a stage whose schedule runs every backward before any forward)
    g = W.chain(2)
    stages = [M.Stage(0, frozenset({0}), 1, frozenset({0}), M.ScheduleConfig(1, 1, 1),
                      (M.Task("bw", 0), M.Task("fw", 0))),
              M.Stage(1, frozenset({1}), 1, frozenset({1}), M.ScheduleConfig(1, 1, 1),
                      (M.Task("fw", 0), M.Task("bw", 0)))]
    sg = M.StageGraph(stages, [(0, 1)], 1)
    sf = tmp_path / "dead.json"
    sf.write_text(cli.dumps(cli.strategy_to_json(sg, g)))
    assert _run(["simulate", "--strategy", str(sf), "--cluster", str(cf)], capsys)[0] == 5
    # invalid strategy -> validate exits 1 with violations listed
    rc, out, _ = _run(["validate", "--strategy", str(sf), "--cluster", str(cf)], capsys)
    assert rc == 1 and json.loads(out)["violations"]


def test_gen_branches_topology(capsys):
    g16, _ = cli._presets("candle-uno", 16)
    assert len(g16.ops) == 16 * 4 + 3
    trace = SIM.emit_trace(SIM.simulate(P.optimize(W.chain(1), M.DeviceCluster(1, 1e12, 1e3, 1e9), 1).stage_graph,
                                        M.DeviceCluster(1, 1e12, 1e3, 1e9), W.chain(1)))
    assert len(json.loads(trace)["traceEvents"]) == 2  # 1-stage 1-task run -> fw + bw
