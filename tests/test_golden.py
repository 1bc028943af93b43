"""Bit-exact parity of the restated model/spgraph/cost against the REFERENCE's outputs.

Fixtures: tests/golden/reference_golden.json, produced by tests/golden/make_golden.py
running the shipped reference modules (/root/reference/pkg/src/gpp/{model,spgraph,cost}.py)
on 62 graphs (workload presets, SPEC example shapes, a 27-branch DLRM-like bundle,
40 random series-parallel and 10 random DAGs).  When /root/reference is present
(build container) the same comparisons also run live against the imported reference.
"""

import json
import os
import sys

import pytest

from paper_2406_17145_b200 import cost as C
from paper_2406_17145_b200 import model as M
from paper_2406_17145_b200 import spgraph as SP

HERE = os.path.dirname(os.path.abspath(__file__))
FIX = json.load(open(os.path.join(HERE, "golden", "reference_golden.json")))


def mk_curve(spec):
    if spec["kind"] == "affine":
        return M.CostCurve.affine(spec["a"], spec["b"])
    return M.CostCurve(kind="table", points=tuple(tuple(p) for p in spec["points"]))


def build(spec):
    ops = [M.Operator(o["id"], o["name"], o["param_bytes"], o["act"], o["out"], mk_curve(o["fwd"]), mk_curve(o["bwd"]))
           for o in spec["ops"]]
    return M.ComputationGraph(ops, [tuple(e) for e in spec["edges"]])


def tree_json(t):
    if isinstance(t, SP.SPLeaf):
        return ["L", t.op]
    if isinstance(t, SP.SPSeries):
        return ["S", tree_json(t.left), tree_json(t.right), t.junction]
    return ["P", [tree_json(c) for c in t.children], t.source, t.sink, t.direct_edges]


def walk(t):
    yield t
    if isinstance(t, SP.SPSeries):
        yield from walk(t.left)
        yield from walk(t.right)
    elif isinstance(t, SP.SPParallel):
        for c in t.children:
            yield from walk(c)


GRAPHS = sorted(FIX["graphs"])


def test_cost_curves_bit_exact():
    for case in FIX["curves"]:
        c = mk_curve(case["curve"])
        for n, v in case["values"]:
            assert c.evaluate(n) == v, (case["curve"], n)
        s = c.scaled(1.7)
        assert [list(p) for p in s.points] == case["scaled"]["points"]
        assert (s.a, s.b) == (case["scaled"]["a"], case["scaled"]["b"])


@pytest.mark.parametrize("name", GRAPHS)
def test_graph_and_normalize(name):
    rec = FIX["graphs"][name]
    g = build(rec["graph"])
    assert list(g.topo_order) == rec["topo"]
    assert list(g.source_ids()) == rec["sources"]
    assert list(g.sink_ids()) == rec["sinks"]
    ng = SP.normalize(g)
    n = rec["normalized"]
    assert [[o.id, o.name] for o in ng.graph.ops] == n["ops"]
    assert sorted(map(list, ng.graph.edges)) == n["edges"]
    assert sorted(ng.virtual_ids) == n["virtual"]
    assert {str(k): v for k, v in sorted(ng.effective_out_bytes.items())} == n["eff_bytes"]
    assert list(ng.graph.topo_order) == n["topo"]
    assert (sorted(map(list, SP.normalize(ng).graph.edges)) == n["edges"]) == rec["renormalize_same"]
    assert SP.linearize(g) == rec["linearize"]


@pytest.mark.parametrize("name", GRAPHS)
def test_decompose_splits_rebuild(name):
    rec = FIX["graphs"][name]
    ng = SP.normalize(build(rec["graph"]))
    if "not_sp_witness" in rec:
        with pytest.raises(SP.NotSeriesParallelError) as ei:
            SP.decompose(ng)
        assert sorted(map(list, ei.value.witness_edges)) == rec["not_sp_witness"]
        return
    tree = SP.decompose(ng)
    assert tree_json(tree) == rec["tree"]
    splits = []
    for node in walk(tree):
        if isinstance(node, SP.SPSeries):
            splits.append(["S", sorted(node.ops), [[sorted(a), sorted(b), j] for a, b, j in SP.series_splits(node)]])
        elif isinstance(node, SP.SPParallel):
            try:
                ps = [[sorted(a), sorted(b)] for a, b in SP.parallel_splits(node)]
            except ValueError as e:
                ps = ["error", str(e)]
            splits.append(["P", sorted(node.ops), ps])
    assert splits == rec["splits"]
    ops_, edges_ = SP.rebuild(tree)
    assert {"ops": sorted(ops_), "edges": sorted(map(list, edges_))} == rec["rebuild"]


@pytest.mark.parametrize("name", GRAPHS)
def test_cost_model_bit_exact(name):
    rec = FIX["graphs"][name]
    g = build(rec["graph"])
    cl = M.DeviceCluster(4, 1e9, 2e3, 1e3, 0.25)
    for ids, b, d, cin, cout, v in rec["tps"]:
        ops = tuple(g.by_id[i] for i in ids)  # same op order as the reference call
        try:
            got = C.estimate_tps(C.StageCostInput(ops, b, d, cin, cout, cl))
        except C.IndivisibleMicroBatchError:
            got = "indivisible"
        assert got == v  # bit-exact
    for ids, d, inf, wm, wb, ab, tot in rec["memory"]:
        m = C.stage_memory([g.by_id[i] for i in ids], d, inf, wm)
        assert (m.weight_bytes, m.activation_bytes, m.total) == (wb, ab, tot)


@pytest.mark.parametrize("name", GRAPHS)
def test_validation_and_depth(name):
    rec = FIX["graphs"][name]
    g = build(rec["graph"])
    cl = M.DeviceCluster(4, 1e9, 2e3, 1e3, 0.25)
    for st in rec["strategies"]:
        stages = [M.Stage(s["id"], frozenset(s["ops"]), s["b"], frozenset(s["devices"]), None,
                          None if s["schedule"] is None else tuple(M.Task(d, j) for d, j in s["schedule"]))
                  for s in st["stages"]]
        sg = M.StageGraph(stages, [tuple(e) for e in st["edges"]], st["B"])
        induced = M.induced_stage_edges(g, [frozenset(s["ops"]) for s in st["stages"]])
        assert sorted(map(list, induced)) == st["induced"]
        rep = M.validate_strategy(g, cl, sg)
        assert [[v.code, v.message, list(v.subjects)] for v in rep] == st["report"]
        try:
            depth = M.pipeline_depth(sg)
        except M.GraphCycleError:
            depth = "cycle"
        assert depth == st["depth"]


def test_spec_examples():
    ex = FIX["spec_examples"]
    op = M.Operator(0, "a", fwd_cost=M.CostCurve.affine(0, 1), bwd_cost=M.CostCurve.affine(0, 2))
    assert C.estimate_tps(C.StageCostInput((op,), 4, 1, 0.0, 0.0, M.DeviceCluster(1, 1e9, 1.0, 1.0))) == ex["tps_affine"] == 3.0
    assert C.comm_time(1000, 2, 1000, 0.0) == ex["comm"] == 2.0


REF = "/root/reference/pkg/src"


@pytest.mark.skipif(not os.path.isdir(REF), reason="reference not present (GPU box)")
def test_live_against_reference_random_sp():
    """Hypothesis-style sweep against the live reference import (build container only)."""
    import random

    # the repo's own `gpp` drop-in namespace (gpp/*.py aliases) shadows the reference's:
    # import the reference's modules with only the reference on the path, then restore
    saved = {k: sys.modules.pop(k) for k in list(sys.modules) if k == "gpp" or k.startswith("gpp.")}
    old_path = sys.path[:]
    sys.path[:] = [REF, HERE] + [p for p in old_path if os.path.abspath(p or ".") != os.path.dirname(HERE)
                                 and p not in ("", ".")]
    try:
        from gpp import model as rm
        from gpp import spgraph as rs
        assert rm.__file__.startswith(REF), rm.__file__
        sys.modules.pop("golden.make_golden", None)
        import golden.make_golden as mg  # binds the reference modules too
    finally:
        sys.path[:] = old_path
        for k in [k for k in sys.modules if k == "gpp" or k.startswith("gpp.")]:
            del sys.modules[k]
        sys.modules.update(saved)

    rng = random.Random(7)
    for _ in range(150):
        k = rng.randint(1, 10)
        edges = mg.rand_sp_edges(rng, k) if rng.random() < 0.8 else mg.rand_dag_edges(rng, k)
        mine = M.ComputationGraph([M.Operator(i, f"o{i}", out_bytes_per_sample=float(i + 1)) for i in range(k)], edges)
        ref = rm.ComputationGraph([rm.Operator(i, f"o{i}", out_bytes_per_sample=float(i + 1)) for i in range(k)], edges)
        a, b = SP.normalize(mine), rs.normalize(ref)
        assert sorted(a.graph.edges) == sorted(b.graph.edges)
        assert a.effective_out_bytes == b.effective_out_bytes
        try:
            tb = rs.decompose(b)
        except rs.NotSeriesParallelError as e:
            with pytest.raises(SP.NotSeriesParallelError) as ei:
                SP.decompose(a)
            assert ei.value.witness_edges == e.witness_edges
            continue
        assert tree_json(SP.decompose(a)) == mg.tree_json(tb)
