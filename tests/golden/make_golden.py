"""Generate golden vectors from the SHIPPED reference modules (run in the build container).

    PYTHONPATH=/root/reference/pkg/src python tests/golden/make_golden.py

Imports the reference's own ``gpp.model``, ``gpp.spgraph`` and ``gpp.cost``
(pure Python, stdlib only — /root/reference/pkg/pyproject.toml:9) and records
their outputs on the workload graphs plus seeded random graphs.  The fixtures
pin this repo's restatement bit-for-bit (tests/test_golden.py); the GPU box
never reads /root/reference.
"""

from __future__ import annotations

import json
import os
import random
import zlib
import sys

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(os.path.dirname(HERE))
sys.path.insert(0, "/root/reference/pkg/src")
sys.path.insert(0, ROOT)

from gpp import cost as rcost  # noqa: E402  (the reference)
from gpp import model as rmodel  # noqa: E402
from gpp import spgraph as rsp  # noqa: E402


# --------------------------------------------------------------------------- graphs
def curve_spec(c):
    return {"kind": c.kind, "a": c.a, "b": c.b, "points": [list(p) for p in c.points]}


def mk_curve(spec):
    if spec["kind"] == "affine":
        return rmodel.CostCurve.affine(spec["a"], spec["b"])
    return rmodel.CostCurve(kind="table", points=tuple(tuple(p) for p in spec["points"]))


def graph_spec(ops, edges):
    return {
        "ops": [
            {"id": o.id, "name": o.name, "param_bytes": o.param_bytes, "act": o.act_bytes_per_sample,
             "out": o.out_bytes_per_sample, "fwd": curve_spec(o.fwd_cost), "bwd": curve_spec(o.bwd_cost)}
            for o in ops
        ],
        "edges": sorted([list(e) for e in edges]),
    }


def build_graph(spec):
    ops = [rmodel.Operator(o["id"], o["name"], o["param_bytes"], o["act"], o["out"], mk_curve(o["fwd"]), mk_curve(o["bwd"]))
           for o in spec["ops"]]
    return rmodel.ComputationGraph(ops, [tuple(e) for e in spec["edges"]])


def rand_curve(rng):
    if rng.random() < 0.5:
        return rmodel.CostCurve.affine(round(rng.uniform(0, 2), 3), round(rng.uniform(0, 3), 3))
    keys = sorted(rng.sample([1, 2, 4, 8, 16], rng.randint(1, 4)))
    v = 0.0
    pts = {}
    for k in keys:
        v += round(rng.uniform(0.1, 3.0), 3)
        pts[k] = v
    return rmodel.CostCurve.table(pts)


def rand_op(rng, i):
    return rmodel.Operator(i, f"op{i}", round(rng.uniform(0, 1e6), 1), round(rng.uniform(0, 1e5), 1),
                           round(rng.uniform(0, 1e5), 1), rand_curve(rng), rand_curve(rng))


def rand_sp_edges(rng, n):
    """Random two-terminal SP graph over n ops (ids shuffled), edges as pairs."""
    ids = list(range(n))
    rng.shuffle(ids)

    def comp(nodes):
        if len(nodes) == 1:
            return nodes[0], nodes[0], []
        if len(nodes) == 2 or rng.random() < 0.5:
            k = rng.randint(1, len(nodes) - 1)
            s1, t1, e1 = comp(nodes[:k])
            s2, t2, e2 = comp(nodes[k:])
            return s1, t2, e1 + e2 + [(t1, s2)]
        # parallel between a fresh source and sink
        src, snk, mid = nodes[0], nodes[-1], nodes[1:-1]
        if not mid:
            return src, snk, [(src, snk)]
        k = rng.randint(1, len(mid))
        parts = []
        rest = mid
        while rest:
            c = rng.randint(1, len(rest))
            parts.append(rest[:c])
            rest = rest[c:]
        edges = []
        for p in parts:
            s, t, e = comp(p)
            edges += e + [(src, s), (t, snk)]
        return src, snk, edges

    _, _, edges = comp(ids)
    return sorted(set(edges))


def rand_dag_edges(rng, n, p=0.35):
    return sorted({(i, j) for i in range(n) for j in range(i + 1, n) if rng.random() < p})


def workload_graphs():
    from paper_2406_17145_b200 import workloads as W  # graph generators only (no reference code)

    out = {}
    for name, g in [("fig2", W.fig2()), ("chain6", W.chain(6)), ("case_study", W.case_study()),
                    ("toy", W.toy().graph), ("candle", W.candle().graph)]:
        ops = [rmodel.Operator(o.id, o.name, o.param_bytes, o.act_bytes_per_sample, o.out_bytes_per_sample,
                               mk_curve(curve_spec(o.fwd_cost)), mk_curve(curve_spec(o.bwd_cost))) for o in g.ops]
        out[name] = graph_spec(ops, g.edges)
    return out


def fixed_graphs():
    def unit(i):
        return rmodel.Operator(i, f"u{i}", 10.0 * i, 3.0 + i, 4.0 + i,
                               rmodel.CostCurve.affine(0.5, 1.0), rmodel.CostCurve.table({1: 2.0, 4: 5.0}))
    g = {}
    g["diamond"] = graph_spec([unit(i) for i in range(4)], [(0, 1), (0, 2), (1, 3), (2, 3)])
    g["three_branch"] = graph_spec([unit(i) for i in range(5)], [(0, 1), (0, 2), (0, 3), (1, 4), (2, 4), (3, 4)])
    g["skip"] = graph_spec([unit(i) for i in range(4)], [(0, 1), (1, 2), (2, 3), (0, 3)])
    g["multi_source"] = graph_spec([unit(i) for i in range(5)], [(0, 2), (1, 2), (2, 3), (2, 4)])
    g["wheatstone"] = graph_spec([unit(i) for i in range(4)], [(0, 1), (0, 2), (1, 2), (1, 3), (2, 3)])
    g["single"] = graph_spec([unit(0)], [])
    br = 27
    ops = [unit(i) for i in range(br + 2)]
    g["dlrm27"] = graph_spec(ops, [(i, br) for i in range(br)] + [(br, br + 1)])
    return g


# --------------------------------------------------------------------------- records
def tree_json(t):
    if isinstance(t, rsp.SPLeaf):
        return ["L", t.op]
    if isinstance(t, rsp.SPSeries):
        return ["S", tree_json(t.left), tree_json(t.right), t.junction]
    return ["P", [tree_json(c) for c in t.children], t.source, t.sink, t.direct_edges]


def walk(t):
    yield t
    if isinstance(t, rsp.SPSeries):
        yield from walk(t.left)
        yield from walk(t.right)
    elif isinstance(t, rsp.SPParallel):
        for c in t.children:
            yield from walk(c)


def record_graph(spec, rng):
    g = build_graph(spec)
    rec = {"graph": spec, "topo": list(g.topo_order), "sources": list(g.source_ids()), "sinks": list(g.sink_ids())}
    ng = rsp.normalize(g)
    rec["normalized"] = {
        "ops": [[o.id, o.name] for o in ng.graph.ops],
        "edges": sorted([list(e) for e in ng.graph.edges]),
        "virtual": sorted(ng.virtual_ids),
        "eff_bytes": {str(k): v for k, v in sorted(ng.effective_out_bytes.items())},
        "topo": list(ng.graph.topo_order),
    }
    rec["renormalize_same"] = sorted(map(list, rsp.normalize(ng).graph.edges)) == rec["normalized"]["edges"]
    try:
        tree = rsp.decompose(ng)
        rec["tree"] = tree_json(tree)
        splits = []
        for node in walk(tree):
            if isinstance(node, rsp.SPSeries):
                splits.append(["S", sorted(node.ops), [[sorted(a), sorted(b), j] for a, b, j in rsp.series_splits(node)]])
            elif isinstance(node, rsp.SPParallel):
                try:
                    ps = [[sorted(a), sorted(b)] for a, b in rsp.parallel_splits(node)]
                except ValueError as e:
                    ps = ["error", str(e)]
                splits.append(["P", sorted(node.ops), ps])
        rec["splits"] = splits
        ops_, edges_ = rsp.rebuild(tree)
        rec["rebuild"] = {"ops": sorted(ops_), "edges": sorted(map(list, edges_))}
    except rsp.NotSeriesParallelError as e:
        rec["not_sp_witness"] = sorted(map(list, e.witness_edges))
    rec["linearize"] = rsp.linearize(g)
    # cost model on random op subsets
    cl = rmodel.DeviceCluster(4, 1e9, 2e3, 1e3, 0.25)
    ops = list(g.ops)
    tps = []
    for _ in range(12):
        sub = rng.sample(ops, rng.randint(1, len(ops)))
        b = rng.choice([1, 2, 3, 4, 8, 16])
        d = rng.choice([1, 2, 4])
        cin = rng.choice([0.0, 100.0, 12345.5])
        cout = rng.choice([0.0, 50.0])
        ids = [o.id for o in sub]  # evaluation order matters for bit-exact float sums
        try:
            v = rcost.estimate_tps(rcost.StageCostInput(tuple(sub), b, d, cin, cout, cl))
            tps.append([ids, b, d, cin, cout, v])
        except rcost.IndivisibleMicroBatchError:
            tps.append([ids, b, d, cin, cout, "indivisible"])
    rec["tps"] = tps
    mem = []
    for _ in range(6):
        sub = rng.sample(ops, rng.randint(1, len(ops)))
        d = rng.choice([1, 2, 4])
        inf = rng.randint(0, 16)
        wm = rng.choice([1.0, 2.0, 3.5])
        m = rcost.stage_memory(sub, d, inf, wm)
        mem.append([[o.id for o in sub], d, inf, wm, m.weight_bytes, m.activation_bytes, m.total])
    rec["memory"] = mem
    # strategies: random partitions of the original op set into blocks in topo order
    strategies = []
    topo = list(g.topo_order)
    for _ in range(4):
        cuts = sorted(rng.sample(range(1, len(topo)), min(len(topo) - 1, rng.randint(0, 3)))) if len(topo) > 1 else []
        blocks, prev = [], 0
        for c in cuts + [len(topo)]:
            blocks.append(topo[prev:c])
            prev = c
        if rng.random() < 0.3 and len(topo) > 2:  # a non-convex block
            blocks = [[topo[0], topo[-1]], topo[1:-1]]
        induced = rmodel.induced_stage_edges(g, [frozenset(b) for b in blocks])
        stages = []
        for i, b in enumerate(blocks):
            mb = rng.choice([1, 2, 3, 4])
            sched = None
            if rng.random() < 0.7:
                n = 8 // mb if 8 % mb == 0 else 2
                seq = [rmodel.Task("fw", j) for j in range(n)] + [rmodel.Task("bw", j) for j in range(n)]
                if rng.random() < 0.3:
                    seq = seq[::-1]
                sched = tuple(seq)
            stages.append(rmodel.Stage(i, frozenset(b), mb, frozenset({i if rng.random() < 0.8 else 0}), None, sched))
        edges = set(induced)
        if rng.random() < 0.3 and edges:
            edges.discard(sorted(edges)[0])
        sgr = rmodel.StageGraph(stages, edges, 8)
        rep = rmodel.validate_strategy(g, cl, sgr)
        try:
            depth = rmodel.pipeline_depth(sgr)
        except rmodel.GraphCycleError:
            depth = "cycle"
        strategies.append({
            "stages": [{"id": s.id, "ops": sorted(s.op_ids), "b": s.micro_batch, "devices": sorted(s.devices),
                        "schedule": None if s.schedule is None else [[t.direction, t.index] for t in s.schedule]}
                       for s in stages],
            "edges": sorted(map(list, edges)), "B": 8,
            "induced": sorted(map(list, induced)),
            "report": [[v.code, v.message, list(v.subjects)] for v in rep],
            "depth": depth,
        })
    rec["strategies"] = strategies
    return rec


def curve_cases(rng):
    out = []
    curves = [rmodel.CostCurve.affine(0.0, 1.0), rmodel.CostCurve.affine(2.5, 0.125),
              rmodel.CostCurve.table({4: 3.0}), rmodel.CostCurve.table({1: 2.0, 2: 3.0}),
              rmodel.CostCurve.table({1: 5.0, 2: 1.0}), rmodel.CostCurve.table({1: 0.3, 4: 0.9, 16: 2.1, 64: 6.0})]
    for _ in range(10):
        curves.append(rand_curve(rng))
    for c in curves:
        pts = [0, 0.5, 1, 1.5, 2, 3, 4, 7, 16, 33, 64, 100]
        out.append({"curve": curve_spec(c), "values": [[n, c.evaluate(n)] for n in pts],
                    "scaled": curve_spec(c.scaled(1.7))})
    return out


def main():
    rng = random.Random(20240617)
    fixtures = {"curves": curve_cases(rng), "graphs": {}}
    specs = dict(workload_graphs())
    specs.update(fixed_graphs())
    for n in range(40):
        k = rng.randint(2, 9)
        ops = [rand_op(rng, i) for i in range(k)]
        specs[f"rand_sp_{n}"] = graph_spec(ops, rand_sp_edges(rng, k))
    for n in range(10):
        k = rng.randint(3, 7)
        ops = [rand_op(rng, i) for i in range(k)]
        specs[f"rand_dag_{n}"] = graph_spec(ops, rand_dag_edges(rng, k))
    for name, spec in specs.items():
        fixtures["graphs"][name] = record_graph(spec, random.Random(zlib.crc32(name.encode())))
    # spec examples verified at survey time
    fixtures["spec_examples"] = {
        "tps_affine": rcost.estimate_tps(rcost.StageCostInput(
            (rmodel.Operator(0, "a", fwd_cost=rmodel.CostCurve.affine(0, 1), bwd_cost=rmodel.CostCurve.affine(0, 2)),),
            4, 1, 0.0, 0.0, rmodel.DeviceCluster(1, 1e9, 1.0, 1.0))),
        "comm": rcost.comm_time(1000, 2, 1000, 0.0),
    }
    path = os.path.join(HERE, "reference_golden.json")
    with open(path, "w") as f:
        json.dump(fixtures, f, sort_keys=True, separators=(",", ":"))
    print(path, os.path.getsize(path), "bytes,", len(fixtures["graphs"]), "graphs")


if __name__ == "__main__":
    main()
