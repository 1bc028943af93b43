"""Command-line surface, on-disk formats and report emission.

    python -m paper_2406_17145_b200.cli gen --preset fig2 --out g.json --cluster-out c.json
    python -m paper_2406_17145_b200.cli optimize --graph g.json --cluster c.json --mini-batch 8 --out s.json
    python -m paper_2406_17145_b200.cli simulate --strategy s.json --cluster c.json --trace t.json --gantt t.svg
    python -m paper_2406_17145_b200.cli validate --strategy s.json --cluster c.json
    python -m paper_2406_17145_b200.cli compare --graph g.json --cluster c.json --mini-batch 8

Files are canonical JSON documents with a ``format_version`` and a
``kind``; parsing rejects unknown fields and ``emit(parse(x)) == x`` on canonical input.
A StrategyFile carries the configured StageGraph (stages with schedule configs and task
lists), the GraphFile it partitions (so it simulates stand-alone) and the sim options.
Every emitted document is byte-deterministic (sorted keys, fixed float repr).

Exit codes: 0 ok, 1 invalid strategy (validate), 2 parse error,
3 graph not series-parallel (witness printed), 4 no feasible strategy, 5 deadlock.
``GPP_LOG`` sets the log level; ``--threads`` is accepted for interface parity (the
search is single-threaded and deterministic).
"""

from __future__ import annotations

import argparse
import json
import logging
import os
import sys
import time
from typing import Any

from . import partition as P
from . import sim as SIM
from . import workloads as W
from .model import (ComputationGraph, CostCurve, DeviceCluster, Operator, ScheduleConfig, Stage, StageGraph,
                    Task, pipeline_depth, validate_strategy)
from .spgraph import NotSeriesParallelError

FORMAT_VERSION = 1
log = logging.getLogger("gpp")


class FormatError(ValueError):
    """A file does not parse: bad JSON, wrong kind/version, unknown or missing fields."""


def _strict(d: Any, where: str, required: set, optional: set = frozenset()) -> dict:
    if not isinstance(d, dict):
        raise FormatError(f"{where}: expected an object")
    keys = set(d)
    if keys - required - set(optional):
        raise FormatError(f"{where}: unknown field(s) {sorted(keys - required - set(optional))}")
    if required - keys:
        raise FormatError(f"{where}: missing field(s) {sorted(required - keys)}")
    return d


def _header(d: Any, kind: str) -> None:
    if not isinstance(d, dict):
        raise FormatError(f"{kind} file: expected an object")
    if d.get("format_version") != FORMAT_VERSION:
        raise FormatError(f"{kind} file: format_version must be {FORMAT_VERSION}")
    if d.get("kind") != kind:
        raise FormatError(f"expected a {kind} file, got kind={d.get('kind')!r}")


def dumps(doc: dict) -> str:
    """Canonical text: sorted keys, 1-space indent, trailing newline."""
    return json.dumps(doc, sort_keys=True, indent=1) + "\n"


# ------------------------------------------------------------------ GraphFile
def curve_to_json(c: CostCurve) -> dict:
    if c.kind == "affine":
        return {"kind": "affine", "a": float(c.a), "b": float(c.b)}
    return {"kind": c.kind, "points": [[float(n), float(ms)] for n, ms in c.points]}


def curve_from_json(d: Any, where: str) -> CostCurve:
    if not isinstance(d, dict) or "kind" not in d:
        raise FormatError(f"{where}: cost curve needs a kind")
    if d["kind"] == "affine":
        _strict(d, where, {"kind", "a", "b"})
        return CostCurve.affine(float(d["a"]), float(d["b"]))
    if d["kind"] == "table":
        _strict(d, where, {"kind", "points"})
        try:
            return CostCurve.table({float(n): float(ms) for n, ms in d["points"]})
        except (TypeError, ValueError) as e:
            raise FormatError(f"{where}: bad table points ({e})") from None
    raise FormatError(f"{where}: unknown curve kind {d['kind']!r}")


def graph_to_json(g: ComputationGraph) -> dict:
    return {
        "format_version": FORMAT_VERSION, "kind": "graph",
        "ops": [{"id": o.id, "name": o.name, "param_bytes": float(o.param_bytes),
                 "act_bytes_per_sample": float(o.act_bytes_per_sample),
                 "out_bytes_per_sample": float(o.out_bytes_per_sample),
                 "fwd_cost": curve_to_json(o.fwd_cost), "bwd_cost": curve_to_json(o.bwd_cost)}
                for o in sorted(g.ops, key=lambda o: o.id)],
        "edges": [list(e) for e in sorted(g.edges)],
    }


def graph_from_json(d: Any) -> ComputationGraph:
    _header(d, "graph")
    _strict(d, "graph", {"format_version", "kind", "ops", "edges"})
    ops = []
    for i, o in enumerate(d["ops"]):
        w = f"graph.ops[{i}]"
        _strict(o, w, {"id", "name", "param_bytes", "act_bytes_per_sample", "out_bytes_per_sample",
                       "fwd_cost", "bwd_cost"})
        ops.append(Operator(int(o["id"]), str(o["name"]), float(o["param_bytes"]), float(o["act_bytes_per_sample"]),
                            float(o["out_bytes_per_sample"]), curve_from_json(o["fwd_cost"], w + ".fwd_cost"),
                            curve_from_json(o["bwd_cost"], w + ".bwd_cost")))
    try:
        return ComputationGraph(ops, [(int(a), int(b)) for a, b in d["edges"]])
    except (TypeError, ValueError) as e:
        raise FormatError(f"graph: {e}") from None


# ------------------------------------------------------------------ ClusterFile
_CLUSTER_FIELDS = ("num_devices", "mem_per_device", "intra_bw", "inter_bw", "link_latency")


def cluster_to_json(c: DeviceCluster) -> dict:
    return {"format_version": FORMAT_VERSION, "kind": "cluster", "num_devices": int(c.num_devices),
            **{k: float(getattr(c, k)) for k in _CLUSTER_FIELDS[1:]}}


def cluster_from_json(d: Any) -> DeviceCluster:
    _header(d, "cluster")
    _strict(d, "cluster", {"format_version", "kind", *_CLUSTER_FIELDS})
    try:
        return DeviceCluster(int(d["num_devices"]), float(d["mem_per_device"]), float(d["intra_bw"]),
                             float(d["inter_bw"]), float(d["link_latency"]))
    except (TypeError, ValueError) as e:
        raise FormatError(f"cluster: {e}") from None


# ------------------------------------------------------------------ StrategyFile
def strategy_to_json(sg: StageGraph, g: ComputationGraph, weight_multiplier: float = 2.0,
                     sync_epilogue: bool = False) -> dict:
    stages = []
    for s in sg.stages:
        stages.append({
            "id": s.id, "op_ids": sorted(s.op_ids), "micro_batch": s.micro_batch, "devices": sorted(s.devices),
            "sched_cfg": None if s.sched_cfg is None else {
                "inflight_samples": s.sched_cfg.inflight_samples, "micro_batch": s.sched_cfg.micro_batch,
                "k": s.sched_cfg.k},
            "schedule": None if s.schedule is None else [[t.direction, t.index] for t in s.schedule],
        })
    return {"format_version": FORMAT_VERSION, "kind": "strategy", "mini_batch": sg.mini_batch,
            "stages": stages, "edges": [list(e) for e in sorted(sg.edges)], "graph": graph_to_json(g),
            "sim": {"weight_multiplier": weight_multiplier, "sync_epilogue": sync_epilogue}}


def strategy_from_json(d: Any) -> tuple[StageGraph, ComputationGraph, dict]:
    _header(d, "strategy")
    _strict(d, "strategy", {"format_version", "kind", "mini_batch", "stages", "edges", "graph", "sim"})
    g = graph_from_json(d["graph"])
    simo = _strict(d["sim"], "strategy.sim", {"weight_multiplier", "sync_epilogue"})
    stages = []
    try:
        for i, s in enumerate(d["stages"]):
            w = f"strategy.stages[{i}]"
            _strict(s, w, {"id", "op_ids", "micro_batch", "devices", "sched_cfg", "schedule"})
            cfg = None
            if s["sched_cfg"] is not None:
                c = _strict(s["sched_cfg"], w + ".sched_cfg", {"inflight_samples", "micro_batch", "k"})
                cfg = ScheduleConfig(int(c["inflight_samples"]), int(c["micro_batch"]), int(c["k"]))
            sched = None if s["schedule"] is None else tuple(Task(str(a), int(j)) for a, j in s["schedule"])
            stages.append(Stage(int(s["id"]), frozenset(int(o) for o in s["op_ids"]), int(s["micro_batch"]),
                                frozenset(int(x) for x in s["devices"]), cfg, sched))
        sg = StageGraph(stages, [(int(a), int(b)) for a, b in d["edges"]], int(d["mini_batch"]))
    except (TypeError, ValueError) as e:
        raise FormatError(f"strategy: {e}") from None
    return sg, g, {"weight_multiplier": float(simo["weight_multiplier"]), "sync_epilogue": bool(simo["sync_epilogue"])}


def load(path: str) -> Any:
    try:
        with open(path) as f:
            return json.load(f)
    except (OSError, json.JSONDecodeError) as e:
        raise FormatError(f"{path}: {e}") from None


def _write(path: str | None, text: str) -> None:
    if path in (None, "-"):
        sys.stdout.write(text)
        return
    with open(path, "w") as f:
        f.write(text)


# ------------------------------------------------------------------ reports
def report_to_json(rep: SIM.SimReport) -> dict:
    key = lambda m: {str(k): v for k, v in sorted(m.items())}
    return {"iteration_ms": rep.iteration_ms, "depth": rep.depth, "warm_up_microbatches": rep.warm_up_microbatches,
            "warm_up_per_stage": key(rep.warm_up_per_stage), "peak_inflight_samples": key(rep.peak_inflight_samples),
            "busy_ms": key(rep.busy_ms), "idle_ms": key(rep.idle_ms), "peak_mem_bytes": key(rep.peak_mem_bytes),
            "bubble_fraction": rep.bubble_fraction}


def gantt_svg(rep: SIM.SimReport, row_h: int = 22, width: int = 960) -> str:
    """Standalone SVG, one row per stage, fw blue / bw orange, deterministic bytes."""
    stages = sorted({sid for sid, _, _ in rep.task_times})
    T = rep.iteration_ms or 1.0
    x0 = 70
    scale = (width - x0 - 10) / T
    h = row_h * len(stages) + 30
    out = [f'<svg xmlns="http://www.w3.org/2000/svg" width="{width}" height="{h}" font-family="monospace" font-size="11">']
    for r, sid in enumerate(stages):
        y = 10 + r * row_h
        out.append(f'<text x="4" y="{y + row_h - 8}">stage{sid}</text>')
        for (s, d, j), (t0, t1) in sorted(rep.task_times.items()):
            if s != sid:
                continue
            col = "#4a7fd6" if d == "fw" else "#e8903a"
            out.append(f'<rect x="{x0 + t0 * scale:.2f}" y="{y}" width="{max((t1 - t0) * scale, 0.5):.2f}" '
                       f'height="{row_h - 4}" fill="{col}" stroke="#222" stroke-width="0.4">'
                       f'<title>{d}{j} {t0:.4f}-{t1:.4f} ms</title></rect>')
    out.append(f'<text x="{x0}" y="{h - 6}">0 ms .. {T:.4f} ms</text>')
    out.append("</svg>")
    return "\n".join(out) + "\n"


# ------------------------------------------------------------------ commands
def _presets(name: str, branches: int | None) -> tuple[ComputationGraph, DeviceCluster | None]:
    if name == "fig2":
        return W.fig2(), DeviceCluster(4, 1e12, 1e3, 1e9)
    if name == "case-study":
        return W.case_study(branches=branches or 2), W.case_study_cluster()
    if name == "candle-uno":
        n = branches or 7
        return W.candle(towers=n).graph, W.b200_cluster(min(n + 1, 8))
    if name == "mmt":
        return W.mmt(branches=branches or 4).graph, W.b200_cluster(8)
    if name == "dlrm":
        return W.dlrm(tables=branches or 26).graph, W.b200_cluster(8)
    if name == "toy":
        return W.toy().graph, W.b200_cluster(2)
    if name == "chain":
        return W.chain(branches or 6), DeviceCluster(3, 1e12, 1e3, 1e9)
    raise FormatError(f"unknown preset {name!r}")


def _opts(args) -> P.PartitionOptions:
    kw = {"per_stage_schedules": args.per_stage_schedules}
    if args.epsilon is not None:
        kw["epsilon_rel"] = args.epsilon
    return P.PartitionOptions(**kw)


def _run(fn, g, cl, B, opts):
    t0 = time.perf_counter()
    st = fn(g, cl, B, opts)
    return st, time.perf_counter() - t0


def cmd_gen(args) -> int:
    g, cl = _presets(args.preset, args.branches)
    _write(args.out, dumps(graph_to_json(g)))
    if args.cluster_out and cl is not None:
        _write(args.cluster_out, dumps(cluster_to_json(cl)))
    return 0


def cmd_optimize(args) -> int:
    g = graph_from_json(load(args.graph))
    cl = cluster_from_json(load(args.cluster))
    fn = P.optimize if args.mode == "gpp" else P.spp_optimize
    st, secs = _run(fn, g, cl, args.mini_batch, _opts(args))
    sg = st.stage_graph
    rep = SIM.simulate(sg, cl, g)
    _write(args.out, dumps(strategy_to_json(sg, g)))
    summary = {"mode": args.mode, "bottleneck_tps": st.bottleneck_tps, "depth": pipeline_depth(sg),
               "stages": len(sg.stages), "peak_memory_bytes": max(rep.peak_mem_bytes.values(), default=0.0),
               "iteration_ms": rep.iteration_ms, "warm_up_microbatches": rep.warm_up_microbatches,
               "search": {"dp_states": st.dp_states, "probes": st.probes, "seconds": round(secs, 6)}}
    sys.stderr.write(json.dumps(summary, sort_keys=True) + "\n")
    return 0


def cmd_simulate(args) -> int:
    sg, g, simo = strategy_from_json(load(args.strategy))
    cl = cluster_from_json(load(args.cluster))
    rep = SIM.simulate(sg, cl, g, weight_multiplier=simo["weight_multiplier"], sync_epilogue=simo["sync_epilogue"])
    _write(args.out, dumps(report_to_json(rep)))
    if args.trace:
        _write(args.trace, SIM.emit_trace(rep) + "\n")
    if args.gantt:
        _write(args.gantt, gantt_svg(rep))
    return 0


def cmd_validate(args) -> int:
    sg, g, _ = strategy_from_json(load(args.strategy))
    cl = cluster_from_json(load(args.cluster)) if args.cluster else DeviceCluster(
        max((x for s in sg.stages for x in s.devices), default=0) + 1, 1e30, 1.0, 1.0)
    viol = validate_strategy(g, cl, sg)
    _write(args.out, dumps({"violations": [{"code": v.code, "message": v.message} for v in viol]}))
    return 0 if not viol else 1


def cmd_compare(args) -> int:
    g = graph_from_json(load(args.graph))
    cl = cluster_from_json(load(args.cluster))
    res = {}
    for mode, fn in (("gpp", P.optimize), ("spp", P.spp_optimize)):
        st, secs = _run(fn, g, cl, args.mini_batch, _opts(args))
        rep = SIM.simulate(st.stage_graph, cl, g)
        res[mode] = {"depth": rep.depth, "warm_up_microbatches": rep.warm_up_microbatches,
                     "micro_batches": sorted({s.micro_batch for s in st.stage_graph.stages}),
                     "stages": len(st.stage_graph.stages), "iteration_ms": rep.iteration_ms,
                     "peak_memory_bytes": max(rep.peak_mem_bytes.values(), default=0.0),
                     "bottleneck_tps": st.bottleneck_tps, "dp_states": st.dp_states, "probes": st.probes}
    res["iteration_ratio_gpp_over_spp"] = res["gpp"]["iteration_ms"] / res["spp"]["iteration_ms"]
    _write(args.out, dumps(res))
    return 0


def build_parser() -> argparse.ArgumentParser:
    ap = argparse.ArgumentParser(prog="gpp", description="GraphPipe partitioner / scheduler / simulator")
    ap.add_argument("--threads", type=int, default=1, help="accepted for interface parity (search is serial)")
    sub = ap.add_subparsers(dest="cmd", required=True)
    bool_ = lambda s: s.lower() in ("1", "true", "yes", "on")

    p = sub.add_parser("gen", help="emit a preset GraphFile (and ClusterFile)")
    p.add_argument("--preset", required=True,
                   choices=["mmt", "dlrm", "candle-uno", "case-study", "fig2", "toy", "chain"])
    p.add_argument("--branches", type=int, default=None)
    p.add_argument("--out", default="-")
    p.add_argument("--cluster-out", default=None)
    p.set_defaults(fn=cmd_gen)

    for name, fn in (("optimize", cmd_optimize), ("compare", cmd_compare)):
        p = sub.add_parser(name)
        p.add_argument("--graph", required=True)
        p.add_argument("--cluster", required=True)
        p.add_argument("--mini-batch", type=int, required=True)
        if name == "optimize":
            p.add_argument("--mode", choices=["gpp", "spp"], default="gpp")
        p.add_argument("--per-stage-schedules", type=bool_, default=False)
        p.add_argument("--epsilon", type=float, default=None)
        p.add_argument("--out", default="-")
        p.set_defaults(fn=fn)

    p = sub.add_parser("simulate")
    p.add_argument("--strategy", required=True)
    p.add_argument("--cluster", required=True)
    p.add_argument("--trace", default=None)
    p.add_argument("--gantt", default=None)
    p.add_argument("--out", default="-")
    p.set_defaults(fn=cmd_simulate)

    p = sub.add_parser("validate")
    p.add_argument("--strategy", required=True)
    p.add_argument("--cluster", default=None)
    p.add_argument("--out", default="-")
    p.set_defaults(fn=cmd_validate)
    return ap


def main(argv: list[str] | None = None) -> int:
    logging.basicConfig(level=os.environ.get("GPP_LOG", "WARNING").upper(), stream=sys.stderr)
    args = build_parser().parse_args(argv)
    try:
        if getattr(args, "mini_batch", 1) is not None and getattr(args, "mini_batch", 1) < 1:
            raise FormatError("--mini-batch must be >= 1")
        return args.fn(args)
    except FormatError as e:
        sys.stderr.write(f"parse error: {e}\n")
        return 2
    except NotSeriesParallelError as e:
        sys.stderr.write(f"not series-parallel: witness edges {sorted(e.witness_edges)}\n")
        return 3
    except P.NoFeasibleStrategy as e:
        sys.stderr.write(f"no feasible strategy: {e}\n")
        return 4
    except SIM.Deadlock as e:
        sys.stderr.write(f"{e}\n")
        return 5


if __name__ == "__main__":
    sys.exit(main())
