"""Workload presets: computation graphs (for the partitioner) + layer specs (for the executor).

Appendix B model shapes as restated by BASELINE.json
``configs`` and SURVEY.md §8(d); the paper gives shapes, not millisecond
profiles, so the cost curves here are analytic B200 estimates (FLOPs at a
fixed fraction of the measured bf16 peak plus a per-launch overhead, bytes at
measured HBM bandwidth).  ``runtime.profiler`` replaces them with measured
table curves.  Graph-only presets (``fig2``, ``case_study``, ``chain``) carry
unit costs for the SPEC acceptance checks.

Op ids are assigned branch by branch, so ``linearize`` (smallest ready id
first) yields the branch-by-branch SPP order.
"""

from __future__ import annotations

import json
import os
from dataclasses import dataclass, field, replace

from .model import ComputationGraph, CostCurve, DeviceCluster, Operator

__all__ = ["LayerSpec", "Workload", "b200_cluster", "PRESETS", "make", "with_measured_curves", "MEASURED_CURVES"]

# B200 constants (MEASURED_PEAKS.json).
BF16_TFLOPS_SUSTAINED = 1397.3
HBM_GBS = 6539.5
GEMM_EFF = 0.6                       # assumed achieved fraction for the analytic curves
FLOP_PER_MS = BF16_TFLOPS_SUSTAINED * 1e9 * GEMM_EFF
FP32_FLOP_PER_MS = 60e9              # SIMT FFMA, ~60 TFLOP/s
BYTES_PER_MS = HBM_GBS * 1e6
LAUNCH_MS = 0.004


@dataclass(frozen=True)
class LayerSpec:
    """What the executor runs for one operator.

    kind: "dense" (Linear + act), "concat", "mse_head", "bce_head", "ce_head",
    "mmt_layer", "embbag", "interaction".
    """

    kind: str
    in_dim: int = 0
    out_dim: int = 0
    act: str = "none"
    data_key: str | None = None      # source ops read this batch tensor
    label_key: str | None = None     # loss heads read this batch tensor
    extra: tuple = ()                # kind-specific (e.g. mmt: (seq, heads, ffn, pool))


@dataclass
class Workload:
    name: str
    graph: ComputationGraph
    layers: dict[int, LayerSpec]
    data: dict[str, tuple[tuple[int, ...], str]]  # key -> (per-sample shape, kind: normal|label|binary|index)
    mini_batch: int
    dtype: str = "bf16"
    flops_per_sample: float = 0.0    # train (fw+bw) algorithmic FLOPs per sample
    bytes_per_sample: float = 0.0    # HBM-bound algorithmic bytes per sample (embeddings)
    notes: str = ""
    meta: dict = field(default_factory=dict)


# Frozen B200 per-operator timings (tools/profile_costs.py on one B200, production
# kernels): the partitioner's table CostCurves.
MEASURED_CURVES = os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "profiles",
                               "cost_curves_b200.json")


def dense_profile_key(spec: "LayerSpec") -> str:
    """Profile key of a dense op: source ops (reading batch data) run no dgrad."""
    return f"dense:{spec.in_dim}x{spec.out_dim}:{spec.act}:{'nodgrad' if spec.data_key else 'dgrad'}"


def mmt_profile_key(spec: "LayerSpec") -> str:
    """Profile key of an MMT encoder layer (tools/profile_costs.py mmt)."""
    S, d, H, ffn, pool = spec.extra
    return f"mmt:{S}x{d}x{H}x{ffn}:{'pool' if pool else 'seq'}"


def profile_key(spec: "LayerSpec | None") -> str | None:
    if spec is None:
        return None
    if spec.kind == "dense":
        return dense_profile_key(spec)
    if spec.kind == "mmt_layer":
        return mmt_profile_key(spec)
    return None


def with_measured_curves(wl: "Workload", profile: dict | str | None = None) -> tuple["Workload", int]:
    """Replace the analytic fw/bw curves of bf16 dense / MMT-layer operators by measured B200 tables.

    ``profile`` is the JSON written by tools/profile_costs.py (default: the committed
    ``profiles/cost_curves_b200.json``): ``curves[key] = {b: [...], fwd_ms: [...], bwd_ms:
    [...]}`` with ms per task at b samples per device.  Operators without a profiled shape
    keep their analytic curves.  Returns (workload, number of operators replaced).
    """
    if profile is None or isinstance(profile, str):
        path = profile or MEASURED_CURVES
        if not os.path.exists(path):
            return wl, 0
        with open(path) as f:
            profile = json.load(f)
    if wl.dtype != "bf16":
        return wl, 0
    curves = profile.get("curves", {})
    ops, n = [], 0
    for op in wl.graph.ops:
        spec = wl.layers.get(op.id)
        key = profile_key(spec)
        c = curves.get(key) if key else None
        if c:
            op = replace(op, fwd_cost=CostCurve.table(dict(zip(c["b"], c["fwd_ms"]))),
                         bwd_cost=CostCurve.table(dict(zip(c["b"], c["bwd_ms"]))))
            n += 1
        ops.append(op)
    if not n:
        return wl, 0
    return replace(wl, graph=ComputationGraph(ops, wl.graph.edges),
                   meta={**wl.meta, "costs": f"measured B200 tables for {n} ops"}), n


# NCCL all-reduce bus bandwidth of 2.4 GB fp32 gradients through libgpp_b200 on one B200
# box (tools/bench_allreduce.py, profiles/allreduce_b200.jsonl): 598 GB/s at 2 GPUs, 660 GB/s
# at 4; the 8-GPU value is assumed equal to the 4-GPU one (not measured: gpurun gives <= 4).
DP_BUSBW = {2: 5.98e8, 4: 6.6e8}


def b200_cluster(n: int, mem_bytes: float = 180e9) -> DeviceCluster:
    """NVLink 5 / NVSwitch box: P2P at the 900 GB/s per-direction link rate (9e8 bytes/ms,
    ~10 us latency); the DP-sync bandwidth (``intra_bw``, priced by cost.dp_sync_time) is
    the measured NCCL all-reduce bus bandwidth."""
    dp = DP_BUSBW.get(n, DP_BUSBW[4]) if n > 1 else 9e8
    return DeviceCluster(num_devices=n, mem_per_device=mem_bytes, intra_bw=dp, inter_bw=9e8, link_latency=0.01)


def _gemm_curve(flops_per_sample: float, launches: int, fp32: bool = False) -> CostCurve:
    rate = FP32_FLOP_PER_MS if fp32 else FLOP_PER_MS
    return CostCurve.affine(LAUNCH_MS * launches, flops_per_sample / rate)


def _dense(oid, name, din, dout, act, bytes_el, data_key=None, fp32=False):
    f = 2.0 * din * dout
    op = Operator(
        id=oid, name=name, param_bytes=4.0 * (din * dout + dout),  # fp32 master weights
        act_bytes_per_sample=bytes_el * (din + dout), out_bytes_per_sample=bytes_el * dout,
        fwd_cost=_gemm_curve(f, 1, fp32), bwd_cost=_gemm_curve(2 * f, 3, fp32),
    )
    return op, LayerSpec("dense", din, dout, act, data_key=data_key)


def _concat(oid, name, dout, bytes_el):
    op = Operator(id=oid, name=name, act_bytes_per_sample=0.0, out_bytes_per_sample=bytes_el * dout,
                  fwd_cost=CostCurve.affine(LAUNCH_MS, bytes_el * dout * 2 / BYTES_PER_MS),
                  bwd_cost=CostCurve.affine(0.0, 0.0))
    return op, LayerSpec("concat", dout, dout)


def _head(oid, name, kind, din, nout, bytes_el, label_key, fp32=False):
    f = 2.0 * din * nout
    op = Operator(id=oid, name=name, param_bytes=4.0 * (din * nout + nout),
                  act_bytes_per_sample=bytes_el * din, out_bytes_per_sample=4.0,
                  fwd_cost=_gemm_curve(f, 2, fp32), bwd_cost=_gemm_curve(2 * f, 3, fp32))
    return op, LayerSpec(kind, din, nout, label_key=label_key)


def multi_tower(name: str, towers: int, layers: int, width: int, in_dim: int, tail_hidden: int,
                B: int, dtype: str = "bf16", act: str = "relu") -> Workload:
    """CANDLE-Uno-style towers -> concat -> [tail Linear+ReLU] -> MSE head."""
    fp32 = dtype == "fp32"
    el = 4 if fp32 else 2
    ops, specs, edges, data = [], {}, [], {}
    oid = 0
    ends = []
    for t in range(towers):
        prev = None
        for l in range(layers):
            din = in_dim if l == 0 else width
            a = act
            op, spec = _dense(oid, f"t{t}_ff{l}", din, width, a, el, data_key=f"x{t}" if l == 0 else None, fp32=fp32)
            ops.append(op)
            specs[oid] = spec
            if prev is not None:
                edges.append((prev, oid))
            prev = oid
            oid += 1
        ends.append(prev)
        data[f"x{t}"] = ((in_dim,), "normal")
    cat = oid
    op, spec = _concat(cat, "concat", towers * width, el)
    ops.append(op)
    specs[cat] = spec
    edges += [(e, cat) for e in ends]
    oid += 1
    prev, dprev = cat, towers * width
    if tail_hidden:
        op, spec = _dense(oid, "tail_ff", dprev, tail_hidden, act, el, fp32=fp32)
        ops.append(op)
        specs[oid] = spec
        edges.append((prev, oid))
        prev, dprev = oid, tail_hidden
        oid += 1
    op, spec = _head(oid, "head_mse", "mse_head", dprev, 1, el, "y", fp32=fp32)
    ops.append(op)
    specs[oid] = spec
    edges.append((prev, oid))
    data["y"] = ((), "normal")
    flops = 0.0
    for s in specs.values():
        if s.kind in ("dense", "mse_head"):
            flops += 6.0 * s.in_dim * max(1, s.out_dim)
    return Workload(name, ComputationGraph(ops, edges), specs, data, B, dtype, flops_per_sample=flops)


def toy(B: int = 64) -> Workload:
    """BASELINE configs[0]: 2 branches x 4 x [Linear(256,256)+ReLU] -> concat 512 ->
    Linear(512,256)+ReLU -> Linear(256,1), MSE; fp32; B=64 (b=16: 4 micro-batches)."""
    return multi_tower("toy", towers=2, layers=4, width=256, in_dim=256, tail_hidden=256, B=B, dtype="fp32")


def candle(B: int = 1024, towers: int = 7) -> Workload:
    """BASELINE configs[1]: CANDLE-Uno, 7 towers x 4 x FF(4096)+ReLU,
    light tail Linear(28672,1024)+ReLU -> Linear(1024,1) MSE."""
    return multi_tower("candle", towers=towers, layers=4, width=4096, in_dim=4096, tail_hidden=1024, B=B)


# ---------------------------------------------------------------------------
# Graph-only presets for the SPEC acceptance checks (unit costs).
# ---------------------------------------------------------------------------


def _unit(oid, name, act=1.0, out=1.0, params=1e3, fw=1.0, bw=1.0):
    return Operator(oid, name, params, act, out, CostCurve.affine(0.0, fw), CostCurve.affine(0.0, bw))


def fig2() -> ComputationGraph:
    """PAPER.md Fig. 2: three 2-op branches merging into a 2-op tail (unit costs)."""
    ops = [_unit(i, f"o{i + 1}") for i in range(8)]
    edges = [(0, 1), (2, 3), (4, 5), (1, 6), (3, 6), (5, 6), (6, 7)]
    return ComputationGraph(ops, edges)


def chain(n: int, costs: list[float] | None = None) -> ComputationGraph:
    costs = costs or [1.0] * n
    ops = [_unit(i, f"c{i}", fw=costs[i], bw=2 * costs[i]) for i in range(n)]
    return ComputationGraph(ops, [(i, i + 1) for i in range(n - 1)])


CASE_STUDY_B = 64  # mini-batch of the §7.5 case study preset


def case_study(blocks: int = 4, branches: int = 2) -> ComputationGraph:
    """§7.5: branches x [attention + 2 linear] blocks, merged by a concat.

    One block = one operator (layer granularity); op ids are branch-major.
    The concat is zero-cost and has no weights, so it is folded into the last block of each
    branch (the branch outputs are the model outputs): GPP can then place it with a block
    as in Fig. 6 instead of spending a device on it.  The documented
    synthetic profile:

    * fw ms {1: 1.0, 2: 1.2, 4: 2.0, 8: 3.8}, bw = 2 x fw: per-sample cost falls 1.8 -> 1.5 ms
      from b = 2 to b = 4 (the compute-efficiency gain source);
    * 1 GB of weights per block: a data-parallel replica pays a ~10 ms all-reduce per
      micro-batch, and two blocks never fit one device under ``case_study_cluster``;
    * 100 MB of activations per sample: with the 4 GB cap the first stage of a depth-D
      1F1B pipeline fits D*b <= 16 samples -> b = 4 at depth 4 (GPP), b = 2 at depth 8 (SPP).
    """
    f = CostCurve.table({1: 1.0, 2: 1.2, 4: 2.0, 8: 3.8})
    bw = CostCurve.table({1: 2.0, 2: 2.4, 4: 4.0, 8: 7.6})
    ops, edges = [], []
    oid = 0
    for br in range(branches):
        prev = None
        for k in range(blocks):
            ops.append(Operator(oid, f"b{br}_blk{k}", 1e9, 1e8, 1e3, f, bw))
            if prev is not None:
                edges.append((prev, oid))
            prev = oid
            oid += 1
    return ComputationGraph(ops, edges)


def case_study_cluster(n: int = 8) -> DeviceCluster:
    """The case study's memory-capped pool: 4 GB per device, 1e8 B/ms links."""
    return DeviceCluster(num_devices=n, mem_per_device=4e9, intra_bw=1e8, inter_bw=1e8, link_latency=0.0)


def dlrm(B: int = 512, tables: int = 26, rows: int = 1_000_000, bag: int = 100, hidden: int = 4096,
         dense_in: int = 13, emb: int = 64) -> Workload:
    """BASELINE configs[3]: DLRM — bottom MLP dense_in -> hidden x3 -> 64, `tables` embedding
    bags (rows x 64, bag 100, sum-pooled), dot interaction (64 + F(F-1)/2 = 415, padded to
    416), top MLP 416 -> hidden x3 -> 1, BCE.
    Op ids: bottom MLP first (feature 0 of the interaction), then the tables."""
    ops, specs, edges, data = [], {}, [], {}
    din = -(-dense_in // 8) * 8  # zero-padded so the TMA row pitch is 16-byte aligned
    data["dense"] = ((din,), f"normal_pad:{dense_in}")
    oid = 0
    prev = None
    dims = [din, hidden, hidden, hidden, emb]
    for l in range(4):
        op, spec = _dense(oid, f"bot{l}", dims[l], dims[l + 1], "relu", 2, data_key="dense" if l == 0 else None)
        ops.append(op)
        specs[oid] = spec
        if prev is not None:
            edges.append((prev, oid))
        prev = oid
        oid += 1
    bottom_end = prev
    table_ids = []
    for t in range(tables):
        fbytes = bag * emb * 4 + bag * 8 + emb * 2          # gather fp32 rows + idx + pooled write
        bbytes = 2 * bag * emb * 4 + bag * 8 + emb * 2      # deferred scatter: RMW of every looked-up row
        op = Operator(oid, f"emb{t}", param_bytes=4.0 * rows * emb, act_bytes_per_sample=0.0,
                      out_bytes_per_sample=2.0 * emb,
                      fwd_cost=CostCurve.affine(LAUNCH_MS, fbytes / BYTES_PER_MS),
                      bwd_cost=CostCurve.affine(LAUNCH_MS, bbytes / BYTES_PER_MS))
        ops.append(op)
        specs[oid] = LayerSpec("embbag", rows, emb, data_key=f"idx{t}", extra=(bag,))
        data[f"idx{t}"] = ((bag,), f"index:{rows}")
        table_ids.append(oid)
        oid += 1
    F = tables + 1
    inter_out = -(-(emb + F * (F - 1) // 2) // 8) * 8
    inter = oid
    ibytes = 2.0 * (F * emb + inter_out)
    ops.append(Operator(inter, "interaction", act_bytes_per_sample=2.0 * F * emb, out_bytes_per_sample=2.0 * inter_out,
                        fwd_cost=CostCurve.affine(LAUNCH_MS * (F + 1), 2 * ibytes / BYTES_PER_MS),
                        bwd_cost=CostCurve.affine(LAUNCH_MS * (F + 1), 3 * ibytes / BYTES_PER_MS)))
    specs[inter] = LayerSpec("interaction", F, inter_out, extra=(emb, emb + F * (F - 1) // 2))
    edges += [(bottom_end, inter)] + [(t, inter) for t in table_ids]
    oid += 1
    prev, dprev = inter, inter_out
    for l in range(3):
        op, spec = _dense(oid, f"top{l}", dprev, hidden, "relu", 2)
        ops.append(op)
        specs[oid] = spec
        edges.append((prev, oid))
        prev, dprev = oid, hidden
        oid += 1
    op, spec = _head(oid, "head_bce", "bce_head", dprev, 1, 2, "y")
    ops.append(op)
    specs[oid] = spec
    edges.append((prev, oid))
    data["y"] = ((), "binary")
    flops = sum(6.0 * s.in_dim * max(1, s.out_dim) for s in specs.values() if s.kind in ("dense", "bce_head"))
    flops += 6.0 * F * (F - 1) / 2 * emb
    byts = tables * (3 * bag * emb * 4 + 2 * bag * 8 + 2 * emb * 2)
    return Workload("dlrm", ComputationGraph(ops, edges), specs, data, B, "bf16",
                    flops_per_sample=flops, bytes_per_sample=float(byts))


def mmt_layer_flops(S: int, d: int, ffn: int) -> float:
    """Forward FLOPs per sample of one encoder layer: 4 projections + QK^T and PV."""
    return 2.0 * S * d * (3 * d) + 2.0 * S * d * d + 2.0 * 2 * S * d * ffn + 2.0 * 2 * S * S * d


def mmt(B: int = 32, branches: int = 4, layers: int = 12, S: int = 512, d: int = 1024, H: int = 16,
        ffn: int = 4096, classes: int = 1000) -> Workload:
    """BASELINE configs[2]/[4]: Multi-Modal Transformer — `branches` x `layers` pre-LN encoder
    layers (d=1024, 16 heads, FFN 4096 GELU, seq 512, non-causal), the last
    layer of each branch mean-pools its tokens, concat [B, branches*d] -> Linear(., classes) CE
    (SURVEY.md §8(d) config 3).  One operator per layer (layer granularity)."""
    ops, specs, edges, data = [], {}, [], {}
    oid = 0
    ends = []
    f_fwd = mmt_layer_flops(S, d, ffn)
    for t in range(branches):
        prev = None
        for l in range(layers):
            pool = l == layers - 1
            out_dim = d if pool else S * d
            params = 4.0 * (4 * d * d + 2 * d * ffn + 9 * d + ffn)
            acts = 2.0 * S * (10 * d + 2 * ffn) + 2.0 * H * S * S
            ops.append(Operator(oid, f"b{t}_layer{l}", param_bytes=params, act_bytes_per_sample=acts,
                                out_bytes_per_sample=2.0 * out_dim,
                                fwd_cost=_gemm_curve(f_fwd, 10), bwd_cost=_gemm_curve(2 * f_fwd, 24)))
            specs[oid] = LayerSpec("mmt_layer", S * d, out_dim, data_key=f"x{t}" if l == 0 else None,
                                   extra=(S, d, H, ffn, pool))
            if prev is not None:
                edges.append((prev, oid))
            prev = oid
            oid += 1
        ends.append(prev)
        data[f"x{t}"] = ((S * d,), "normal")
    cat = oid
    op, spec = _concat(cat, "concat", branches * d, 2)
    ops.append(op)
    specs[cat] = spec
    edges += [(e, cat) for e in ends]
    oid += 1
    op, spec = _head(oid, "head_ce", "ce_head", branches * d, classes, 2, "label")
    ops.append(op)
    specs[oid] = spec
    edges.append((cat, oid))
    data["label"] = ((), f"label:{classes}")
    flops = branches * layers * 3 * f_fwd + 6.0 * branches * d * classes
    return Workload("mmt", ComputationGraph(ops, edges), specs, data, B, "bf16", flops_per_sample=flops)


PRESETS = {"toy": toy, "candle": candle, "dlrm": dlrm, "mmt": mmt}


def make(name: str, **kw) -> Workload:
    if name not in PRESETS:
        raise ValueError(f"unknown preset {name!r}; known: {sorted(PRESETS)}")
    return PRESETS[name](**kw)
