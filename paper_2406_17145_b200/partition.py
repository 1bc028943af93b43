"""Pipeline-stage partitioner: bisection over bottleneck TPS + memoised SP-DP (Alg. 1).

SPEC.md:333-415, PAPER.md:595-729 (the reference ships no code for it).

``optimize`` bisects the target TPS t_m between 0 and MAXTPS; every probe runs
``search_stage_graph``: for each candidate source-stage config c, a memoised
``dp`` over the SP tree of the normalised graph with the dummy config c0 on the
sink side.  ``dp(node, c_f, c_b, d, t_max)`` returns the feasible fragment with
the fewest in-flight samples at its source stage, considering

* the node as ONE stage on d devices (TPS <= t_max, Eq. (2) memory <= M),
* every series cut (G1 ; G2) x device split d1 + d2 = d x boundary config c_m:
  G2 is solved first, its source in-flight i_m then feeds G1,
* every parallel split (G1 | G2) x device split, both halves sharing (c_f, c_b)
  and the join taking the larger in-flight count.

Design decisions beyond SPEC (documented in DESIGN.md):

* Virtual junction ops (``spgraph.normalize``) are zero-cost: a series part or
  parallel branch made only of virtual ops takes 0 devices and forms no stage,
  and virtual ops are stripped from the output, which is expressed over the
  ORIGINAL graph (so ``validate_strategy(g, ...)`` applies unchanged).
* Parallel enumeration: bundles of <= 6 branches use the
  reference ``parallel_splits`` cuts (one-vs-rest + balanced); larger bundles
  use contiguous cuts of the canonically ordered branch list, so DP states grow
  O(n^2) instead of 2^n (DLRM has 27 branches).
* PickBetter order: (peak per-device memory, #stages, canonical encoding)
  (SPEC.md:403); inside the DP the fewest source in-flight samples come first.
"""

from __future__ import annotations

import math
from dataclasses import dataclass, field
from typing import Iterable

from .cost import (DEFAULT_WEIGHT_MULTIPLIER, IndivisibleMicroBatchError, StageCostInput, dp_sync_time,
                   estimate_tps, stage_memory)
from .model import ComputationGraph, DeviceCluster, Operator, Stage, StageGraph, induced_stage_edges
from .sched import compute_in_flight, round_up, schedule_stage_graph
from .spgraph import (
    NormalizedGraph,
    SPLeaf,
    SPParallel,
    SPSeries,
    _as_series,
    decompose,
    flatten_parallel,
    flatten_series,
    linearize,
    normalize,
    parallel_splits,
)

__all__ = [
    "NoFeasibleStrategy",
    "PartitionOptions",
    "Strategy",
    "candidate_configs",
    "optimize",
    "spp_optimize",
    "search_stage_graph",
    "stage_comm_bytes",
]


class NoFeasibleStrategy(RuntimeError):
    pass


@dataclass(frozen=True)
class PartitionOptions:
    per_stage_schedules: bool = False  # SPEC.md:320 opt-in per-stage (b, k)
    epsilon_rel: float = 1e-3           # eps = 1e-3 * MAXTPS
    # "spec": stop when t_r - t_l <= eps_rel * MAXTPS.  "relative": stop when
    # t_r - t_l <= eps_rel * t_r — MAXTPS is priced at the smallest b, where launch overheads
    # dominate, so the SPEC rule can leave the optimum unresolved by >20% on B200 curves.
    epsilon_mode: str = "relative"
    weight_multiplier: float = DEFAULT_WEIGHT_MULTIPLIER
    max_exhaustive_branches: int = 6
    micro_batches: tuple[int, ...] | None = None  # restrict b candidates (e.g. fixed-b sweeps)
    # SPEC cost model charges the DP all-reduce once per MICRO-batch (cost.py:68-70).  The
    # B200 executor all-reduces once per ITERATION; True prices that.
    sync_per_iteration: bool = False
    # B200 extension (off for the SPEC tests): a parallel bundle's join and the series
    # segment after it may share a stage with one branch group -- Fig. 6's "one stage
    # necessarily contains the concatenation operator", which the
    # SP-aligned DP alone cannot express (it would spend a device on the join).
    merge_join: bool = False
    # B200 extension (off for the SPEC tests): bundles of <= max_exhaustive_branches also
    # try every contiguous cut of the canonical branch order besides the reference's
    # one-vs-rest + balanced cuts (spgraph.parallel_splits), so e.g. 6 towers can form
    # three 2-tower stages -- unreachable from one-vs-rest / halves.
    rich_splits: bool = False


@dataclass
class Strategy:
    stage_graph: StageGraph
    bottleneck_tps: float
    t_r: float
    maxtps: float
    probes: int
    dp_states: int
    mode: str
    stage_tps: dict[int, float] = field(default_factory=dict)


def candidate_configs(B: int, per_stage: bool = False) -> list[tuple[int, int]]:
    """(b, k) candidates: b = powers of two dividing B; k = 1, or powers of two <= B/b."""
    out = []
    b = 1
    while b <= B:
        if B % b == 0:
            if per_stage:
                k = 1
                while k <= B // b:
                    out.append((b, k))
                    k *= 2
            else:
                out.append((b, 1))
        b *= 2
    return out


def stage_comm_bytes(ng: NormalizedGraph, ops: frozenset) -> float:
    """Per-sample bytes entering ``ops`` (one tensor per outside producer)."""
    g = ng.graph
    producers = {u for v in ops for u in g.predecessors(v) if u not in ops}
    return float(sum(ng.effective_out_bytes[u] for u in sorted(producers)))


@dataclass(frozen=True)
class _FStage:
    ops: frozenset
    b: int
    k: int
    d: int
    i: int
    mem: float


@dataclass(frozen=True)
class _Frag:
    i_f: int | None
    stages: tuple
    mem: float

    def key(self):
        canon = tuple(sorted((tuple(sorted(s.ops)), s.b, s.d, s.k) for s in self.stages))
        return (self.i_f if self.i_f is not None else -1, self.mem, len(self.stages), canon)


_EMPTY = _Frag(None, (), 0.0)


@dataclass(frozen=True)
class _OpSet:
    """A stage candidate that is not an SP subtree (merge-join stages)."""

    ops: frozenset


class _DP:
    """One probe's memoised DP over the SP tree."""

    def __init__(self, ng: NormalizedGraph, cluster: DeviceCluster, B: int, t_max: float,
                 configs: list[tuple[int, int]], opts: PartitionOptions, uniform: bool):
        self.ng = ng
        self.g = ng.graph
        self.cluster = cluster
        self.B = B
        self.t_max = t_max
        self.configs = configs
        self.opts = opts
        self.uniform = uniform
        self.memo: dict = {}
        self.virtual = ng.virtual_ids
        self._tps_cache: dict = {}

    def real_ops(self, ops: frozenset) -> list[Operator]:
        return [self.g.by_id[o] for o in sorted(ops) if o not in self.virtual]

    def is_virtual(self, node) -> bool:
        return node.ops <= self.virtual

    def tps(self, ops: frozenset, b: int, d: int) -> float | None:
        key = (ops, b, d)
        if key not in self._tps_cache:
            cb = stage_comm_bytes(self.ng, ops)
            try:
                real = tuple(self.real_ops(ops))
                v = estimate_tps(StageCostInput(real, b, d, cb, cb, self.cluster))
                if self.opts.sync_per_iteration and d > 1:
                    sync = dp_sync_time(sum(o.param_bytes for o in real), d, self.cluster.intra_bw)
                    v = v - sync / b + sync / self.B
            except IndivisibleMicroBatchError:
                v = None
            self._tps_cache[key] = v
        return self._tps_cache[key]

    def boundary_configs(self, c_f):
        if self.uniform:
            return [(c_f[0], 1)]
        return self.configs

    # -- the three DP cases ------------------------------------------------
    def solve(self, node, c_f, c_b, d) -> _Frag | None:
        key = (node.ops, c_f, c_b, d)
        if key in self.memo:
            return self.memo[key]
        self.memo[key] = None  # cycle guard (cannot happen on a tree)
        res = self._solve(node, c_f, c_b, d)
        self.memo[key] = res
        return res

    def _consider(self, best, cand):
        if cand is None:
            return best
        if best is None or cand.key() < best.key():
            return cand
        return best

    def _base(self, node, c_f, c_b, d):
        """The whole node as a single stage on d devices (Alg. 1 base case)."""
        if self.is_virtual(node) or d < 1:
            return _EMPTY if (self.is_virtual(node) and d == 0) else None
        b_f, k_f = c_f
        t = self.tps(node.ops, b_f, d)
        if t is None or t > self.t_max:
            return None
        if c_b is None:
            i_f = b_f
        else:
            i_b, b_b, k_b = c_b
            i_f = round_up(compute_in_flight(k_f, b_f, k_b, b_b, i_b), b_f)
        i_f = min(i_f, self.B)
        mem = stage_memory(self.real_ops(node.ops), d, i_f, self.opts.weight_multiplier).total
        if mem > self.cluster.mem_per_device:
            return None
        return _Frag(i_f, (_FStage(node.ops, b_f, k_f, d, i_f, mem),), mem)

    def _solve(self, node, c_f, c_b, d):
        if self.is_virtual(node):
            return _EMPTY if d == 0 else None
        if d < 1:
            return None
        best = self._base(node, c_f, c_b, d)
        if isinstance(node, SPSeries):
            best = self._series(node, c_f, c_b, d, best)
        elif isinstance(node, SPParallel):
            best = self._parallel(node, c_f, c_b, d, best)
        return best

    def _series(self, node, c_f, c_b, d, best):
        # Every series cut (G1 ; G2) of the maximal chain, organised as a suffix DP:
        # G1 = the first segment units[0:q] (one stage, or a single unit solved
        # recursively), G2 = the rest.  This enumerates the same segmentations as
        # all cuts x all sub-chains, with O(n) instead of O(n^2) sub-problems.
        units = flatten_series(node)
        return self._consider(best, self._chain(tuple(units), 0, c_f, c_b, d))

    def _chain(self, units, start, c_f, c_b, d):
        key = ("chain", units[start].ops, len(units) - start, units[-1].ops, c_f, c_b, d)
        if key in self.memo:
            return self.memo[key]
        self.memo[key] = None
        best = None
        n = len(units)
        if start == n - 1:
            res = self.solve(units[start], c_f, c_b, d)
            self.memo[key] = res
            return res
        rest_virtual_from = [False] * (n + 1)
        rest_virtual_from[n] = True
        for q in range(n - 1, start - 1, -1):
            rest_virtual_from[q] = rest_virtual_from[q + 1] and self.is_virtual(units[q])
        if start > 0:  # whole remainder as one stage (start == 0: the node's own base case)
            best = self._consider(best, self._base(_as_series(list(units[start:])), c_f, c_b, d))
        for q in range(start + 1, n):
            seg_units = units[start:q]
            seg = _as_series(list(seg_units))
            if rest_virtual_from[q]:
                best = self._consider(best, self._segment(seg, c_f, c_b, d))
                continue
            if self.is_virtual(seg):
                best = self._consider(best, self._chain(units, q, c_f, c_b, d))
                continue
            any_ok = False
            for d1 in range(1, d):
                d2 = d - d1
                if len(seg_units) > 1:
                    t = self.tps(seg.ops, c_f[0], d1)
                    if t is None or t > self.t_max:
                        continue
                any_ok = True
                for c_m in self.boundary_configs(c_f):
                    r2 = self._chain(units, q, c_m, c_b, d2)
                    if r2 is None or r2.i_f is None:
                        continue
                    r1 = self._segment(seg, c_f, (r2.i_f, c_m[0], c_m[1]), d1)
                    if r1 is None:
                        continue
                    best = self._consider(best, _Frag(r1.i_f, r1.stages + r2.stages, max(r1.mem, r2.mem)))
            if not any_ok and len(seg_units) > 1 and d > 1:
                # TPS of a longer first segment on the same devices only grows; the
                # whole-remainder case (q == n) was already taken care of above.
                tps_all = [self.tps(seg.ops, c_f[0], d1) for d1 in range(1, d)]
                if all(t is not None and t > self.t_max for t in tps_all):
                    break
        if self.opts.merge_join and isinstance(units[start], SPParallel) and d >= 2:
            best = self._consider(best, self._merge_join(units, start, c_f, c_b, d, rest_virtual_from))
        self.memo[key] = best
        return best

    def _merge_join(self, units, start, c_f, c_b, d, rest_virtual_from):
        """Parallel unit P followed by a segment T: one branch group g of P and T form one
        stage M on d_m devices; the other branches o (d_o devices) feed M; the chain after T
        gets the remaining devices.  M is solved first (its successor is the rest of the
        chain), then o with M as its successor; the join takes the larger in-flight count."""
        par = units[start]
        n = len(units)
        best = None
        # wide bundles (DLRM's 27 branches): every merged-stage successor config would
        # re-solve all sub-bundles, so the extension is limited to <= 8 branches
        if len(flatten_parallel(par)) > self.opts.max_exhaustive_branches + 2:
            return None
        for q in range(start + 2, n + 1):
            tail = units[start + 1:q]
            if all(self.is_virtual(u) for u in tail):
                continue
            t_ops = frozenset().union(*(u.ops for u in tail))
            rest_virtual = rest_virtual_from[q]
            for n1, n2 in self._par_splits(par):
                for g, o in ((n1, n2), (n2, n1)):
                    if self.is_virtual(g) or self.is_virtual(o):
                        continue
                    m = _OpSet(g.ops | t_ops)
                    for d_m in range(1, d):
                        for d_o in range(1, d - d_m + 1):
                            d_r = d - d_m - d_o
                            if rest_virtual:
                                if d_r:
                                    continue
                                succs = [(c_b, None)]
                            else:
                                if d_r < 1:
                                    continue
                                succs = []
                                for c_m in self.boundary_configs(c_f):
                                    r2 = self._chain(units, q, c_m, c_b, d_r)
                                    if r2 is not None and r2.i_f is not None:
                                        succs.append(((r2.i_f, c_m[0], c_m[1]), r2))
                            for succ, r2 in succs:
                                rm = self._base(m, c_f, succ, d_m)
                                if rm is None:
                                    continue
                                ro = self.solve(o, c_f, (rm.i_f, c_f[0], c_f[1]), d_o)
                                if ro is None or ro.i_f is None:
                                    continue
                                stages = rm.stages + ro.stages + (r2.stages if r2 is not None else ())
                                mem = max([rm.mem, ro.mem] + ([r2.mem] if r2 is not None else []))
                                best = self._consider(best, _Frag(max(rm.i_f, ro.i_f), stages, mem))
        return best

    def _segment(self, seg, c_f, c_b, d):
        """A first segment: one stage (multi-unit) or a single unit solved recursively."""
        if isinstance(seg, SPSeries):
            return self._base(seg, c_f, c_b, d)
        return self.solve(seg, c_f, c_b, d)

    def _par_splits(self, node):
        kids = flatten_parallel(node)

        def bundle(children):
            children = tuple(children)
            if len(children) == 1:
                return children[0]
            return SPParallel(children=children, source=node.source, sink=node.sink, direct_edges=0)

        if len(kids) <= self.opts.max_exhaustive_branches:
            out = []
            seen = set()
            for one, rest in parallel_splits(node):
                out.append((bundle([c for c in kids if c.ops <= one]), bundle([c for c in kids if c.ops <= rest])))
                seen.add(frozenset((one, rest)))
            if self.opts.rich_splits:
                for k in range(2, len(kids) - 1):
                    one = frozenset().union(*(c.ops for c in kids[:k]))
                    rest = frozenset().union(*(c.ops for c in kids[k:]))
                    if frozenset((one, rest)) not in seen:
                        seen.add(frozenset((one, rest)))
                        out.append((bundle(kids[:k]), bundle(kids[k:])))
            return out
        return [(bundle(kids[:k]), bundle(kids[k:])) for k in range(1, len(kids))]

    def _parallel(self, node, c_f, c_b, d, best):
        for n1, n2 in self._par_splits(node):
            v1, v2 = self.is_virtual(n1), self.is_virtual(n2)
            lo1, lo2 = (0 if v1 else 1), (0 if v2 else 1)
            for d1 in range(lo1, d - lo2 + 1):
                d2 = d - d1
                if (d1 == 0) != v1 or (d2 == 0) != v2:
                    continue
                r1 = self.solve(n1, c_f, c_b, d1)
                if r1 is None:
                    continue
                r2 = self.solve(n2, c_f, c_b, d2)
                if r2 is None:
                    continue
                ifs = [x.i_f for x in (r1, r2) if x.i_f is not None]
                best = self._consider(best, _Frag(max(ifs) if ifs else None, r1.stages + r2.stages, max(r1.mem, r2.mem)))
        return best


def merge_join_applicable(g: ComputationGraph, opts: PartitionOptions | None = None) -> bool:
    """Whether PartitionOptions.merge_join can change the search on ``g``: some parallel
    bundle of <= max_exhaustive_branches + 2 branches exists."""
    limit = (opts or PartitionOptions()).max_exhaustive_branches + 2
    _, tree = _tree_and_graph(g)
    stack = [tree]
    while stack:
        n = stack.pop()
        if isinstance(n, SPParallel):
            kids = flatten_parallel(n)
            if len(kids) <= limit:
                return True
            stack.extend(kids)
        elif isinstance(n, SPSeries):
            stack.extend((n.left, n.right))
    return False


def _tree_and_graph(g: ComputationGraph):
    ng = normalize(g)
    return ng, decompose(ng)


def search_stage_graph(ng, tree, cluster, B, t_m, opts, configs, uniform):
    """One bisection probe (Alg. 1 SearchStageGraph). Returns (fragment, dp_states)."""
    dp = _DP(ng, cluster, B, t_m, configs, opts, uniform)
    best = None
    best_key = None
    # All devices first; fewer only if nothing fits (C3 does not require covering the
    # cluster, model.py:473-481, and MAXTPS is priced on ONE device, so it stays safe).
    for d_total in range(cluster.num_devices, 0, -1):
        for c in configs:
            frag = dp.solve(tree, c, None, d_total)
            if frag is None or not frag.stages:
                continue
            k = (frag.mem, len(frag.stages), frag.key()[3])
            if best is None or k < best_key:
                best, best_key = frag, k
        if best is not None:
            break
    return best, len(dp.memo)


def _to_stage_graph(g: ComputationGraph, ng: NormalizedGraph, frag: _Frag, B: int, opts: PartitionOptions,
                    chain: bool = False) -> StageGraph:
    topo_pos = {o: n for n, o in enumerate(g.topo_order)}
    real = [(s, frozenset(o for o in s.ops if o in g.by_id)) for s in frag.stages]
    real = [(s, ops) for s, ops in real if ops]
    real.sort(key=lambda t: min(topo_pos[o] for o in t[1]))
    stages = []
    dev = 0
    fixed_k = {}
    for sid, (s, ops) in enumerate(real):
        stages.append(Stage(id=sid, op_ids=ops, micro_batch=s.b, devices=frozenset(range(dev, dev + s.d))))
        fixed_k[sid] = s.k
        dev += s.d
    edges = set(induced_stage_edges(g, [st.op_ids for st in stages]))
    if chain:
        edges |= {(i, i + 1) for i in range(len(stages) - 1)}
    sg = StageGraph(stages, edges, B)
    cfg = schedule_stage_graph(sg, None, g, per_stage=False, fixed_k=fixed_k, weight_multiplier=opts.weight_multiplier)
    return cfg


def _optimize_on(g_eval: ComputationGraph, g_out: ComputationGraph, cluster: DeviceCluster, B: int,
                 opts: PartitionOptions, mode: str, chain: bool) -> Strategy:
    ng, tree = _tree_and_graph(g_eval)
    configs = candidate_configs(B, opts.per_stage_schedules)
    if opts.micro_batches is not None:
        configs = [c for c in configs if c[0] in opts.micro_batches]
    if not configs:
        raise NoFeasibleStrategy(f"no candidate micro-batch size divides B={B}")
    uniform = not opts.per_stage_schedules
    b_min = min(c[0] for c in configs)
    all_real = tuple(o for o in ng.graph.ops if o.id not in ng.virtual_ids)
    maxtps = 2.0 * estimate_tps(StageCostInput(all_real, b_min, 1, 0.0, 0.0, cluster))
    if maxtps <= 0:
        maxtps = 1.0
    eps = opts.epsilon_rel * maxtps
    probes = 0
    states = 0
    best, st = search_stage_graph(ng, tree, cluster, B, maxtps, opts, configs, uniform)
    probes += 1
    states += st
    if best is None:
        raise NoFeasibleStrategy("no strategy fits the memory budget even at MAXTPS")
    t_l, t_r = 0.0, maxtps
    while t_r - t_l > (eps if opts.epsilon_mode == "spec" else opts.epsilon_rel * t_r):
        t_m = (t_l + t_r) / 2.0
        cand, st = search_stage_graph(ng, tree, cluster, B, t_m, opts, configs, uniform)
        probes += 1
        states += st
        if cand is None:
            t_l = t_m
        else:
            t_r = t_m
            best = cand
    sg = _to_stage_graph(g_out, ng, best, B, opts, chain=chain)
    stage_tps = {}
    for fs in best.stages:
        if fs.ops <= ng.virtual_ids:
            continue
        cb = stage_comm_bytes(ng, fs.ops)
        real_ops = tuple(ng.graph.by_id[o] for o in sorted(fs.ops) if o not in ng.virtual_ids)
        v = estimate_tps(StageCostInput(real_ops, fs.b, fs.d, cb, cb, cluster))
        stage_tps[min(o for o in fs.ops if o not in ng.virtual_ids)] = v
    return Strategy(sg, max(stage_tps.values()), t_r, maxtps, probes, states, mode, stage_tps)


def optimize(g: ComputationGraph, cluster: DeviceCluster, B: int, opts: PartitionOptions | None = None) -> Strategy:
    """GPP strategy search (Alg. 1)."""
    opts = opts or PartitionOptions()
    return _optimize_on(g, g, cluster, B, opts, "gpp", chain=False)


def linearized_chain(g: ComputationGraph) -> ComputationGraph:
    """SPP view of g: ops in ``linearize`` order chained; each op's out-bytes are the
    bytes of every tensor live across the cut after it (what SPP must forward)."""
    order = linearize(g)
    pos = {o: n for n, o in enumerate(order)}
    ops = []
    for n, oid in enumerate(order):
        op = g.by_id[oid]
        crossing = {u for (u, v) in g.edges if pos[u] <= n < pos[v]}
        live = float(sum(g.by_id[u].out_bytes_per_sample for u in sorted(crossing)))
        ops.append(Operator(op.id, op.name, op.param_bytes, op.act_bytes_per_sample, live, op.fwd_cost, op.bwd_cost))
    edges = [(order[n], order[n + 1]) for n in range(len(order) - 1)]
    return ComputationGraph(ops, edges)


def spp_optimize(g: ComputationGraph, cluster: DeviceCluster, B: int, opts: PartitionOptions | None = None) -> Strategy:
    """SPP baseline: the same bisection + DP over ``linearize(g)``."""
    opts = opts or PartitionOptions()
    return _optimize_on(linearized_chain(g), g, cluster, B, opts, "spp", chain=True)
