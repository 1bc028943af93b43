"""TEST INFRASTRUCTURE ONLY.  SPEC oracle module: brute-force ground truth.

* ``exhaustive_optimize`` — every partition of the ops into convex blocks with an
  acyclic induced stage graph, every split of the cluster's devices over the
  blocks, every uniform power-of-two micro-batch size; stages priced with the
  same cost model (``cost.estimate_tps``) and scheduled with the same scheduler
  (Eq. (2) memory check) -> the min-max bottleneck TPS (Eq. (1)).
* ``min_inflight_search`` — see ``sim.measure_min_inflight`` (two-stage chains).
"""

from __future__ import annotations

import itertools
from dataclasses import dataclass

from paper_2406_17145_b200.cost import IndivisibleMicroBatchError, StageCostInput, estimate_tps
from paper_2406_17145_b200.model import ComputationGraph, DeviceCluster, Stage, StageGraph, induced_stage_edges
from paper_2406_17145_b200.model import _leaves_and_reenters as non_convex
from paper_2406_17145_b200.partition import candidate_configs
from paper_2406_17145_b200.sched import schedule_stage_graph


class BudgetExceeded(RuntimeError):
    pass


@dataclass
class BruteResult:
    tps: float
    blocks: list
    devices: list
    b: int


def _set_partitions(items):
    if not items:
        yield []
        return
    first, rest = items[0], items[1:]
    for part in _set_partitions(rest):
        for i in range(len(part)):
            yield part[:i] + [[first] + part[i]] + part[i + 1:]
        yield [[first]] + part


def _compositions(total, k):
    if k == 1:
        yield (total,)
        return
    for first in range(1, total - k + 2):
        for rest in _compositions(total - first, k - 1):
            yield (first,) + rest


def _in_bytes(g: ComputationGraph, block: frozenset) -> float:
    prods = sorted({u for v in block for u in g.predecessors(v) if u not in block})
    return float(sum(g.by_id[u].out_bytes_per_sample for u in prods))


def _acyclic(n, edges):
    indeg = [0] * n
    for _, b in edges:
        indeg[b] += 1
    ready = [i for i in range(n) if indeg[i] == 0]
    seen = 0
    while ready:
        x = ready.pop()
        seen += 1
        for a, b in edges:
            if a == x:
                indeg[b] -= 1
                if indeg[b] == 0:
                    ready.append(b)
    return seen == n


def sp_stage_candidates(g: ComputationGraph, cluster: DeviceCluster, B: int) -> set[frozenset]:
    """Every op set the SP-DP of ``partition.optimize`` can make a stage of:
    recorded from the DP's base case (Alg. 1 line "the whole node as one stage") while it
    explores with an unbounded t_max, virtual junction ops stripped.  Restricting the brute
    force to these blocks gives the optimum over SP-aligned partitions -- the space the
    SPEC's DP searches -- against which optimize must match exactly (acceptance 4)."""
    from paper_2406_17145_b200 import partition as P

    seen: set[frozenset] = set()
    orig = P._DP._base

    def rec(self, node, c_f, c_b, d):
        real = frozenset(o for o in node.ops if o not in self.virtual)
        if real:
            seen.add(real)
        return orig(self, node, c_f, c_b, d)

    P._DP._base = rec
    try:
        P.optimize(g, cluster, B, P.PartitionOptions(epsilon_mode="spec"))
    finally:
        P._DP._base = orig
    return seen


def exhaustive_optimize(g: ComputationGraph, cluster: DeviceCluster, B: int, max_ops: int = 8,
                        allowed_blocks: set | None = None) -> BruteResult | None:
    """``allowed_blocks``: only partitions whose every block is in the set (e.g.
    ``sp_stage_candidates``)."""
    ops = [o.id for o in g.ops]
    if len(ops) > max_ops or cluster.num_devices > 4 or B > 16:
        raise BudgetExceeded(f"{len(ops)} ops / {cluster.num_devices} devices / B={B}")
    best: BruteResult | None = None
    for part in _set_partitions(ops):
        blocks = [frozenset(b) for b in part]
        if len(blocks) > cluster.num_devices:
            continue
        if allowed_blocks is not None and any(blk not in allowed_blocks for blk in blocks):
            continue
        if any(non_convex(g, blk) for blk in blocks):
            continue
        edges = induced_stage_edges(g, blocks)
        if not _acyclic(len(blocks), edges):
            continue
        for devs in (c for tot in range(len(blocks), cluster.num_devices + 1) for c in _compositions(tot, len(blocks))):
            for b, _ in candidate_configs(B):
                tps = []
                ok = True
                for blk, d in zip(blocks, devs):
                    cb = _in_bytes(g, blk)
                    try:
                        tps.append(estimate_tps(StageCostInput(tuple(g.by_id[o] for o in sorted(blk)), b, d, cb, cb, cluster)))
                    except IndivisibleMicroBatchError:
                        ok = False
                        break
                if not ok:
                    continue
                t = max(tps)
                if best is not None and t >= best.tps:
                    continue
                stages, dev0 = [], 0
                for i, (blk, d) in enumerate(zip(blocks, devs)):
                    stages.append(Stage(i, blk, b, frozenset(range(dev0, dev0 + d))))
                    dev0 += d
                sg = schedule_stage_graph(StageGraph(stages, edges, B), cluster.mem_per_device, g)
                if sg is None:
                    continue
                best = BruteResult(t, [sorted(x) for x in blocks], list(devs), b)
    return best
