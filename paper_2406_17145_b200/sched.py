"""Static micro-batch scheduler (§6, Alg. 2, Appendix A).

* ``compute_in_flight`` — the 10-row Appendix-A table,
  rows tried in table order, raising ``NoConditionMatches`` outside its domain;
* ``choose_k`` — argmin_k max over successors, smallest k on ties;
* ``schedule_tasks`` — kFkB task list: l = i/b warm-up forwards, then blocks of
  k backwards / k forwards, then the remaining backwards;
* ``schedule_stage`` — Alg. 2 ScheduleStage with the Eq. (2) memory check;
* ``schedule_stage_graph`` — reverse-topological pass over a StageGraph, the
  parallel-join rule taking the max over successors.

The reference ships no code for this module; this is the
SPEC/PAPER restatement the runtime executes.  In-flight counts are in SAMPLES
(``i``), rounded up to a multiple of the stage micro-batch.
"""

from __future__ import annotations

from dataclasses import dataclass
from typing import Iterable, Mapping, Sequence

from .cost import DEFAULT_WEIGHT_MULTIPLIER, stage_memory
from .model import ComputationGraph, ScheduleConfig, StageGraph, Task, TaskSchedule

__all__ = [
    "NoConditionMatches",
    "InFlightQuery",
    "compute_in_flight",
    "matched_row",
    "choose_k",
    "round_up",
    "schedule_tasks",
    "schedule_stage",
    "schedule_stage_graph",
]


class NoConditionMatches(ValueError):
    """(k_x, b_x, k_y, b_y, i_y) lies outside every Appendix-A row."""

    def __init__(self, q: "InFlightQuery"):
        self.query = q
        super().__init__(f"no Appendix-A condition matches {q}")


@dataclass(frozen=True)
class InFlightQuery:
    k_x: int
    b_x: int
    k_y: int
    b_y: int
    i_y: int

    def __post_init__(self):
        if min(self.k_x, self.b_x, self.k_y, self.b_y, self.i_y) < 1:
            raise ValueError("in-flight query fields must be >= 1")


def _rows(q: InFlightQuery):
    """(row number, condition, result) for the 10 rows of PAPER.md:1058-1067, in order."""
    bx, by, iy = q.b_x, q.b_y, q.i_y
    X, Y = q.k_x * q.b_x, q.k_y * q.b_y
    m = max(bx, by)
    return (
        (1, m < X < Y, iy + 2 * m),
        (2, m == X < Y, iy + m),
        (3, bx <= by < Y < X, iy + X - Y + 2 * by),
        (4, bx <= by == Y < X, iy + X),
        (5, by <= bx < Y < X, iy + X - Y + 2 * bx),
        (6, by <= bx == Y < X, iy + X),
        (7, m == Y == X, iy + Y),
        (8, m < Y == X, iy + 2 * m),
        (9, bx <= X < by <= Y, iy + by),
        (10, by <= Y < bx <= X, iy + X - Y + bx),
    )


def matched_row(q: InFlightQuery) -> int:
    for row, cond, _ in _rows(q):
        if cond:
            return row
    raise NoConditionMatches(q)


def compute_in_flight(k_x: int, b_x: int, k_y: int, b_y: int, i_y: int) -> int:
    """Minimum in-flight SAMPLES of stage x given its successor y (Appendix A table)."""
    q = InFlightQuery(k_x, b_x, k_y, b_y, i_y)
    for _, cond, result in _rows(q):
        if cond:
            return result
    raise NoConditionMatches(q)


def round_up(i: int, b: int) -> int:
    return -(-i // b) * b


def choose_k(
    b_x: int,
    successors: Sequence[tuple[int, int, int]],
    mini_batch: int,
    candidates: Iterable[int] | None = None,
) -> tuple[int, int]:
    """argmin_k max_y ComputeInFlight(k, b_x, k_y, b_y, i_y); returns (k, i rounded up).

    ``successors`` holds (k_y, b_y, i_y) per successor.  No successors: the stage
    waits for nothing, so k = 1 and i = b.
    """
    if not successors:
        return 1, b_x
    ks = list(candidates) if candidates is not None else list(range(1, mini_batch // b_x + 1))
    best_k, best_i = None, None
    for k in ks:
        i = max(compute_in_flight(k, b_x, ky, by, iy) for ky, by, iy in successors)
        if best_i is None or i < best_i:  # strict: ties keep the smaller k
            best_k, best_i = k, i
    return best_k, round_up(best_i, b_x)


def schedule_tasks(cfg: ScheduleConfig, mini_batch: int) -> TaskSchedule:
    """kFkB list for c = (i, b, k): l=i/b forwards, [k bw, <=k fw]*, remaining bw.

    Backward blocks never exceed the forwards already issued, so C4 always holds.
    """
    n = mini_batch // cfg.micro_batch
    warm = cfg.warmup_microbatches
    if warm > n:
        raise ValueError(f"warm-up of {warm} micro-batches exceeds the {n} micro-batches of a mini-batch")
    out: list[Task] = [Task("fw", j) for j in range(warm)]
    nf, nb = warm, 0
    while nf < n:
        for _ in range(min(cfg.k, nf - nb)):
            out.append(Task("bw", nb))
            nb += 1
        for _ in range(min(cfg.k, n - nf)):
            out.append(Task("fw", nf))
            nf += 1
    out.extend(Task("bw", j) for j in range(nb, n))
    return tuple(out)


def schedule_stage(
    ops: Sequence,
    b_f: int,
    k_f: int,
    c_b: tuple[int, int, int] | None,
    dp_degree: int,
    mini_batch: int,
    mem_limit: float | None = None,
    weight_multiplier: float = DEFAULT_WEIGHT_MULTIPLIER,
):
    """Alg. 2 ScheduleStage: (ScheduleConfig, TaskSchedule), or None if over memory.

    ``c_b`` = (i_b, b_b, k_b) of the successor stage, or None for a sink stage.
    """
    if c_b is None:
        i_f = b_f
    else:
        i_b, b_b, k_b = c_b
        i_f = min(round_up(compute_in_flight(k_f, b_f, k_b, b_b, i_b), b_f), mini_batch)
    if mem_limit is not None:
        if stage_memory(ops, dp_degree, i_f, weight_multiplier).total > mem_limit:
            return None
    cfg = ScheduleConfig(inflight_samples=i_f, micro_batch=b_f, k=k_f)
    return cfg, schedule_tasks(cfg, mini_batch)


def schedule_stage_graph(
    s: StageGraph,
    mem_limit: float | None = None,
    g: ComputationGraph | None = None,
    per_stage: bool = False,
    fixed_k: Mapping[int, int] | None = None,
    weight_multiplier: float = DEFAULT_WEIGHT_MULTIPLIER,
) -> StageGraph | None:
    """Configure every stage in reverse topological order.

    Default mode: k = 1 (graph-adjusted 1F1B).  ``per_stage``:
    k from ``choose_k`` over powers of two <= B/b.  ``fixed_k``
    pins k per stage (the partitioner's choice).  Returns None if any stage's
    Eq. (2) memory exceeds ``mem_limit`` (needs ``g`` for op byte counts).
    """
    cfgs: dict[int, ScheduleConfig] = {}
    scheds: dict[int, TaskSchedule] = {}
    B = s.mini_batch
    for sid in reversed(s.topo_order()):
        st = s.by_id[sid]
        succ = [(cfgs[y].k, cfgs[y].micro_batch, cfgs[y].inflight_samples) for y in s.successors(sid)]
        if fixed_k is not None and sid in fixed_k:
            ks = [fixed_k[sid]]
        elif per_stage:
            ks = [1 << e for e in range(0, 64) if (1 << e) <= B // st.micro_batch]
        else:
            ks = [1]
        if succ:
            k, i = choose_k(st.micro_batch, succ, B, ks)
            i = min(i, B)  # a stage never holds more than the whole mini-batch
        else:
            k, i = (ks[0] if fixed_k is not None and sid in fixed_k else 1), st.micro_batch
        if mem_limit is not None and g is not None:
            ops = [g.by_id[o] for o in st.op_ids if o in g.by_id]
            if stage_memory(ops, st.dp_degree, i, weight_multiplier).total > mem_limit:
                return None
        cfgs[sid] = ScheduleConfig(inflight_samples=i, micro_batch=st.micro_batch, k=k)
        scheds[sid] = schedule_tasks(cfgs[sid], B)
    return s.with_schedules(cfgs, scheds)
