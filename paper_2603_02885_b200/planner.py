"""hTask planner: the cost model (Eq. 3, Eq. 4) and task fusion by dynamic
programming (Eq. 6) of paper §3.3 "Hybrid Task Abstraction",
SURVEY.md §8(f) NEXT-4.  Host-side logic only (no kernels): it decides which
tasks share one multiplexed `mux_linear_*` call (one hTask) and which run as
separate hTasks interleaved by orchestrate.py.

* Tasks are sorted ascending by token count n_i; an hTask
  H_{i->j} is a contiguous range of that order.
* Per-stage latency, Eq. 3:
      L^(s)(H) = sum_o t_o(sum_k n_k) / N_g^(s)
               + sum_a max( sum_k u_a(n_k) t_a(n_k),  max_k t_a(n_k) )
  t_o(x): latency of BaseOp o at x tokens; t_a / u_a: latency and GPU
  utilisation of adapter a at x tokens.
* End-to-end latency of an hTask over S pipeline stages with C micro-batches,
  Eq. 4:  L(H) = 2 sum_{s=1}^{S-1} L^(s)(H) + 2C max_s L^(s)(H).
* DP, Eq. 6, reading R20 in DESIGN.md:
      F(m, 1) = L(H_{1->m})
      F(m, n) = min_{n-1 <= i <= m-1} F(i, n-1) + L(H_{(i+1)->m}) / S
      F* = min_N F(M, N)
  (the paper's upper index `k` in H_{(i+1)->k} is read as m, and its range
  `i <= m` as i <= m-1 so the last hTask is non-empty).  Ties go to fewer
  hTasks, then to earlier split points.  An optional `feasible(i, j)` gate
  gives infinite cost to ranges that would not fit (the paper's memory model,
  Eq. 5, is out of scope here; the gate is the hook for it).

Measured profiles: `OpProfile` interpolates a table of (tokens, ms) measured
on the B200 with the fused kernels (tools/op_profile.py ->
profiles/r02_op_profile.json), piecewise linear, extrapolated linearly from
the last two points.
"""
from __future__ import annotations

import bisect
import json
import math
from dataclasses import dataclass, field
from typing import Callable, Dict, List, Optional, Sequence, Tuple


@dataclass(frozen=True)
class Task:
    name: str
    tokens: int          # n_i
    rank: int = 16


class OpProfile:
    """t(x) from a measured table: piecewise-linear in x, linear extrapolation
    beyond either end (clamped at >= 0)."""

    def __init__(self, xs: Sequence[float], ys: Sequence[float]):
        if len(xs) != len(ys) or len(xs) < 2:
            raise ValueError("a profile needs >= 2 points")
        pts = sorted(zip(map(float, xs), map(float, ys)))
        self.xs = [p[0] for p in pts]
        self.ys = [p[1] for p in pts]
        if len(set(self.xs)) != len(self.xs):
            raise ValueError("duplicate x in profile")

    def __call__(self, x: float) -> float:
        xs, ys = self.xs, self.ys
        j = bisect.bisect_right(xs, x)
        j = min(max(j, 1), len(xs) - 1)
        x0, x1, y0, y1 = xs[j - 1], xs[j], ys[j - 1], ys[j]
        return max(0.0, y0 + (y1 - y0) * (x - x0) / (x1 - x0))


@dataclass
class Stage:
    """One pipeline stage: BaseOps t_o (callables of the hTask's total tokens),
    fused adapters (t_a, u_a callables of one task's tokens), GPUs N_g."""
    base_ops: List[Callable[[float], float]]
    adapters: List[Tuple[Callable[[float], float], Callable[[float], float]]] = field(default_factory=list)
    n_gpus: int = 1


def stage_latency(stage: Stage, tokens: Sequence[int]) -> float:
    """Eq. 3 for the hTask whose tasks have token counts `tokens`."""
    n = float(sum(tokens))
    base = sum(t_o(n) for t_o in stage.base_ops) / stage.n_gpus
    adap = 0.0
    for t_a, u_a in stage.adapters:
        if not tokens:
            continue
        weighted = sum(u_a(k) * t_a(k) for k in tokens)
        adap += max(weighted, max(t_a(k) for k in tokens))
    return base + adap


def pipeline_latency(stage_lats: Sequence[float], C: int) -> float:
    """Eq. 4: warm-up + drain (2 x the first S-1 stages) + steady phase
    (2C x the slowest stage)."""
    S = len(stage_lats)
    if S == 0:
        raise ValueError("no stages")
    return 2.0 * sum(stage_lats[:S - 1]) + 2.0 * C * max(stage_lats)


def htask_latency(stages: Sequence[Stage], C: int) -> Callable[[Sequence[int]], float]:
    """L(H) as a function of the hTask's task token counts (Eq. 3 + Eq. 4)."""
    def L(tokens: Sequence[int]) -> float:
        return pipeline_latency([stage_latency(s, tokens) for s in stages], C)
    return L


@dataclass
class FusionPlan:
    order: List[Task]                       # tasks sorted ascending by tokens
    ranges: List[Tuple[int, int]]           # hTasks as [i, j) ranges of `order`
    cost: float                             # F*
    table: List[List[float]]                # F(m, n), m = 0..M, n = 0..M (inf where undefined)

    @property
    def htasks(self) -> List[List[Task]]:
        return [self.order[i:j] for i, j in self.ranges]


def sort_tasks(tasks: Sequence[Task]) -> List[Task]:
    """Ascending by token count; stable for equal counts."""
    return sorted(tasks, key=lambda t: t.tokens)


def fuse_tasks(tasks: Sequence[Task], L: Callable[[Sequence[int]], float], S: int = 1,
               max_htasks: Optional[int] = None,
               feasible: Optional[Callable[[int, int], bool]] = None) -> FusionPlan:
    """Eq. 6 over the sorted tasks.  L(tokens) = end-to-end latency of one
    hTask; S = pipeline stages; feasible(i, j) -> False marks H over sorted
    tasks [i, j) as infeasible (infinite cost)."""
    order = sort_tasks(tasks)
    M = len(order)
    if M == 0:
        raise ValueError("no tasks")
    Nmax = M if max_htasks is None else max(1, min(M, max_htasks))
    INF = math.inf
    memo: Dict[Tuple[int, int], float] = {}

    def cost(i: int, j: int) -> float:      # L(H over sorted tasks [i, j))
        key = (i, j)
        if key not in memo:
            ok = feasible is None or feasible(i, j)
            memo[key] = L([t.tokens for t in order[i:j]]) if ok else INF
        return memo[key]

    F = [[INF] * (M + 1) for _ in range(M + 1)]
    arg = [[-1] * (M + 1) for _ in range(M + 1)]
    for m in range(1, M + 1):
        F[m][1] = cost(0, m)
    for n in range(2, Nmax + 1):
        for m in range(n, M + 1):
            best, bi = INF, -1
            for i in range(n - 1, m):          # last hTask = sorted tasks [i, m), non-empty
                v = F[i][n - 1] + cost(i, m) / S
                if v < best:                    # strict: ties keep the earliest split
                    best, bi = v, i
            F[m][n], arg[m][n] = best, bi
    best_n, best = 1, F[M][1]
    for n in range(2, Nmax + 1):
        if F[M][n] < best:                      # strict: ties keep fewer hTasks
            best, best_n = F[M][n], n
    if best == INF:
        raise ValueError("every partition is infeasible")
    ranges: List[Tuple[int, int]] = []
    m, n = M, best_n
    while n > 1:
        i = arg[m][n]
        ranges.append((i, m))
        m, n = i, n - 1
    ranges.append((0, m))
    ranges.reverse()
    return FusionPlan(order, ranges, best, F)


# ------------------------------------------------------------------ measured profiles
def load_profile(path: str) -> dict:
    """profiles/r02_op_profile.json (tools/op_profile.py): per linear shape, a
    table of fused fwd+bwd latency (ms) vs packed tokens for rank-0 (BaseOp
    only) and rank-r adapters."""
    with open(path) as f:
        return json.load(f)


def stage_from_profile(prof: dict, n_gpus: int = 1) -> Stage:
    """A single-stage model of the profiled layer stack: one BaseOp per linear
    (rank-0 timings, halved to one pass), adapters folded in as (extra latency of the rank-r run,
    utilisation 1).  The adapters run inside the fused kernel (R18), so their
    cost is additive and fully utilised: max(sum, max) = sum."""
    # Eq. 3 is one pass; Eq. 4's factor 2 adds the backward (fwd ~ bwd without
    # dW).  The profile times fwd+bwd, so one pass = half.
    base, adap = [], []
    for lin in prof["linears"]:
        xs = lin["tokens"]
        base.append(OpProfile(xs, [0.5 * v for v in lin["ms_rank0"]]))
        extra = [0.5 * max(0.0, a - b) for a, b in zip(lin["ms_rank"], lin["ms_rank0"])]
        # per-task adapter latency at k tokens: the extra cost scales with that task's rows
        adap.append((OpProfile(xs, extra), lambda k: 1.0))
    return Stage(base, adap, n_gpus)
