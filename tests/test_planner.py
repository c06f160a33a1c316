"""hTask planner (paper_2603_02885_b200/planner.py; Eq. 3, 4, 6 of P:546-611,
SURVEY §8(f) NEXT-4).  Pins: hand-computed values of Eq. 3 / Eq. 4, the DP
against exhaustive enumeration of every contiguous partition (the recurrence's
objective written out independently), the tie rules, the infeasibility gate
and the fuse-below / split-above-saturation shape of Fig. 6(a)."""
import itertools
import math
import random

import pytest

from paper_2603_02885_b200 import planner as pl


def test_profile_interpolation():
    p = pl.OpProfile([100, 200, 400], [1.0, 1.5, 3.5])
    assert p(100) == 1.0 and p(200) == 1.5 and p(400) == 3.5
    assert p(150) == pytest.approx(1.25)
    assert p(300) == pytest.approx(2.5)
    assert p(600) == pytest.approx(5.5)          # extrapolated from the last segment
    assert p(0) == pytest.approx(0.5)            # and from the first
    assert pl.OpProfile([0, 10], [0, -1])(5) == 0.0   # clamped at 0
    with pytest.raises(ValueError):
        pl.OpProfile([1], [1])


def test_stage_latency_eq3_by_hand():
    ident = lambda x: float(x)  # noqa: E731
    st = pl.Stage([ident, ident], [(ident, lambda k: 0.5)], n_gpus=2)
    # base: 2 ops x 8 tokens / 2 GPUs = 8; adapter: max(0.5*(2+6), max(2, 6)) = 6
    assert pl.stage_latency(st, [2, 6]) == 14.0
    # base 15; adapter max(0.5*15, 5) = 7.5
    assert pl.stage_latency(st, [5, 5, 5]) == 22.5
    # two adapter groups add
    st2 = pl.Stage([ident], [(ident, lambda k: 1.0), (lambda k: 3.0, lambda k: 0.1)], n_gpus=1)
    # base 4; a1: max(4, 3) = 4; a2: max(0.1*3*2, 3) = 3
    assert pl.stage_latency(st2, [1, 3]) == 11.0


def test_pipeline_latency_eq4_by_hand():
    assert pl.pipeline_latency([1.0, 2.0, 3.0], C=4) == 2 * (1 + 2) + 2 * 4 * 3
    assert pl.pipeline_latency([5.0], C=2) == 20.0
    assert pl.pipeline_latency([3.0, 1.0], C=1) == 2 * 3 + 2 * 3
    with pytest.raises(ValueError):
        pl.pipeline_latency([], C=1)


def _brute(order_tokens, L, S):
    """min over every contiguous partition of L(first) + sum_rest L(part)/S."""
    M = len(order_tokens)
    best = (math.inf, None)
    for mask in range(1 << (M - 1)):
        cuts = [0] + [g + 1 for g in range(M - 1) if mask >> g & 1] + [M]
        parts = [order_tokens[a:b] for a, b in zip(cuts, cuts[1:])]
        c = L(parts[0]) + sum(L(p) for p in parts[1:]) / S
        if c < best[0] - 1e-12 * max(1.0, abs(c)):
            best = (c, parts)
    return best


def _sat_profile(rng):
    """saturating latency: flat up to a knee, then linear (GPU saturation)."""
    knee = rng.choice([256, 1024, 4096])
    c0 = rng.uniform(0.2, 2.0)
    return lambda x: c0 * max(1.0, x / knee)


def test_dp_equals_exhaustive_partitions():
    rng = random.Random(5)
    for _ in range(150):
        M = rng.randint(1, 8)
        tasks = [pl.Task(f"t{i}", rng.randint(64, 4096)) for i in range(M)]
        stages = [pl.Stage([_sat_profile(rng) for _ in range(rng.randint(1, 3))],
                           [(lambda k, a=rng.uniform(1e-4, 1e-3): a * k, lambda k: 0.5)],
                           n_gpus=rng.choice([1, 2, 4]))
                  for _ in range(rng.choice([1, 2, 4]))]
        S = len(stages)
        C = rng.choice([1, 4, 8])
        L = pl.htask_latency(stages, C)
        plan = pl.fuse_tasks(tasks, L, S)
        toks = [t.tokens for t in plan.order]
        assert toks == sorted(toks)
        want, _ = _brute(toks, L, S)
        assert plan.cost == pytest.approx(want, rel=1e-12)
        # the returned ranges realise F*
        parts = [toks[a:b] for a, b in plan.ranges]
        assert [a for a, _ in plan.ranges][0] == 0 and plan.ranges[-1][1] == M
        assert all(b == c for (_, b), (c, _) in zip(plan.ranges, plan.ranges[1:]))
        got = L(parts[0]) + sum(L(p) for p in parts[1:]) / S
        assert got == pytest.approx(plan.cost, rel=1e-12)


def test_single_task_and_ties():
    L = lambda toks: float(sum(toks))  # noqa: E731
    plan = pl.fuse_tasks([pl.Task("a", 7)], L, S=1)
    assert plan.ranges == [(0, 1)] and plan.cost == 7.0
    # linear cost and S = 1: every partition costs the same -> the fewest hTasks
    plan = pl.fuse_tasks([pl.Task(str(i), 10 * (i + 1)) for i in range(5)], L, S=1)
    assert plan.ranges == [(0, 5)]
    # a constant per-hTask cost with S = 2: any split into 2 costs 1.5 (< 2 fused? no: fused = 1)
    plan = pl.fuse_tasks([pl.Task(str(i), 1) for i in range(4)], lambda t: 1.0, S=2)
    assert plan.ranges == [(0, 4)] and plan.cost == 1.0
    # equal-cost splits: the earliest split point wins
    L2 = lambda toks: 1.0 if len(toks) <= 2 else 100.0  # noqa: E731
    plan = pl.fuse_tasks([pl.Task(str(i), 5) for i in range(3)], L2, S=1)
    assert plan.ranges == [(0, 1), (1, 3)] and plan.cost == 2.0
    with pytest.raises(ValueError):
        pl.fuse_tasks([], L, S=1)


def test_sorting_is_ascending_and_stable():
    ts = [pl.Task("a", 30), pl.Task("b", 10), pl.Task("c", 30), pl.Task("d", 20)]
    assert [t.name for t in pl.sort_tasks(ts)] == ["b", "d", "a", "c"]


def test_fig6a_fuse_below_saturation_split_above():
    """Two tasks on a 4-stage pipeline, C = 4, a BaseOp flat up to a knee of
    2048 tokens then linear: batching wins while the GPU is unsaturated,
    interleaving wins beyond saturation (Fig. 6(a))."""
    t_o = lambda x: max(1.0, x / 2048.0)  # noqa: E731
    stages = [pl.Stage([t_o]) for _ in range(4)]
    L = pl.htask_latency(stages, C=4)
    small = pl.fuse_tasks([pl.Task("a", 512), pl.Task("b", 512)], L, S=4)
    assert small.ranges == [(0, 2)]
    big = pl.fuse_tasks([pl.Task("a", 8192), pl.Task("b", 8192)], L, S=4)
    assert big.ranges == [(0, 1), (1, 2)]
    # at the knee: fused 1 unit, split 1 + 1/4 -> fused
    knee = pl.fuse_tasks([pl.Task("a", 1024), pl.Task("b", 1024)], L, S=4)
    assert knee.ranges == [(0, 2)]


def test_feasibility_gate():
    L = lambda toks: 1.0  # noqa: E731   (fusing everything would be optimal)
    tasks = [pl.Task(str(i), 100 * (i + 1)) for i in range(4)]
    # at most 2 tasks per hTask fit
    plan = pl.fuse_tasks(tasks, L, S=2, feasible=lambda i, j: j - i <= 2)
    assert all(b - a <= 2 for a, b in plan.ranges)
    assert plan.ranges == [(0, 2), (2, 4)] and plan.cost == 1.5
    with pytest.raises(ValueError):
        pl.fuse_tasks(tasks, L, S=1, feasible=lambda i, j: False)


def test_max_htasks_cap_and_table():
    rng = random.Random(9)
    tasks = [pl.Task(str(i), rng.randint(100, 5000)) for i in range(6)]
    L = pl.htask_latency([pl.Stage([lambda x: max(1.0, x / 1500.0)])] * 2, C=2)
    plan = pl.fuse_tasks(tasks, L, S=2, max_htasks=2)
    assert len(plan.ranges) <= 2
    toks = [t.tokens for t in plan.order]
    best2 = min(L(toks[:i]) + L(toks[i:]) / 2 for i in range(1, 6))
    assert plan.cost == pytest.approx(min(best2, L(toks)), rel=1e-12)
    # F(m, 1) = L(H_{1->m}) (the base case as written)
    for m in range(1, 7):
        assert plan.table[m][1] == pytest.approx(L(toks[:m]))


def test_stage_from_profile_roundtrip():
    prof = {"linears": [{"shape": [4096, 4096], "tokens": [512, 1024, 2048],
                         "ms_rank0": [0.1, 0.15, 0.25], "ms_rank": [0.12, 0.18, 0.3]}]}
    st = pl.stage_from_profile(prof)
    # one pass = half the fwd+bwd profile: base 0.15/2 at 1024 tokens;
    # adapters (u = 1): (extra(512) + extra(512)) / 2 = (0.02 + 0.02) / 2
    assert pl.stage_latency(st, [512, 512]) == pytest.approx(0.075 + 0.02)
    # with S = 1, C = 1, Eq. 4 doubles it back to the fwd+bwd time
    assert pl.htask_latency([st], C=1)([512, 512]) == pytest.approx(0.19)
