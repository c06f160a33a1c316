"""Pins for the fp64 linear oracle (oracle/linear.c) — each against something
other than the oracle: the hand-worked fixture, library matmuls on special
cases, the isolation identity of Eq. 1-2, exact finite
differences / adjoint identities, integer exactness and NaN isolation.
"""
import json
import os

import numpy as np
import pytest

from oracle import linear as olin
import synth

GOLD = os.path.join(os.path.dirname(__file__), "golden")


def _rand_case(seed, K, N, seg_lens, ranks, scales=None, variant="normal"):
    rng = np.random.default_rng(seed)
    seg_off = np.concatenate([[0], np.cumsum(seg_lens)]).astype(np.int32)
    R = int(seg_off[-1])
    S = len(seg_lens)
    seg_task = np.arange(S, dtype=np.int32) % len(ranks)
    X = rng.standard_normal((R, K))
    W = rng.standard_normal((N, K)) / np.sqrt(K)
    dY = rng.standard_normal((R, N))
    A = [rng.standard_normal((r, K)) / np.sqrt(K) for r in ranks]
    B = [rng.standard_normal((N, r)) for r in ranks]
    if scales is None:
        scales = [float(1 + t) for t in range(len(ranks))]
    return dict(seg_off=seg_off, seg_task=seg_task, X=X, W=W, dY=dY, A=A, B=B,
                ranks=list(ranks), scales=list(scales))


def _fwd(c, r_cap=None, **kw):
    r_cap = r_cap or max(max(c["ranks"]), 1)
    return olin.linear_fwd(c["seg_off"], c["seg_task"], c["A"], c["B"], c["ranks"], c["scales"],
                           c["X"], c["W"], r_cap, **kw)


def _bwd(c, r_cap=None, **kw):
    r_cap = r_cap or max(max(c["ranks"]), 1)
    return olin.linear_bwd(c["seg_off"], c["seg_task"], c["A"], c["B"], c["ranks"], c["scales"],
                           c["dY"], c["X"], c["W"], r_cap, **kw)


# --------------------------------------------------------------- fixture L1
def test_fixture_L1():
    g = json.load(open(os.path.join(GOLD, "linear_L1.json")))
    c = dict(seg_off=np.array(g["seg_off"], np.int32), seg_task=np.array(g["seg_task"], np.int32),
             X=np.array(g["X"], float), W=np.array(g["W"], float), dY=np.array(g["dY"], float),
             A=[np.array(a, float) for a in g["A"]], B=[np.array(b, float) for b in g["B"]],
             ranks=[1, 1], scales=[float(s) for s in g["scale"]])
    Y, Hs = _fwd(c, 1)
    e = g["expect"]
    assert np.array_equal(Y, np.array(e["Y"], float))
    assert np.array_equal(Hs, np.array(e["Hs"], float))
    dX, Gs, grads = _bwd(c, 1)
    assert np.array_equal(dX, np.array(e["dX"], float))
    assert np.array_equal(Gs, np.array(e["Gs"], float))
    for t in range(2):
        assert np.array_equal(grads[t][0], np.array(e["dA"][t], float))
        assert np.array_equal(grads[t][1], np.array(e["dB"][t], float))


# --------------------------------------------------------------- special cases
def test_zero_B_is_backbone():
    """B_t = 0 (LoRA init) -> Y = X W^T (numpy matmul), dA = 0, dB != 0, dX = dY W."""
    c = _rand_case(1, 24, 20, [5, 7, 3], [4, 2, 3])
    c["B"] = [np.zeros_like(b) for b in c["B"]]
    Y, Hs = _fwd(c)
    np.testing.assert_allclose(Y, c["X"] @ c["W"].T, rtol=1e-12, atol=1e-12)
    dX, Gs, grads = _bwd(c)
    np.testing.assert_allclose(dX, c["dY"] @ c["W"], rtol=1e-12, atol=1e-12)
    for dA, dB in grads:
        assert np.all(dA == 0.0)
        assert np.any(dB != 0.0)


@pytest.mark.parametrize("which", ["A0", "s0", "r0"])
def test_no_adapter_is_backbone(which):
    ranks = [3, 2] if which != "r0" else [0, 0]
    c = _rand_case(2, 16, 12, [4, 6], ranks)
    if which == "A0":
        c["A"] = [np.zeros_like(a) for a in c["A"]]
    if which == "s0":
        c["scales"] = [0.0, 0.0]
    Y, Hs = _fwd(c, 4)
    np.testing.assert_allclose(Y, c["X"] @ c["W"].T, rtol=1e-12, atol=1e-12)
    assert np.all(Hs == 0.0)
    dX, Gs, grads = _bwd(c, 4)
    np.testing.assert_allclose(dX, c["dY"] @ c["W"], rtol=1e-12, atol=1e-12)
    if which == "A0":
        for dA, dB in grads:
            assert np.all(dB == 0.0)          # H = 0 -> dB = 0


def test_zero_W_is_pure_lora_and_identity_W():
    """W = 0 -> Y is the LoRA term alone; W = I (K = N) -> Y = X + LoRA term.
    The LoRA term is computed with numpy's matmul per segment."""
    c = _rand_case(3, 16, 16, [4, 5], [3, 2])
    lora = np.zeros((9, 16))
    for s in range(2):
        a, b = c["seg_off"][s], c["seg_off"][s + 1]
        t = c["seg_task"][s]
        lora[a:b] = c["scales"][t] * (c["X"][a:b] @ c["A"][t].T) @ c["B"][t].T
    c["W"] = np.zeros((16, 16))
    Y, _ = _fwd(c)
    np.testing.assert_allclose(Y, lora, rtol=1e-12, atol=1e-12)
    c["W"] = np.eye(16)
    Y, _ = _fwd(c)
    np.testing.assert_allclose(Y, c["X"] + lora, rtol=1e-12, atol=1e-12)


# --------------------------------------------------------------- isolation (Eq. 1-2)
def test_multiplexed_equals_each_task_alone_bitwise():
    """[X_1;X_2]W = [X_1 W; X_2 W] (and the bwd analogue): the
    multiplexed result of every task equals that task run alone, bitwise
    (fixed summation order)."""
    c = _rand_case(4, 32, 24, [6, 9, 4], [4, 1, 3])
    Y, Hs = _fwd(c)
    dX, Gs, grads = _bwd(c)
    for s in range(3):
        a, b = int(c["seg_off"][s]), int(c["seg_off"][s + 1])
        t = int(c["seg_task"][s])
        c1 = dict(c)
        c1.update(seg_off=np.array([0, b - a], np.int32), seg_task=np.array([0], np.int32),
                  X=c["X"][a:b], dY=c["dY"][a:b], A=[c["A"][t]], B=[c["B"][t]],
                  ranks=[c["ranks"][t]], scales=[c["scales"][t]])
        Y1, Hs1 = _fwd(c1, Hs.shape[1])
        dX1, Gs1, g1 = _bwd(c1, Hs.shape[1])
        assert np.array_equal(Y[a:b], Y1)
        assert np.array_equal(Hs[a:b], Hs1)
        assert np.array_equal(dX[a:b], dX1)
        assert np.array_equal(Gs[a:b], Gs1)
        assert np.array_equal(grads[t][0], g1[0][0])
        assert np.array_equal(grads[t][1], g1[0][1])


def test_task_owning_two_segments_equals_one_segment():
    c = _rand_case(5, 16, 12, [4, 3, 5], [2, 3])
    c["seg_task"] = np.array([0, 1, 0], np.int32)      # task 0 owns segments 0 and 2
    dX, Gs, grads = _bwd(c)
    # reorder rows so task 0's rows are contiguous: [seg0; seg2; seg1]
    idx = np.r_[0:4, 7:12, 4:7]
    c2 = dict(c)
    c2.update(seg_off=np.array([0, 9, 12], np.int32), seg_task=np.array([0, 1], np.int32),
              X=c["X"][idx], dY=c["dY"][idx])
    dX2, Gs2, g2 = _bwd(c2)
    assert np.array_equal(dX[idx], dX2)
    for t in range(2):
        np.testing.assert_allclose(grads[t][0], g2[t][0], rtol=1e-13, atol=1e-13)
        np.testing.assert_allclose(grads[t][1], g2[t][1], rtol=1e-13, atol=1e-13)


# --------------------------------------------------------------- gradients
def _loss(c):
    Y, _ = _fwd(c)
    return float(np.sum(c["dY"] * Y))


def test_adjoint_dX():
    """L = <dY, Y> is linear in X, so <dX, X'> = <dY, Y(X')> exactly (up to rounding)."""
    c = _rand_case(6, 20, 14, [5, 6], [3, 2])
    dX, _, _ = _bwd(c)
    rng = np.random.default_rng(60)
    for _ in range(3):
        Xp = rng.standard_normal(c["X"].shape)
        c2 = dict(c)
        c2["X"] = Xp
        lhs = float(np.sum(dX * Xp))
        rhs = _loss(c2)
        assert abs(lhs - rhs) <= 1e-10 * (1 + abs(rhs))


@pytest.mark.parametrize("which", ["A", "B"])
def test_finite_difference_adapter_grads(which):
    """L is linear in A_t (B fixed) and in B_t (A fixed): the central difference
    (L(P+E) - L(P-E)) / 2 equals <dP, E> up to rounding."""
    c = _rand_case(7, 18, 15, [4, 5, 3], [3, 2, 4])
    _, _, grads = _bwd(c)
    rng = np.random.default_rng(70)
    for t in range(3):
        E = rng.standard_normal(c[which][t].shape)
        cp, cm = dict(c), dict(c)
        cp[which] = list(c[which]); cm[which] = list(c[which])
        cp[which][t] = c[which][t] + E
        cm[which][t] = c[which][t] - E
        fd = (_loss(cp) - _loss(cm)) / 2.0
        g = grads[t][0] if which == "A" else grads[t][1]
        assert abs(float(np.sum(g * E)) - fd) <= 1e-9 * (1 + abs(fd))


# --------------------------------------------------------------- integer exactness
def test_integer_inputs_exact():
    """Integer-valued inputs (SURVEY §8(c) integer fixture): every fp64 sum is
    exact, so the oracle equals numpy's int64 matmuls exactly."""
    wl = synth.workload("1")
    rng = np.random.default_rng(8)
    K = N = 64
    seg_off = np.array([0, 64, 128], np.int32)
    X = rng.integers(-4, 5, (128, K))
    W = rng.integers(-4, 5, (N, K))
    dY = rng.integers(-4, 5, (128, N))
    A = [rng.integers(-2, 3, (8, K)), rng.integers(-2, 3, (8, K))]
    B = [rng.integers(-2, 3, (N, 8)), rng.integers(-2, 3, (N, 8))]
    sc = [1, 2]
    c = dict(seg_off=seg_off, seg_task=np.array([0, 1], np.int32), X=X.astype(float),
             W=W.astype(float), dY=dY.astype(float), A=[a.astype(float) for a in A],
             B=[b.astype(float) for b in B], ranks=[8, 8], scales=[1.0, 2.0])
    Y, Hs = _fwd(c)
    dX, Gs, grads = _bwd(c)
    for t in range(2):
        a, b = 64 * t, 64 * (t + 1)
        H = X[a:b] @ A[t].T
        G = dY[a:b] @ B[t]
        assert np.array_equal(Y[a:b], (X[a:b] @ W.T + sc[t] * H @ B[t].T).astype(float))
        assert np.array_equal(dX[a:b], (dY[a:b] @ W + sc[t] * G @ A[t]).astype(float))
        assert np.array_equal(Hs[a:b], (sc[t] * H).astype(float))
        assert np.array_equal(grads[t][0], (sc[t] * G.T @ X[a:b]).astype(float))
        assert np.array_equal(grads[t][1], (sc[t] * dY[a:b].T @ H).astype(float))


# --------------------------------------------------------------- NaN isolation
@pytest.mark.parametrize("where", ["X", "A", "B", "dY"])
def test_nan_isolation(where):
    c = _rand_case(9, 16, 12, [4, 6, 5], [2, 3, 2])
    a, b = 4, 10                     # segment 1 = task 1
    if where == "X":
        c["X"][a + 1, 3] = np.nan
    elif where == "dY":
        c["dY"][a + 2, 5] = np.nan
    else:
        c[where][1][0, 0] = np.nan
    Y, Hs = _fwd(c)
    dX, Gs, grads = _bwd(c)
    for arr in (Y, Hs, dX, Gs):
        assert np.all(np.isfinite(arr[:a])) and np.all(np.isfinite(arr[b:]))
    for t in (0, 2):
        assert np.all(np.isfinite(grads[t][0])) and np.all(np.isfinite(grads[t][1]))
    bad = np.concatenate([Y[a:b].ravel(), dX[a:b].ravel(), grads[1][0].ravel(), grads[1][1].ravel()])
    assert np.any(np.isnan(bad))


def test_row_sample_matches_full():
    c = _rand_case(10, 16, 12, [4, 6], [2, 3])
    Y, _ = _fwd(c)
    rows = np.array([9, 0, 5], np.int64)
    Ys, _ = _fwd(c, rows=rows)
    assert np.array_equal(Ys, Y[rows])
    dX, _, _ = _bwd(c)
    dXs, _, _ = _bwd(c, rows=rows)
    assert np.array_equal(dXs, dX[rows])


def test_hs_pad_columns_zero():
    c = _rand_case(11, 16, 12, [4, 6], [2, 5])
    Y, Hs = _fwd(c, 8)
    assert np.all(Hs[:4, 2:] == 0.0) and np.all(Hs[4:, 5:] == 0.0)


# ---------------------------------------------------------------- fused projections (column slices)
def _sliced_case(seed, K, col_off, seg_lens, ranks, scales):
    """ranks[t][s], scales[t][s]; B_{t,s} [slice width, rank]."""
    rng = np.random.default_rng(seed)
    N = col_off[-1]
    S = len(col_off) - 1
    seg_off = np.concatenate([[0], np.cumsum(seg_lens)]).astype(np.int32)
    R = int(seg_off[-1])
    seg_task = np.arange(len(seg_lens), dtype=np.int32) % len(ranks)
    A = [[rng.standard_normal((ranks[t][s], K)) / np.sqrt(K) for s in range(S)] for t in range(len(ranks))]
    B = [[rng.standard_normal((col_off[s + 1] - col_off[s], ranks[t][s])) for s in range(S)]
         for t in range(len(ranks))]
    return dict(seg_off=seg_off, seg_task=seg_task, col_off=list(col_off), A=A, B=B, ranks=ranks, scales=scales,
                X=rng.standard_normal((R, K)), W=rng.standard_normal((N, K)) / np.sqrt(K),
                dY=rng.standard_normal((R, N)))


def _block_diag_equivalent(c):
    """The same layer as ONE adapter per task of rank sum_s r_{t,s}: A = [A_{t,0}; A_{t,1}; ...]
    stacked, B = blockdiag(B_{t,0}, B_{t,1}, ...) (valid when a task's slices share one scale)."""
    S = len(c["col_off"]) - 1
    N = c["col_off"][-1]
    A, B, ranks, scales = [], [], [], []
    for t in range(len(c["ranks"])):
        rt = sum(c["ranks"][t])
        A.append(np.concatenate([c["A"][t][s] for s in range(S)], axis=0).reshape(rt, -1))
        Bt = np.zeros((N, rt))
        j = 0
        for s in range(S):
            r = c["ranks"][t][s]
            Bt[c["col_off"][s]:c["col_off"][s + 1], j:j + r] = c["B"][t][s]
            j += r
        B.append(Bt)
        ranks.append(rt)
        scales.append(c["scales"][t][0])
    return A, B, ranks, scales


def test_sliced_equals_block_diagonal_adapter():
    """Pin: stacking the slices' A and placing their B on a block diagonal gives one LoRA adapter of
    rank sum_s r_s whose product X A^T B^T is, column block by column block, X A_s^T B_s^T — so the
    sliced oracle must equal the plain oracle on that adapter (Y, Hs columns, dX, dA rows, dB
    diagonal blocks).  Catches a wrong slice offset, a transposed B slice or a dropped slice in the
    dX sum."""
    col_off = [0, 24, 40, 72]
    ranks = [[2, 3, 1], [4, 0, 2], [1, 1, 1]]
    scales = [[2.0] * 3, [0.5] * 3, [1.5] * 3]
    c = _sliced_case(7, 32, col_off, [5, 7, 3, 6], ranks, scales)
    r_cap = 4
    Y, Hs = olin.linear_fwd_sliced(c["seg_off"], c["seg_task"], col_off, c["A"], c["B"], ranks, scales, c["X"],
                                   c["W"], r_cap)
    dX, Gs, grads = olin.linear_bwd_sliced(c["seg_off"], c["seg_task"], col_off, c["A"], c["B"], ranks, scales,
                                           c["dY"], c["X"], c["W"], r_cap)
    A, B, rk, sc = _block_diagonal = _block_diag_equivalent(c)
    rc = max(rk)
    Y1, Hs1 = olin.linear_fwd(c["seg_off"], c["seg_task"], A, B, rk, sc, c["X"], c["W"], rc)
    dX1, Gs1, g1 = olin.linear_bwd(c["seg_off"], c["seg_task"], A, B, rk, sc, c["dY"], c["X"], c["W"], rc)
    np.testing.assert_array_equal(Y, Y1)       # zero off-block terms: same sums exactly
    np.testing.assert_allclose(dX, dX1, rtol=0, atol=1e-12 * np.max(np.abs(dX1)))  # sum split by slice
    seg_task = c["seg_task"]
    for i in range(int(c["seg_off"][-1])):
        t = int(seg_task[np.searchsorted(c["seg_off"], i, side="right") - 1])
        j = 0
        for s in range(3):
            r = ranks[t][s]
            np.testing.assert_array_equal(Hs[i, s * r_cap:s * r_cap + r], Hs1[i, j:j + r])
            np.testing.assert_array_equal(Hs[i, s * r_cap + r:(s + 1) * r_cap], 0.0)
            np.testing.assert_array_equal(Gs[i, s * r_cap:s * r_cap + r], Gs1[i, j:j + r])
            j += r
    for t in range(3):
        j = 0
        for s in range(3):
            r = ranks[t][s]
            dA, dB = grads[t][s]
            np.testing.assert_array_equal(dA, g1[t][0][j:j + r])
            np.testing.assert_array_equal(dB, g1[t][1][col_off[s]:col_off[s + 1], j:j + r])
            j += r


def test_sliced_rank0_slice_is_backbone_and_scales_are_per_slice():
    """Pin: a slice whose adapters all have rank 0 is the plain backbone X W_s^T (numpy matmul), and
    each slice uses its own scale (doubling s_{t,1} doubles only slice 1's LoRA term)."""
    col_off = [0, 16, 48]
    ranks = [[0, 2], [0, 3]]
    c = _sliced_case(11, 24, col_off, [4, 6], ranks, [[1.0, 1.0], [1.0, 1.0]])
    Y, _ = olin.linear_fwd_sliced(c["seg_off"], c["seg_task"], col_off, c["A"], c["B"], ranks,
                                  [[1.0, 1.0], [1.0, 1.0]], c["X"], c["W"], 4)
    np.testing.assert_allclose(Y[:, :16], c["X"] @ c["W"][:16].T, rtol=1e-13, atol=1e-13)
    Y2, _ = olin.linear_fwd_sliced(c["seg_off"], c["seg_task"], col_off, c["A"], c["B"], ranks,
                                   [[1.0, 2.0], [1.0, 2.0]], c["X"], c["W"], 4)
    base = c["X"] @ c["W"][16:].T
    np.testing.assert_allclose(Y2[:, 16:] - base, 2 * (Y[:, 16:] - base), rtol=1e-12, atol=1e-12)
    np.testing.assert_array_equal(Y2[:, :16], Y[:, :16])
