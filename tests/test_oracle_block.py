"""Pins for the fp64 decoder-block oracle (oracle/block.py, NEXT-3), each
against something other than the oracle's own formula: closed forms on
special inputs, invariances, the sequence-isolation identity of packing
(a packed sequence attends exactly as it would alone), causality,
orthogonality / relative-position identities of RoPE, and central finite
differences for every backward (fp64, tiny shapes)."""
import numpy as np
import pytest

from oracle import block as ob


def _fd(f, x, dy, h=1e-6):
    """central finite-difference gradient of <dy, f(x)> w.r.t. x."""
    g = np.zeros_like(x)
    it = np.nditer(x, flags=["multi_index"])
    for _ in it:
        i = it.multi_index
        xp, xm = x.copy(), x.copy()
        xp[i] += h
        xm[i] -= h
        g[i] = (np.sum(dy * f(xp)) - np.sum(dy * f(xm))) / (2 * h)
    return g


# ------------------------------------------------------------------ row map
def test_row_seq_start_from_pack_fixture():
    # pack fixture P1 (tests/golden/pack_P1.json): seq_row [0,40,64,94,128], lens [40,20,30,30,100]
    rs = ob.row_seq_start([0, 40, 64, 94, 128], [40, 20, 30, 30, 100], 256)
    assert (rs[0:40] == 0).all() and (rs[40:60] == 40).all() and (rs[60:64] == -1).all()
    assert (rs[64:94] == 64).all() and (rs[94:124] == 94).all() and (rs[124:128] == -1).all()
    assert (rs[128:228] == 128).all() and (rs[228:] == -1).all()
    assert ob._sequences(rs) == [(0, 40), (40, 20), (64, 30), (94, 30), (128, 100)]


# ------------------------------------------------------------------ RMSNorm
def test_rmsnorm_closed_forms():
    rng = np.random.default_rng(0)
    x = rng.standard_normal((5, 16))
    w = np.full(16, 3.0)
    y = ob.rmsnorm_fwd(x, w, 0.0)
    np.testing.assert_allclose(np.sqrt(np.mean(y * y, axis=1)), 3.0, rtol=1e-13)   # RMS = |w|
    np.testing.assert_allclose(ob.rmsnorm_fwd(7.5 * x, w, 0.0), y, rtol=1e-13)     # scale invariant
    # a constant row c: y = sign(c) * w (eps = 0)
    np.testing.assert_allclose(ob.rmsnorm_fwd(np.full((1, 4), -2.0), np.arange(4.0), 0.0), [[-0., -1., -2., -3.]])


def test_rmsnorm_bwd_fd_and_orthogonality():
    rng = np.random.default_rng(1)
    x = rng.standard_normal((3, 8))
    w = rng.standard_normal(8)
    dy = rng.standard_normal((3, 8))
    dx = ob.rmsnorm_bwd(dy, x, w, 1e-5)
    np.testing.assert_allclose(dx, _fd(lambda t: ob.rmsnorm_fwd(t, w, 1e-5), x, dy), rtol=1e-6, atol=1e-8)
    # eps = 0: y(c x) = y(x)  =>  <dx, x> = 0 per row
    dx0 = ob.rmsnorm_bwd(dy, x, w, 0.0)
    np.testing.assert_allclose(np.sum(dx0 * x, axis=1), 0.0, atol=1e-12)


# ------------------------------------------------------------------ SwiGLU
def test_swiglu_special_points_and_fd():
    g = np.array([0.0, 50.0, -50.0, 1.0])
    u = np.array([2.0, 3.0, 4.0, 1.0])
    h = ob.swiglu_fwd(g, u)
    assert h[0] == 0.0
    assert h[1] == pytest.approx(150.0, rel=1e-15)          # silu(g) -> g for large g
    assert abs(h[2]) < 1e-18                                 # -> 0 for very negative g
    assert h[3] == pytest.approx(1.0 / (1.0 + np.exp(-1.0)))  # silu(1) = sigma(1)
    dg, du = ob.swiglu_bwd(np.ones(4), g, u)
    assert dg[0] == pytest.approx(0.5 * 2.0)                 # silu'(0) = 1/2
    assert du[0] == 0.0 and du[1] == pytest.approx(50.0)
    rng = np.random.default_rng(2)
    g, u, dh = rng.standard_normal((3, 6)), rng.standard_normal((3, 6)), rng.standard_normal((3, 6))
    dg, du = ob.swiglu_bwd(dh, g, u)
    np.testing.assert_allclose(dg, _fd(lambda t: ob.swiglu_fwd(t, u), g, dh), rtol=1e-6, atol=1e-9)
    np.testing.assert_allclose(du, _fd(lambda t: ob.swiglu_fwd(g, t), u, dh), rtol=1e-6, atol=1e-9)


# ------------------------------------------------------------------ RoPE
def test_rope_d2_rotation_by_hand():
    # d = 2: theta = pos (inv freq 1); row 3 of a sequence starting at row 1 has pos 2
    rs = np.array([-1, 1, 1, 1])
    x = np.zeros((4, 1, 2))
    x[:, 0, 0] = 1.0
    y = ob.rope_fwd(x, rs)
    np.testing.assert_allclose(y[0, 0], [1.0, 0.0])               # pad row untouched
    np.testing.assert_allclose(y[1, 0], [1.0, 0.0])               # pos 0: identity
    np.testing.assert_allclose(y[3, 0], [np.cos(2.0), np.sin(2.0)], rtol=1e-15)


def test_rope_orthogonal_relative_and_inverse():
    rng = np.random.default_rng(3)
    R, H, d = 40, 2, 16
    rs = np.array([0] * 25 + [25] * 15)
    x = rng.standard_normal((R, H, d))
    y = ob.rope_fwd(x, rs)
    a, b = y[..., :d // 2], y[..., d // 2:]
    xa, xb = x[..., :d // 2], x[..., d // 2:]
    np.testing.assert_allclose(a * a + b * b, xa * xa + xb * xb, rtol=1e-12)   # pairwise norms
    np.testing.assert_allclose(ob.rope_bwd(y, rs), x, atol=1e-12)               # R^T R = I
    # <rope(q, m), rope(k, n)> depends on m - n only: same query/key at offsets (3,1) and (13,11)
    q, k = rng.standard_normal(d), rng.standard_normal(d)
    z = np.zeros((R, 1, d))
    z[3, 0], z[1, 0], z[13, 0], z[11, 0] = q, k, q, k
    rz = ob.rope_fwd(z, np.zeros(R, dtype=int))
    assert np.dot(rz[3, 0], rz[1, 0]) == pytest.approx(np.dot(rz[13, 0], rz[11, 0]), rel=1e-12)
    dy = rng.standard_normal((R, H, d))
    np.testing.assert_allclose(ob.rope_bwd(dy, rs), _fd(lambda t: ob.rope_fwd(t, rs), x, dy), rtol=1e-6, atol=1e-8)


# ------------------------------------------------------------------ attention
def _rs(lens, pad_after=0):
    rs = []
    r = 0
    for L in lens:
        rs += [r] * L
        r += L
        rs += [-1] * pad_after
        r += pad_after
    return np.array(rs)


def test_attention_closed_forms():
    rng = np.random.default_rng(4)
    rs = _rs([1, 5, 3], pad_after=2)
    R, H, d = len(rs), 2, 8
    v = rng.standard_normal((R, H, d))
    # all scores equal (q = 0): o_q = mean of v over the causal prefix of its sequence
    q = np.zeros((R, H, d))
    k = rng.standard_normal((R, H, d))
    o, lse = ob.attention_fwd(q, k, v, rs, 0.5)
    for a, L in ob._sequences(rs):
        for i in range(L):
            np.testing.assert_allclose(o[a + i], v[a:a + i + 1].mean(axis=0), rtol=1e-13, atol=1e-15)
            np.testing.assert_allclose(lse[a + i], np.log(i + 1), rtol=1e-13)
    pads = rs < 0
    assert (o[pads] == 0).all() and np.isneginf(lse[pads]).all()
    # a one-token sequence returns its own value row
    np.testing.assert_allclose(o[0], v[0])


def test_attention_isolation_and_causality():
    rng = np.random.default_rng(5)
    lens = [7, 4, 9]
    rs = _rs(lens, pad_after=1)
    R, H, d = len(rs), 3, 8
    q, k, v = (rng.standard_normal((R, H, d)) for _ in range(3))
    o, _ = ob.attention_fwd(q, k, v, rs, 0.3)
    # each sequence alone (its own rows, row_start 0) == packed
    for a, L in ob._sequences(rs):
        oa, _ = ob.attention_fwd(q[a:a + L], k[a:a + L], v[a:a + L], np.zeros(L, dtype=int), 0.3)
        np.testing.assert_array_equal(oa, o[a:a + L])
    # causality: perturbing the last row's key/value changes no earlier output
    k2, v2 = k.copy(), v.copy()
    last = len(rs) - 2          # last valid row (the final row is a pad)
    k2[last] += 5.0
    v2[last] -= 3.0
    o2, _ = ob.attention_fwd(q, k2, v2, rs, 0.3)
    np.testing.assert_array_equal(o2[:last], o[:last])


def test_attention_bwd_finite_differences():
    rng = np.random.default_rng(6)
    rs = _rs([3, 4], pad_after=1)
    R, H, d = len(rs), 2, 4
    q, k, v, do = (rng.standard_normal((R, H, d)) for _ in range(4))
    dq, dk, dv = ob.attention_bwd(do, q, k, v, rs, 0.7)
    f = lambda qq, kk, vv: ob.attention_fwd(qq, kk, vv, rs, 0.7)[0]  # noqa: E731
    np.testing.assert_allclose(dq, _fd(lambda t: f(t, k, v), q, do), rtol=1e-6, atol=1e-8)
    np.testing.assert_allclose(dk, _fd(lambda t: f(q, t, v), k, do), rtol=1e-6, atol=1e-8)
    np.testing.assert_allclose(dv, _fd(lambda t: f(q, k, t), v, do), rtol=1e-6, atol=1e-8)
    pads = rs < 0
    assert (dq[pads] == 0).all() and (dk[pads] == 0).all() and (dv[pads] == 0).all()


# ------------------------------------------------------------------ hand-computed values
# These pin the constants the identities above cannot see (they hold for any
# frequency schedule, pairing, logit scale or eps).  Expected numbers are
# written out by hand from the stated definitions, not produced by the oracle.
COS = {3.0: -0.9899924966004454, 0.3: 0.955336489125606, 0.03: 0.9995500337489875, 0.003: 0.9999955000033750}
SIN = {3.0: 0.1411200080598672, 0.3: 0.29552020666133955, 0.03: 0.029995500202495664, 0.003: 0.0029999955000020251}


def test_rope_d8_position3_hand_values():
    """d = 8, base 1e4: inv_freq_i = base^(-2i/d) = 1, 1e-1, 1e-2, 1e-3 (i = 0..3); rotate-half pairing
    (i, i + d/2).  Row 3 of a sequence that starts at row 0 has position 3: angles 3, 0.3, 0.03, 0.003.
    x = [1,1,1,1, 0,0,0,0] -> [cos a_i | sin a_i];  x = [0,0,0,0, 1,1,1,1] -> [-sin a_i | cos a_i].
    An interleaved pairing ((2i, 2i+1)) or an exponent of -i/d instead of -2i/d fails this."""
    angles = (3.0, 0.3, 0.03, 0.003)
    x = np.zeros((4, 2, 8))
    x[3, 0, :4] = 1.0
    x[3, 1, 4:] = 1.0
    y = ob.rope_fwd(x, np.zeros(4, dtype=int), base=10000.0)
    np.testing.assert_allclose(y[3, 0], [COS[a] for a in angles] + [SIN[a] for a in angles], rtol=0, atol=1e-15)
    np.testing.assert_allclose(y[3, 1], [-SIN[a] for a in angles] + [COS[a] for a in angles], rtol=0, atol=1e-15)
    # position 0 (row 0) is the identity
    np.testing.assert_array_equal(ob.rope_fwd(x[[3, 3]], np.array([1, 1]))[1], x[3])


def test_attention_two_keys_hand_value():
    """Nonzero logits pin the scale: d = 2, scale 0.5, query row 1 q = [2, 0], keys k0 = [0, 0],
    k1 = [ln 3, 0] -> logits 0 and 0.5 * 2 * ln 3 = ln 3 -> softmax [1/4, 3/4]; v0 = [4, 0],
    v1 = [0, 8] -> o1 = [1, 6], lse1 = ln(1 + 3) = ln 4.  Row 0 sees only itself: o0 = v0,
    lse0 = 0.5 <q0, k0> = 0 for q0 = [0, 0]."""
    ln3 = 1.0986122886681098
    q = np.array([[[0.0, 0.0]], [[2.0, 0.0]]])
    k = np.array([[[0.0, 0.0]], [[ln3, 0.0]]])
    v = np.array([[[4.0, 0.0]], [[0.0, 8.0]]])
    o, lse = ob.attention_fwd(q, k, v, np.array([0, 0]), 0.5)
    np.testing.assert_allclose(o[1, 0], [1.0, 6.0], rtol=1e-15)
    assert lse[1, 0] == pytest.approx(1.3862943611198906, rel=1e-15)   # ln 4
    np.testing.assert_allclose(o[0, 0], [4.0, 0.0])
    assert lse[0, 0] == 0.0
    # backward of <dO, o> with dO = [1, 0] at row 1 only: dV = P^T dO -> dv0 = 1/4 [1,0], dv1 = 3/4 [1,0]
    do = np.zeros_like(q)
    do[1, 0] = [1.0, 0.0]
    dq, dk, dv = ob.attention_bwd(do, q, k, v, np.array([0, 0]), 0.5)
    np.testing.assert_allclose(dv[:, 0], [[0.25, 0.0], [0.75, 0.0]], rtol=1e-15)
    # dP = dO V^T = [4, 0]; dS = P (dP - <P, dP>) = [1/4 (4 - 1), 3/4 (0 - 1)] = [3/4, -3/4]
    # dq1 = scale * dS K = 0.5 * (-3/4) * [ln 3, 0];  dk0 = 0.5 * 3/4 * q1, dk1 = 0.5 * (-3/4) * q1
    np.testing.assert_allclose(dq[1, 0], [-0.375 * ln3, 0.0], rtol=1e-14)
    np.testing.assert_allclose(dk[:, 0], [[0.75, 0.0], [-0.75, 0.0]], rtol=1e-14)


def test_rmsnorm_eps_hand_values():
    """eps inside the root, added to the mean square: x = [3, 4] (mean square 12.5), eps = 3.5 ->
    rms = sqrt(16) = 4, y = x / 4 * w = [1.5, -1] for w = [2, -1].  Backward of y_0 (dy = [1, 0]):
    d/dx_0 (2 x_0 / s) = 2/s - x_0^2 / s^3 = 1/2 - 9/64,  d/dx_1 = -x_0 x_1 / s^3 = -12/64  (s = 4)."""
    x = np.array([[3.0, 4.0]])
    w = np.array([2.0, -1.0])
    np.testing.assert_allclose(ob.rmsnorm_fwd(x, w, 3.5), [[1.5, -1.0]], rtol=1e-15)
    np.testing.assert_allclose(ob.rmsnorm_bwd(np.array([[1.0, 0.0]]), x, w, 3.5), [[0.359375, -0.1875]], rtol=1e-15)
