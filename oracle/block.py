"""fp64 ORACLE for the non-BaseOp parts of the decoder block (SURVEY §8(f)
NEXT-3): chunked causal attention with KV reuse, RoPE, RMSNorm, SwiGLU.

ORACLE — test infrastructure only (see oracle/__init__.py).  Plain numpy,
fp64, written from the definitions; inputs are the exact bf16 values the GPU
receives, widened to fp64 by the caller.

Row layout (§3.5 "Chunk-based alignment"): the packed rows of an
hTask hold each sequence on consecutive rows (a pack is split into
consecutive chunks; a sequence never leaves its pack).  `row_start[r]` is the
first packed row of row r's sequence, or -1 for a pad row.  Causal attention
inside a sequence is what the paper's chunk dependency ("KV cache reuse in
causal attention", Fig. alignment caption) computes: the queries
of chunk j attend to the keys of the earlier chunks of the same pack, and the
attention mask keeps them inside their own sequence (packing without masks
"wastes attention computation across sequences").  So, for a
query row q with s = row_start[q]:
    o_q = sum_{k=s..q} softmax_k(scale * <q_q, k_k>) v_k     (per head)
Position of row r inside its sequence: pos_r = r - row_start[r].

The decoder-block ops follow LLaMA (the backbones of the paper's workloads,
P:940-946): RMSNorm, rotary position embedding (rotate-half form, base
10000), SwiGLU MLP.  The backbone is frozen, so RMSNorm's weight gets
no gradient.
"""
from __future__ import annotations

import numpy as np


# ------------------------------------------------------------------ row map
def row_seq_start(seq_row, seq_len, max_rows):
    """row_start[r] from the pack outputs: rows [seq_row[s], seq_row[s]+len_s)
    belong to sequence s; every other row is a pad (-1)."""
    out = np.full(max_rows, -1, dtype=np.int64)
    for s in range(len(seq_len)):
        a = int(seq_row[s])
        out[a:a + int(seq_len[s])] = a
    return out


# ------------------------------------------------------------------ RMSNorm
def rmsnorm_fwd(x, w, eps):
    """y = x / sqrt(mean_j x_j^2 + eps) * w   (per row)."""
    x = np.asarray(x, np.float64)
    rstd = 1.0 / np.sqrt(np.mean(x * x, axis=-1, keepdims=True) + eps)
    return x * rstd * np.asarray(w, np.float64)


def rmsnorm_bwd(dy, x, w, eps):
    """dx of y = rmsnorm(x) * w for upstream dy (w frozen: no dw).
    With r = rstd, xh = x r, g = dy * w:  dx = r * (g - xh * mean_j(g_j xh_j))."""
    x = np.asarray(x, np.float64)
    g = np.asarray(dy, np.float64) * np.asarray(w, np.float64)
    r = 1.0 / np.sqrt(np.mean(x * x, axis=-1, keepdims=True) + eps)
    xh = x * r
    return r * (g - xh * np.mean(g * xh, axis=-1, keepdims=True))


# ------------------------------------------------------------------ SwiGLU
def _sigmoid(z):
    return 1.0 / (1.0 + np.exp(-z))


def swiglu_fwd(g, u):
    """h = silu(g) * u, silu(g) = g * sigmoid(g)."""
    g = np.asarray(g, np.float64)
    return g * _sigmoid(g) * np.asarray(u, np.float64)


def swiglu_bwd(dh, g, u):
    """dg = dh * u * sigma(g) (1 + g (1 - sigma(g))),  du = dh * silu(g)."""
    g = np.asarray(g, np.float64)
    u = np.asarray(u, np.float64)
    dh = np.asarray(dh, np.float64)
    sg = _sigmoid(g)
    return dh * u * sg * (1.0 + g * (1.0 - sg)), dh * g * sg


# ------------------------------------------------------------------ RoPE
def rope_angles(pos, d, base=10000.0):
    """theta[r, i] = pos_r * base^(-2i/d), i < d/2."""
    inv = base ** (-np.arange(0, d // 2, dtype=np.float64) * 2.0 / d)
    return np.asarray(pos, np.float64)[:, None] * inv[None, :]


def rope_fwd(x, row_start, base=10000.0):
    """x [R, H, d]: pairs (i, i + d/2) rotated by theta_i at the row's
    position in its sequence:  x'_i = x_i cos - x_{i+d/2} sin,
    x'_{i+d/2} = x_{i+d/2} cos + x_i sin.  Pad rows pass through."""
    x = np.asarray(x, np.float64)
    R, H, d = x.shape
    rs = np.asarray(row_start)
    pos = np.where(rs >= 0, np.arange(R) - rs, 0)
    th = rope_angles(pos, d, base)[:, None, :]
    c, s = np.cos(th), np.sin(th)
    a, b = x[..., :d // 2], x[..., d // 2:]
    return np.concatenate([a * c - b * s, b * c + a * s], axis=-1)


def rope_bwd(dy, row_start, base=10000.0):
    """The rotation is orthogonal: dx = R(theta)^T dy = rotation by -theta."""
    dy = np.asarray(dy, np.float64)
    R, H, d = dy.shape
    rs = np.asarray(row_start)
    pos = np.where(rs >= 0, np.arange(R) - rs, 0)
    th = rope_angles(pos, d, base)[:, None, :]
    c, s = np.cos(th), np.sin(th)
    a, b = dy[..., :d // 2], dy[..., d // 2:]
    return np.concatenate([a * c + b * s, b * c - a * s], axis=-1)


# ------------------------------------------------------------------ attention
def _sequences(row_start):
    """(start, length) of every sequence, in row order."""
    rs = np.asarray(row_start)
    out = []
    r = 0
    R = len(rs)
    while r < R:
        if rs[r] < 0:
            r += 1
            continue
        a = r
        while r < R and rs[r] == a:
            r += 1
        out.append((a, r - a))
    return out


def attention_fwd(q, k, v, row_start, scale):
    """q, k, v [R, H, d] -> (o [R, H, d], lse [R, H]); causal inside each
    sequence; pad rows: o = 0, lse = -inf."""
    q, k, v = (np.asarray(t, np.float64) for t in (q, k, v))
    R, H, d = q.shape
    o = np.zeros((R, H, d))
    lse = np.full((R, H), -np.inf)
    for a, L in _sequences(row_start):
        mask = np.tril(np.ones((L, L), dtype=bool))
        for h in range(H):
            S = scale * (q[a:a + L, h] @ k[a:a + L, h].T)
            S = np.where(mask, S, -np.inf)
            m = S.max(axis=1, keepdims=True)
            E = np.exp(S - m)
            Z = E.sum(axis=1, keepdims=True)
            o[a:a + L, h] = (E / Z) @ v[a:a + L, h]
            lse[a:a + L, h] = (m + np.log(Z))[:, 0]
    return o, lse


def attention_bwd(do, q, k, v, row_start, scale):
    """Gradients of sum(do * o) w.r.t. q, k, v (chain rule through softmax):
    P = softmax(S), dV = P^T dO, dP = dO V^T, dS = P * (dP - rowsum(dP * P)),
    dQ = scale dS K, dK = scale dS^T Q.  Pad rows get 0."""
    do, q, k, v = (np.asarray(t, np.float64) for t in (do, q, k, v))
    R, H, d = q.shape
    dq, dk, dv = np.zeros_like(q), np.zeros_like(k), np.zeros_like(v)
    for a, L in _sequences(row_start):
        mask = np.tril(np.ones((L, L), dtype=bool))
        sl = slice(a, a + L)
        for h in range(H):
            S = np.where(mask, scale * (q[sl, h] @ k[sl, h].T), -np.inf)
            P = np.exp(S - S.max(axis=1, keepdims=True))
            P /= P.sum(axis=1, keepdims=True)
            dv[sl, h] = P.T @ do[sl, h]
            dP = do[sl, h] @ v[sl, h].T
            dS = P * (dP - np.sum(dP * P, axis=1, keepdims=True))
            dq[sl, h] = scale * dS @ k[sl, h]
            dk[sl, h] = scale * dS.T @ q[sl, h]
    return dq, dk, dv
