"""Tensor-parallel decoder block (paper_2603_02885_b200/tp_block.py; SURVEY §8(d)
configs 4/5, §8(e)) on CPU: world size 2, 4 and 8 over gloo, with fp64 oracle
ops injected as each rank's local kernels (linears: oracle/linear.c; RMSNorm,
RoPE, attention, SwiGLU: oracle/block.py).  The TP block — column-parallel
q/k/v/gate/up, head-sharded attention (GQA groups kept on one rank),
row-parallel o/down, sequence-parallel AG/RS around them — must equal the
single-process fp64 composition of the whole block on the full problem:
output rows, input-gradient rows, and every adapter gradient of all seven
linears (column layers: dA all-reduced, dB sharded on N; row layers: dA
sharded on K, dB all-reduced)."""
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from oracle import block as ob
from oracle import linear as olin
from tp_oracle_backend import OracleOps

LIN = ("q", "k", "v", "o", "gate", "up", "down")
SEG = [16, 24, 24]            # rows per task segment (R = 64)
SEQS = [[10, 6], [20, 4], [7, 5, 8]]   # sequences inside each segment; the rest are pad rows
RANKS = [4, 8, 2]
SCALES = [2.0, 1.0, 0.5]
EPS = 1e-5


def _shape(world):
    kv = max(2, world)
    return dict(hidden=32, ffn=48, heads=8, kv_heads=kv, head_dim=4)


def _row_start():
    rs = []
    for seg, seqs in zip(SEG, SEQS):
        r0 = len(rs)
        for L in seqs:
            rs += [len(rs)] * L
        rs += [-1] * (seg - (len(rs) - r0))
    return np.array(rs, dtype=np.int64)


def _problem(sh):
    rng = np.random.default_rng(7)
    H, F, d = sh["hidden"], sh["ffn"], sh["head_dim"]
    dims = {"q": (H, sh["heads"] * d), "k": (H, sh["kv_heads"] * d), "v": (H, sh["kv_heads"] * d),
            "o": (sh["heads"] * d, H), "gate": (H, F), "up": (H, F), "down": (F, H)}
    W = {n: rng.standard_normal((N, K)) / np.sqrt(K) for n, (K, N) in dims.items()}
    W["norm1"] = 1 + 0.1 * rng.standard_normal(H)
    W["norm2"] = 1 + 0.1 * rng.standard_normal(H)
    A = {n: [rng.standard_normal((r, dims[n][0])) / np.sqrt(dims[n][0]) for r in RANKS] for n in LIN}
    B = {n: [rng.standard_normal((dims[n][1], r)) / np.sqrt(r) for r in RANKS] for n in LIN}
    rs = _row_start()
    R = len(rs)
    X = rng.standard_normal((R, H))
    X[rs < 0] = 0.0
    dY = rng.standard_normal((R, H))
    seg_off = np.concatenate([[0], np.cumsum(SEG)]).astype(np.int32)
    return W, A, B, X, dY, seg_off, rs


def _reference(sh, W, A, B, X, dY, seg_off, rs):
    """Single-process fp64 composition of the block (same op order as block.py)."""
    H, Hkv, d = sh["heads"], sh["kv_heads"], sh["head_dim"]
    R, G, st = X.shape[0], sh["heads"] // sh["kv_heads"], [0, 1, 2]
    lin = lambda n, x: olin.linear_fwd(seg_off, st, A[n], B[n], RANKS, SCALES, x, W[n], 16)[0]  # noqa: E731
    linb = lambda n, dy, x: olin.linear_bwd(seg_off, st, A[n], B[n], RANKS, SCALES, dy, x, W[n], 16)  # noqa
    h1 = ob.rmsnorm_fwd(X, W["norm1"], EPS)
    q, k, v = lin("q", h1), lin("k", h1), lin("v", h1)
    qr, kr = ob.rope_fwd(q.reshape(R, H, d), rs), ob.rope_fwd(k.reshape(R, Hkv, d), rs)
    Kf, Vf = np.repeat(kr, G, axis=1), np.repeat(v.reshape(R, Hkv, d), G, axis=1)
    a = ob.attention_fwd(qr, Kf, Vf, rs, d ** -0.5)[0].reshape(R, H * d)
    x2 = X + lin("o", a)
    h2 = ob.rmsnorm_fwd(x2, W["norm2"], EPS)
    g, u = lin("gate", h2), lin("up", h2)
    m = ob.swiglu_fwd(g, u)
    y = x2 + lin("down", m)
    grads = {}
    dm, _, grads["down"] = linb("down", dY, m)
    dg, du = ob.swiglu_bwd(dm, g, u)
    dh2g, _, grads["gate"] = linb("gate", dg, h2)
    dh2u, _, grads["up"] = linb("up", du, h2)
    dx2 = ob.rmsnorm_bwd(dh2g + dh2u, x2, W["norm2"], EPS) + dY
    da, _, grads["o"] = linb("o", dx2, a)
    dq, dk, dv = ob.attention_bwd(da.reshape(R, H, d), qr, Kf, Vf, rs, d ** -0.5)
    dk = ob.rope_bwd(dk.reshape(R, Hkv, G, d).sum(axis=2), rs).reshape(R, Hkv * d)
    dv = dv.reshape(R, Hkv, G, d).sum(axis=2).reshape(R, Hkv * d)
    dq = ob.rope_bwd(dq, rs).reshape(R, H * d)
    dh1q, _, grads["q"] = linb("q", dq, h1)
    dh1k, _, grads["k"] = linb("k", dk, h1)
    dh1v, _, grads["v"] = linb("v", dv, h1)
    dx = ob.rmsnorm_bwd(dh1q + dh1k + dh1v, X, W["norm1"], EPS) + dx2
    return y, dx, grads


def _worker(rank, world, port, q, fused=False, shared_shrink=False):
    import sys
    sys.path.insert(0, os.path.dirname(os.path.abspath(__file__)))
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        from paper_2603_02885_b200 import tp, tp_block
        sh = _shape(world)
        W, A, B, X, dY, seg_off, rs = _problem(sh)
        T = torch.from_numpy
        full_w = {n: T(w) for n, w in W.items()}
        full_a = {n: [tp.ShardAdapter(T(A[n][t]), T(B[n][t]), RANKS[t], SCALES[t]) for t in range(3)] for n in LIN}
        mk = lambda A_, B_, r, s: tp.ShardAdapter(A_, B_, r, s)  # noqa: E731
        col_off = None
        if fused:   # q|k|v and gate|up as one column-sliced call each (include/mux.h "Fused projections")
            Wp, ap, col_off = tp_block.shard_block_fused(full_w, full_a, world, rank, mk)
        else:
            Wp, ap = tp_block.shard_block(full_w, full_a, world, rank, mk)
        shape = tp_block.TPBlockShape(eps=EPS, p=world, **sh)
        blk = tp_block.TPDecoderBlock(OracleOps(sh["head_dim"]), shape, Wp, ap, 16, col_off=col_off,
                                      shared_shrink=shared_shrink, shared_gs=shared_shrink)
        rows = X.shape[0] // world
        sl = slice(rank * rows, (rank + 1) * rows)
        y = blk.forward(T(X[sl]).contiguous(), T(seg_off), [0, 1, 2], T(rs))
        dx = blk.backward(T(dY[sl]).contiguous())
        g = {n: ([t.numpy() for t in dA], [t.numpy() for t in dB]) for n, (dA, dB) in blk.adapter_grads().items()}
        q.put((rank, y.numpy(), dx.numpy(), g))
    finally:
        dist.destroy_process_group()


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


@pytest.mark.parametrize("world,fused,shared_shrink", [(2, False, False), (4, False, False), (8, False, False),
                                                       (2, True, False), (4, True, True), (8, True, False),
                                                       (8, False, True)])
def test_tp_block_matches_single_process(world, fused, shared_shrink):
    """fused: q|k|v and gate|up as one column-sliced linear each; shared_shrink: column layers shrink
    their own rows and all-gather Hs, row layers likewise Gs in the backward (rows they do not own are
    NaN in the oracle backend's shrinks).
    Both must equal the unfused single-process composition."""
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, q, fused, shared_shrink)) for r in range(world)]
    for p in procs:
        p.start()
    res = sorted([q.get(timeout=300) for _ in range(world)], key=lambda x: x[0])
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    sh = _shape(world)
    W, A, B, X, dY, seg_off, rs = _problem(sh)
    y, dx, grads = _reference(sh, W, A, B, X, dY, seg_off, rs)
    np.testing.assert_allclose(np.concatenate([r[1] for r in res]), y, rtol=1e-10, atol=1e-10)
    np.testing.assert_allclose(np.concatenate([r[2] for r in res]), dx, rtol=1e-10, atol=1e-10)
    for n in LIN:
        col = n in ("q", "k", "v", "gate", "up")
        for t in range(3):
            dA_ref, dB_ref = grads[n][t]
            if col:   # dA all-reduced (every rank holds the full one), dB sharded on N
                for r in res:
                    np.testing.assert_allclose(r[3][n][0][t], dA_ref, rtol=1e-10, atol=1e-10)
                np.testing.assert_allclose(np.concatenate([r[3][n][1][t] for r in res]), dB_ref, rtol=1e-10,
                                           atol=1e-10)
            else:     # dA sharded on K, dB all-reduced
                np.testing.assert_allclose(np.concatenate([r[3][n][0][t] for r in res], axis=1), dA_ref,
                                           rtol=1e-10, atol=1e-10)
                for r in res:
                    np.testing.assert_allclose(r[3][n][1][t], dB_ref, rtol=1e-10, atol=1e-10)
