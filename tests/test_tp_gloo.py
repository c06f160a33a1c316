"""Tensor-parallel orchestration (paper_2603_02885_b200/tp.py) on
CPU: world_size 2, 4 and 8 over gloo, with the fp64 oracle injected as each rank's
local linear.  The TP result (gathered) must equal the single-process oracle
on the full problem: a column-parallel layer followed by a row-parallel layer
(e.g. up -> down), forward and backward, including dA_t / dB_t."""
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from oracle import linear as olin
from tp_oracle_backend import OracleBackend

K, N, R = 32, 48, 256          # up: K -> N (column), down: N -> K (row)
SEG = [64, 128, 64]
RANKS = [4, 8, 2]
SCALES = [2.0, 1.0, 0.5]


def _problem():
    rng = np.random.default_rng(123)
    seg_off = np.concatenate([[0], np.cumsum(SEG)]).astype(np.int32)
    X = rng.standard_normal((R, K))
    W1 = rng.standard_normal((N, K)) / np.sqrt(K)
    W2 = rng.standard_normal((K, N)) / np.sqrt(N)
    A1 = [rng.standard_normal((r, K)) for r in RANKS]
    B1 = [rng.standard_normal((N, r)) for r in RANKS]
    A2 = [rng.standard_normal((r, N)) for r in RANKS]
    B2 = [rng.standard_normal((K, r)) for r in RANKS]
    dY2 = rng.standard_normal((R, K))
    return seg_off, X, W1, W2, A1, B1, A2, B2, dY2


def _worker(rank, world, port, q, shared_shrink=False):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        from paper_2603_02885_b200 import tp
        seg_off, X, W1, W2, A1, B1, A2, B2, dY2 = _problem()
        T = torch.from_numpy
        mk = lambda A, B, r, s: tp.ShardAdapter(A, B, r, s)  # noqa: E731
        ads1 = [tp.ShardAdapter(T(A1[t]), T(B1[t]), RANKS[t], SCALES[t]) for t in range(3)]
        ads2 = [tp.ShardAdapter(T(A2[t]), T(B2[t]), RANKS[t], SCALES[t]) for t in range(3)]
        W1p, a1p = tp.shard_column(T(W1), ads1, world, rank, mk)
        W2p, a2p = tp.shard_row(T(W2), ads2, world, rank, mk)
        be = OracleBackend()
        up = tp.ColumnParallelMuxLinear(be, W1p, a1p, 16, shared_shrink=shared_shrink)
        down = tp.RowParallelMuxLinear(be, W2p, a2p, 16)
        so = T(seg_off)
        st = [0, 1, 2]
        rows = R // world
        x_rows = T(X[rank * rows:(rank + 1) * rows]).contiguous()
        h = up.forward(so, st, x_rows)                 # [R, N/p]
        y_rows = down.forward(so, st, h)               # [R/p, K]
        dy_rows = T(dY2[rank * rows:(rank + 1) * rows]).contiguous()
        dh, dA2, dB2 = down.backward(so, st, dy_rows)  # [R, N/p]
        dx_rows, dA1, dB1 = up.backward(so, st, dh)    # [R/p, K]
        q.put((rank, y_rows.numpy(), dx_rows.numpy(), [g.numpy() for g in dA1], [g.numpy() for g in dB1],
               [g.numpy() for g in dA2], [g.numpy() for g in dB2]))
    finally:
        dist.destroy_process_group()


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


@pytest.mark.parametrize("world,shared_shrink", [(2, False), (4, False), (8, False), (2, True), (4, True)])
def test_tp_column_row_matches_single_process(world, shared_shrink):
    """shared_shrink: each rank shrinks only its own rows (NaN elsewhere) and the Hs rows are
    all-gathered before the forward with the shrink given."""
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, q, shared_shrink)) for r in range(world)]
    for p in procs:
        p.start()
    res = sorted([q.get(timeout=240) for _ in range(world)], key=lambda x: x[0])
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    # single-process reference: up then down, full problem
    seg_off, X, W1, W2, A1, B1, A2, B2, dY2 = _problem()
    st = [0, 1, 2]
    H1, _ = olin.linear_fwd(seg_off, st, A1, B1, RANKS, SCALES, X, W1, 16)
    Y2, _ = olin.linear_fwd(seg_off, st, A2, B2, RANKS, SCALES, H1, W2, 16)
    dH1, _, g2 = olin.linear_bwd(seg_off, st, A2, B2, RANKS, SCALES, dY2, H1, W2, 16)
    dX, _, g1 = olin.linear_bwd(seg_off, st, A1, B1, RANKS, SCALES, dH1, X, W1, 16)
    y = np.concatenate([r[1] for r in res])
    dx = np.concatenate([r[2] for r in res])
    np.testing.assert_allclose(y, Y2, rtol=1e-10, atol=1e-10)
    np.testing.assert_allclose(dx, dX, rtol=1e-10, atol=1e-10)
    n, k = N // world, N // world
    for t in range(3):
        # column layer: dA all-reduced (full), dB sharded on N
        np.testing.assert_allclose(res[0][3][t], g1[t][0], rtol=1e-10, atol=1e-10)
        np.testing.assert_allclose(np.concatenate([r[4][t] for r in res]), g1[t][1], rtol=1e-10, atol=1e-10)
        # row layer: dA sharded on K (= N of the up layer), dB all-reduced (full)
        np.testing.assert_allclose(np.concatenate([r[5][t] for r in res], axis=1), g2[t][0], rtol=1e-10,
                                   atol=1e-10)
        np.testing.assert_allclose(res[1][6][t], g2[t][1], rtol=1e-10, atol=1e-10)
    del n, k
