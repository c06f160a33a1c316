"""Intra-stage orchestration (paper_2603_02885_b200/orchestrate.py, SURVEY
§8(f) NEXT-1; paper P:705-775, Alg. 1) on CPU.

* segmentation of a TP layer chain into subgraphs (compute clustered, each
  collective appended to the subgraph it depends on);
* Alg. 1 on hand-built DAGs: lowest depth first, longest latency among
  equals, timer = prefix sums of latencies; a Kahn-valid order on random DAGs;
* world 2 over gloo: two hTasks (disjoint task groups, each packed and run as
  its own multiplexed call) orchestrated through one TP column/row/column
  chain equal the single-process fp64 oracle of each hTask, and equal the
  un-orchestrated layer classes of tp.py bit for bit."""
import os
import random
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from paper_2603_02885_b200 import orchestrate as orc


def _noop(e):
    return None


class _DummyLayer:
    pass


def test_chain_segmentation():
    lays = [_DummyLayer(), _DummyLayer(), _DummyLayer()]
    ops = orc.linear_chain_ops(lays, ["col", "row", "col"], None, [0], lambda e: None, None, [1.0, 2.0, 3.0])
    sgs = orc.build_subgraphs(0, ops)
    names = [[o.name for o in sg.ops] for sg in sgs]
    assert names == [
        ["dispatch", "AG(x0)"],
        ["fwd0", "fwd1", "RS(y1)", "AG(x2)"],
        ["fwd2", "loss_grad", "bwd2", "AR(dA2)", "RS(dx2)", "AG(dy1)"],
        ["bwd1", "AR(dB1)", "bwd0", "AR(dA0)", "RS(dx0)"],
    ]
    assert [sg.depth for sg in sgs] == [0, 1, 2, 3]
    assert [sg.latency for sg in sgs] == [0.0, 3.0, 6.0, 3.0]   # fwd and bwd of a layer cost the same model
    assert [sg.deps for sg in sgs] == [[], [0], [1], [2]]


def test_segmentation_rules():
    C = lambda n, r, w, lat=1.0: orc.Op(n, "compute", r, w, _noop, lat)  # noqa: E731
    M = lambda n, r, w: orc.Op(n, "comm", r, w, _noop)  # noqa: E731
    # a comm result that no compute reads does not split; one that is read does
    ops = [C("a", (), ("x",)), M("ar", ("x",), ("x_sum",)), C("b", ("x",), ("y",)),
           M("rs", ("y",), ("z",)), C("c", ("z",), ("u",)), C("d", ("u",), ("v",))]
    sgs = orc.build_subgraphs(3, ops)
    assert [[o.name for o in sg.ops] for sg in sgs] == [["a", "ar", "b", "rs"], ["c", "d"]]
    assert all(sg.htask == 3 for sg in sgs)
    with pytest.raises(ValueError):
        orc.build_subgraphs(0, [orc.Op("bad", "other", (), (), _noop)])


def _chain(h, lats):
    return [orc.Subgraph(h, i, [orc.Op(f"h{h}s{i}", "compute", (), (), _noop, l)], [i - 1] if i else [], i)
            for i, l in enumerate(lats)]


def test_alg1_priority_then_latency():
    dags = [_chain(0, [1.0, 5.0, 2.0]), _chain(1, [3.0, 4.0]), _chain(2, [2.0, 7.0, 1.0])]
    sched = orc.subgraph_schedule(dags)
    order = [sg.key for sg, _ in sched]
    # depth 0: latencies 1, 3, 2 -> h1, h2, h0; depth 1: 5, 4, 7 -> h2, h0, h1; depth 2: 2, 1 -> h0, h2
    assert order == [(1, 0), (2, 0), (0, 0), (2, 1), (0, 1), (1, 1), (0, 2), (2, 2)]
    ts = [t for _, t in sched]
    lat = [sg.latency for sg, _ in sched]
    assert ts == list(np.concatenate([[0.0], np.cumsum(lat)[:-1]]))
    # equal depth and latency: hTask index breaks the tie (deterministic)
    sched = orc.subgraph_schedule([_chain(1, [1.0]), _chain(0, [1.0])])
    assert [sg.key for sg, _ in sched] == [(0, 0), (1, 0)]


def test_alg1_kahn_valid_on_random_dags():
    rng = random.Random(7)
    for _ in range(200):
        dags = []
        for h in range(rng.randint(1, 4)):
            n = rng.randint(1, 6)
            sgs = []
            for i in range(n):
                deps = sorted({j for j in range(i) if rng.random() < 0.4} | ({i - 1} if i and rng.random() < 0.5 else set()))
                depth = 0 if not deps else 1 + max(sgs[j].depth for j in deps)
                sgs.append(orc.Subgraph(h, i, [orc.Op("o", "compute", (), (), _noop, rng.choice([0.5, 1.0, 2.0]))],
                                        deps, depth))
            dags.append(sgs)
        sched = orc.subgraph_schedule(dags)
        pos = {sg.key: k for k, (sg, _) in enumerate(sched)}
        assert len(pos) == sum(len(d) for d in dags)
        for d in dags:
            for sg in d:
                assert all(pos[(sg.htask, j)] < pos[sg.key] for j in sg.deps)


def test_alg1_cycle_detected():
    a = orc.Subgraph(0, 0, [], [1], 0)
    b = orc.Subgraph(0, 1, [], [0], 1)
    with pytest.raises(ValueError):
        orc.subgraph_schedule([[a, b]])


# ------------------------------------------------------------------ gloo, world 2
K0, N0 = 32, 48          # chain: K0 -> N0 (col) -> K0 (row) -> N0 (col)
HTASKS = [
    {"seg": [64, 128], "ranks": [4, 8], "scales": [2.0, 1.0]},
    {"seg": [64, 64, 128], "ranks": [2, 16, 8], "scales": [0.5, 1.0, 2.0]},
]


CHAINS = {"crc": ["col", "row", "col"],   # K0 -> N0 -> K0 -> N0
          "rcr": ["row", "col", "row"]}   # K0 -> K0 -> N0 -> K0 (Megatron's o / up / down pairing)


def _htask_problem(h, chain="crc"):
    cfg = HTASKS[h]
    rng = np.random.default_rng(1000 + h)
    R = sum(cfg["seg"])
    seg_off = np.concatenate([[0], np.cumsum(cfg["seg"])]).astype(np.int32)
    X = rng.standard_normal((R, K0))
    shapes = [(N0, K0), (K0, N0), (N0, K0)] if chain == "crc" else [(K0, K0), (N0, K0), (K0, N0)]
    Ws = [rng.standard_normal(s) / np.sqrt(s[1]) for s in shapes]
    As = [[rng.standard_normal((r, s[1])) for r in cfg["ranks"]] for s in shapes]
    Bs = [[rng.standard_normal((s[0], r)) for r in cfg["ranks"]] for s in shapes]
    dY = rng.standard_normal((R, shapes[-1][0]))
    return seg_off, X, Ws, As, Bs, dY


def _worker(rank, world, port, q, chain="crc"):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        from paper_2603_02885_b200 import tp
        from test_tp_gloo import OracleBackend
        T = torch.from_numpy
        kinds = CHAINS[chain]

        def make_layers(h):
            seg_off, X, Ws, As, Bs, dY = _htask_problem(h, chain)
            cfg = HTASKS[h]
            be = OracleBackend()
            lays = []
            for li, kind in enumerate(kinds):
                ads = [tp.ShardAdapter(T(As[li][t]), T(Bs[li][t]), cfg["ranks"][t], cfg["scales"][t])
                       for t in range(len(cfg["ranks"]))]
                shard = tp.shard_column if kind == "col" else tp.shard_row
                Wp, ap = shard(T(Ws[li]), ads, world, rank, tp.ShardAdapter)
                lays.append((tp.ColumnParallelMuxLinear if kind == "col" else tp.RowParallelMuxLinear)(be, Wp, ap, 16))
            R = X.shape[0]
            rows = R // world
            if chain == "crc":     # row block of X in; loss gradient of the column output: N shard
                nl = dY.shape[1] // world
                x_rows = T(X[rank * rows:(rank + 1) * rows]).contiguous()
                dy = T(dY[:, rank * nl:(rank + 1) * nl]).contiguous()
            else:                  # column shard of X in (all rows); row-parallel output: row block
                kl = X.shape[1] // world
                x_rows = T(X[:, rank * kl:(rank + 1) * kl]).contiguous()
                dy = T(dY[rank * rows:(rank + 1) * rows]).contiguous()
            return T(seg_off), list(range(len(cfg["ranks"]))), lays, x_rows, dy

        # orchestrated: both hTasks interleaved by Alg. 1
        envs, dags, keep = [], [], []
        for h in range(len(HTASKS)):
            so, st, lays, x_rows, dy = make_layers(h)
            ops = orc.linear_chain_ops(lays, kinds, so, st, lambda e, x=x_rows: x, dy,
                                       [float(h + 1)] * 3)
            dags.append(orc.build_subgraphs(h, ops))
            envs.append({})
            keep.append(lays)
        sched = orc.subgraph_schedule(dags)
        orc.run_schedule(sched, envs)
        got = [(envs[h]["Y2"].numpy(), envs[h]["dX0"].numpy(),
                [[g.numpy() for g in envs[h][f"dA{i}"]] for i in range(3)],
                [[g.numpy() for g in envs[h][f"dB{i}"]] for i in range(3)]) for h in range(len(HTASKS))]
        # sequential layer classes of tp.py on the same shards
        seq = []
        for h in range(len(HTASKS)):
            so, st, lays, x_rows, dy = make_layers(h)
            y = x_rows
            for lay in lays:
                y = lay.forward(so, st, y)
            g = dy
            dA, dB = [None] * 3, [None] * 3
            for i in reversed(range(3)):
                g, dA[i], dB[i] = lays[i].backward(so, st, g)
            seq.append((y.numpy(), g.numpy(), [[x.numpy() for x in a] for a in dA], [[x.numpy() for x in b] for b in dB]))
        q.put((rank, None, [(sg.htask, sg.index) for sg, _ in sched], got, seq))
    finally:
        dist.destroy_process_group()


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def test_two_htasks_orchestrated_tp_world2():
    from oracle import linear as olin
    world = 2
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, q)) for r in range(world)]
    for p in procs:
        p.start()
    res = sorted([q.get(timeout=240) for _ in range(world)], key=lambda x: x[0])
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    order = res[0][2]
    # interleaved: hTask 1 (modeled latency 2 per layer) leads each depth level with compute;
    # the dispatch subgraphs (no modeled latency) tie and go by hTask index
    assert order == [(0, 0), (1, 0), (1, 1), (0, 1), (1, 2), (0, 2), (1, 3), (0, 3)]
    for h in range(len(HTASKS)):
        cfg = HTASKS[h]
        seg_off, X, Ws, As, Bs, dY = _htask_problem(h)
        st = list(range(len(cfg["ranks"])))
        args = lambda li: (As[li], Bs[li], cfg["ranks"], cfg["scales"])  # noqa: E731
        H0, _ = olin.linear_fwd(seg_off, st, *args(0), X, Ws[0], 16)
        H1, _ = olin.linear_fwd(seg_off, st, *args(1), H0, Ws[1], 16)
        Y2, _ = olin.linear_fwd(seg_off, st, *args(2), H1, Ws[2], 16)
        dH1, _, g2 = olin.linear_bwd(seg_off, st, *args(2), dY, H1, Ws[2], 16)
        dH0, _, g1 = olin.linear_bwd(seg_off, st, *args(1), dH1, H0, Ws[1], 16)
        dX, _, g0 = olin.linear_bwd(seg_off, st, *args(0), dH0, X, Ws[0], 16)
        y = np.concatenate([r[3][h][0] for r in res], axis=1)          # column output: N-sharded
        dx = np.concatenate([r[3][h][1] for r in res], axis=0)         # row blocks
        np.testing.assert_allclose(y, Y2, rtol=1e-10, atol=1e-10)
        np.testing.assert_allclose(dx, dX, rtol=1e-10, atol=1e-10)
        for t in range(len(st)):
            # layer 0 / 2 column: dA all-reduced, dB N-sharded; layer 1 row: dA K-sharded, dB all-reduced
            for li, g in ((0, g0), (2, g2)):
                np.testing.assert_allclose(res[0][3][h][2][li][t], g[t][0], rtol=1e-10, atol=1e-10)
                np.testing.assert_allclose(np.concatenate([r[3][h][3][li][t] for r in res]), g[t][1],
                                           rtol=1e-10, atol=1e-10)
            np.testing.assert_allclose(np.concatenate([r[3][h][2][1][t] for r in res], axis=1), g1[t][0],
                                       rtol=1e-10, atol=1e-10)
            np.testing.assert_allclose(res[0][3][h][3][1][t], g1[t][1], rtol=1e-10, atol=1e-10)
        # orchestrated == sequential tp.py layer classes, bit for bit
        for r in res:
            got, seq = r[3][h], r[4][h]
            assert np.array_equal(got[0], seq[0]) and np.array_equal(got[1], seq[1])
            for i in range(3):
                for t in range(len(st)):
                    assert np.array_equal(got[2][i][t], seq[2][i][t]) and np.array_equal(got[3][i][t], seq[3][i][t])


def test_two_htasks_orchestrated_tp_world2_row_col_row():
    """The bench's config-2 chain pairing [row, col, row] (every collective is K0 wide: the row-parallel
    L0 takes the column shard of X, the row-parallel L2 takes L1's column-sharded output with no
    collective): orchestrated == the sequential tp.py layer classes bit for bit, and == the fp64
    single-device oracle chain."""
    from oracle import linear as olin
    world = 2
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, q, "rcr")) for r in range(world)]
    for p in procs:
        p.start()
    res = sorted([q.get(timeout=240) for _ in range(world)], key=lambda x: x[0])
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    for h in range(len(HTASKS)):
        cfg = HTASKS[h]
        seg_off, X, Ws, As, Bs, dY = _htask_problem(h, "rcr")
        st = list(range(len(cfg["ranks"])))
        args = lambda li: (As[li], Bs[li], cfg["ranks"], cfg["scales"])  # noqa: E731
        H0, _ = olin.linear_fwd(seg_off, st, *args(0), X, Ws[0], 16)
        H1, _ = olin.linear_fwd(seg_off, st, *args(1), H0, Ws[1], 16)
        Y2, _ = olin.linear_fwd(seg_off, st, *args(2), H1, Ws[2], 16)
        dH1, _, g2 = olin.linear_bwd(seg_off, st, *args(2), dY, H1, Ws[2], 16)
        dH0, _, g1 = olin.linear_bwd(seg_off, st, *args(1), dH1, H0, Ws[1], 16)
        dX, _, g0 = olin.linear_bwd(seg_off, st, *args(0), dH0, X, Ws[0], 16)
        y = np.concatenate([r[3][h][0] for r in res], axis=0)          # row-parallel output: row blocks
        dx = np.concatenate([r[3][h][1] for r in res], axis=1)         # column shards of dX
        np.testing.assert_allclose(y, Y2, rtol=1e-10, atol=1e-10)
        np.testing.assert_allclose(dx, dX, rtol=1e-10, atol=1e-10)
        for t in range(len(st)):
            # layers 0 / 2 row: dA K-sharded, dB all-reduced; layer 1 column: dA all-reduced, dB N-sharded
            for li, g in ((0, g0), (2, g2)):
                np.testing.assert_allclose(np.concatenate([r[3][h][2][li][t] for r in res], axis=1), g[t][0],
                                           rtol=1e-10, atol=1e-10)
                np.testing.assert_allclose(res[0][3][h][3][li][t], g[t][1], rtol=1e-10, atol=1e-10)
            np.testing.assert_allclose(res[0][3][h][2][1][t], g1[t][0], rtol=1e-10, atol=1e-10)
            np.testing.assert_allclose(np.concatenate([r[3][h][3][1][t] for r in res]), g1[t][1],
                                       rtol=1e-10, atol=1e-10)
        for r in res:
            got, seq = r[3][h], r[4][h]
            assert np.array_equal(got[0], seq[0]) and np.array_equal(got[1], seq[1])
            for i in range(3):
                for t in range(len(st)):
                    assert np.array_equal(got[2][i][t], seq[2][i][t]) and np.array_equal(got[3][i][t], seq[3][i][t])
