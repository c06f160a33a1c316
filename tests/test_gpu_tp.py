"""Tensor-parallel wrapper on the GPU (world size 1, NCCL): the column/row
chain through paper_2603_02885_b200.tp with the libmux backend must equal the
same layers called directly through the binding, bit for bit (with one rank
every collective is an identity)."""
import os

import pytest

pytestmark = pytest.mark.gpu

torch = pytest.importorskip("torch")
if not torch.cuda.is_available():
    pytest.skip("needs a CUDA device", allow_module_level=True)

import torch.distributed as dist  # noqa: E402

from paper_2603_02885_b200 import mux, orchestrate, tp  # noqa: E402


def _bits(t):
    return t.view(torch.int16) if t.dtype == torch.bfloat16 else t


@pytest.fixture(scope="module")
def pg():
    os.environ.setdefault("MASTER_ADDR", "127.0.0.1")
    os.environ.setdefault("MASTER_PORT", "29533")
    if not dist.is_initialized():
        dist.init_process_group("nccl", rank=0, world_size=1, device_id=torch.device("cuda", 0))
    yield
    dist.destroy_process_group()


@pytest.mark.parametrize("shared_shrink", [False, True])
def test_tp_world1_equals_direct(pg, shared_shrink):
    if True:
        g = torch.Generator(device="cuda").manual_seed(3)
        R, K, N = 512, 256, 384
        seg_off = torch.tensor([0, 192, 320, 512], dtype=torch.int32, device="cuda")
        st = [0, 1, 2]
        ranks = [16, 8, 32]

        def make(KK, NN):
            W = (torch.randn(NN, KK, device="cuda", generator=g) / KK ** 0.5).bfloat16()
            ads = []
            for r in ranks:
                B = mux.make_B_storage(NN, r)
                B.copy_(torch.randn(NN, r, device="cuda", generator=g).bfloat16())
                ads.append(mux.Adapter((torch.randn(r, KK, device="cuda", generator=g) / KK ** 0.5).bfloat16(),
                                       B, r, 2.0))
            return W, ads

        W1, a1 = make(K, N)   # column-parallel layer K -> N
        W2, a2 = make(N, K)   # row-parallel layer N -> K
        X = torch.randn(R, K, device="cuda", generator=g).bfloat16()
        dY = torch.randn(R, K, device="cuda", generator=g).bfloat16()
        mk = lambda A, B, r, s: mux.Adapter(A, B, r, s)  # noqa: E731
        be = tp.MuxBackend()
        W1p, a1p = tp.shard_column(W1, a1, 1, 0, mk)
        W2p, a2p = tp.shard_row(W2, a2, 1, 0, mk)
        up = tp.ColumnParallelMuxLinear(be, W1p, a1p, 32, shared_shrink=shared_shrink)
        down = tp.RowParallelMuxLinear(be, W2p, a2p, 32)
        h = up.forward(seg_off, st, X)
        y = down.forward(seg_off, st, h)
        dh, dA2, dB2 = down.backward(seg_off, st, dY)
        dx, dA1, dB1 = up.backward(seg_off, st, dh)
        torch.cuda.synchronize()
        got = [y.clone(), dx.clone()] + [t.clone() for t in dA1 + dB1 + dA2 + dB2]

        H, Hs1 = mux.linear_fwd(seg_off, st, a1, X, W1, 32)
        Y, Hs2 = mux.linear_fwd(seg_off, st, a2, H, W2, 32)
        dH = mux.linear_bwd(seg_off, st, a2, dY, H, W2, Hs2, 32)
        dX = mux.linear_bwd(seg_off, st, a1, dH, X, W1, Hs1, 32)
        torch.cuda.synchronize()
        ref = [Y, dX] + [a.dA for a in a1] + [a.dB for a in a1] + [a.dA for a in a2] + [a.dB for a in a2]
        for a_, b_ in zip(got, ref):
            assert torch.equal(_bits(a_), _bits(b_))


@pytest.mark.parametrize("chain", ["crc", "rcr"])
def test_orchestrated_htasks_world1_equals_direct(pg, chain):
    """Two hTasks through a column/row/column (crc) or row/column/row (rcr, the bench's config-2
    chain) layer chain, interleaved by Alg. 1 with asynchronous NCCL collectives (orchestrate.py,
    NEXT-1), equal each hTask run through the binding directly, bit for bit."""
    g = torch.Generator(device="cuda").manual_seed(11)
    K, N = 256, 512
    if chain == "crc":
        shapes, kinds = [(N, K), (K, N), (N, K)], ["col", "row", "col"]
    else:
        shapes, kinds = [(K, K), (N, K), (K, N)], ["row", "col", "row"]
    mk = lambda A, B, r, s: mux.Adapter(A, B, r, s)  # noqa: E731
    Ws = [(torch.randn(n, k, device="cuda", generator=g) / k ** 0.5).bfloat16() for n, k in shapes]
    cfgs = [([0, 256, 448], [16, 8]), ([0, 128, 192, 640], [4, 32, 16])]
    hts = []
    for so_l, ranks in cfgs:
        so = torch.tensor(so_l, dtype=torch.int32, device="cuda")
        ads_all = []
        for n, k in shapes:
            ads = []
            for r in ranks:
                B = mux.make_B_storage(n, r)
                B.copy_(torch.randn(n, r, device="cuda", generator=g).bfloat16())
                ads.append(mux.Adapter((torch.randn(r, k, device="cuda", generator=g) / k ** 0.5).bfloat16(),
                                       B, r, 2.0))
            ads_all.append(ads)
        R = so_l[-1]
        X = torch.randn(R, K, device="cuda", generator=g).bfloat16()
        dY = torch.randn(R, shapes[-1][0], device="cuda", generator=g).bfloat16()
        be = tp.MuxBackend()
        lays = []
        for li, kind in enumerate(kinds):
            shard = tp.shard_column if kind == "col" else tp.shard_row
            Wp, ap = shard(Ws[li], ads_all[li], 1, 0, mk)
            lays.append((tp.ColumnParallelMuxLinear if kind == "col" else tp.RowParallelMuxLinear)(be, Wp, ap, 32))
        hts.append((so, list(range(len(ranks))), ads_all, X, dY, lays))
    dags, envs = [], []
    for i, (so, st, ads_all, X, dY, lays) in enumerate(hts):
        ops = orchestrate.linear_chain_ops(lays, kinds, so, st, lambda e, X=X: X, dY, [1.0 + i] * 3)
        dags.append(orchestrate.build_subgraphs(i, ops))
        envs.append({})
    orchestrate.run_schedule(orchestrate.subgraph_schedule(dags), envs)
    torch.cuda.synchronize()
    got = [(envs[i]["Y2"].clone(), envs[i]["dX0"].clone(),
            [a.dA.clone() for li in range(3) for a in hts[i][5][li].ads],
            [a.dB.clone() for li in range(3) for a in hts[i][5][li].ads]) for i in range(len(hts))]
    for i, (so, st, ads_all, X, dY, lays) in enumerate(hts):
        x, Hs = X, []
        xs = []
        for li in range(3):
            xs.append(x)
            x, hs = mux.linear_fwd(so, st, ads_all[li], x, Ws[li], 32)
            Hs.append(hs)
        y = x.clone()
        d = dY
        for li in reversed(range(3)):
            d = mux.linear_bwd(so, st, ads_all[li], d, xs[li], Ws[li], Hs[li], 32)
        torch.cuda.synchronize()
        assert torch.equal(_bits(got[i][0]), _bits(y))
        assert torch.equal(_bits(got[i][1]), _bits(d))
        ref_dA = [a.dA for li in range(3) for a in ads_all[li]]
        ref_dB = [a.dB for li in range(3) for a in ads_all[li]]
        for a_, b_ in zip(got[i][2] + got[i][3], ref_dA + ref_dB):
            assert torch.equal(a_, b_)


def test_tp_fused_rs_world1_equals_direct(pg):
    """The tp.py layers with the reduce-scatter fused into the GEMMs (peer-store path through torch
    symmetric memory; at world 1 the 'peer' is this GPU) == direct binding calls, bit for bit."""
    g = torch.Generator(device="cuda").manual_seed(21)
    R, K, N = 512, 256, 384
    seg_off = torch.tensor([0, 192, 320, 512], dtype=torch.int32, device="cuda")
    st = [0, 1, 2]
    ranks = [16, 8, 32]

    def make(KK, NN):
        W = (torch.randn(NN, KK, device="cuda", generator=g) / KK ** 0.5).bfloat16()
        ads = []
        for r in ranks:
            B = mux.make_B_storage(NN, r)
            B.copy_(torch.randn(NN, r, device="cuda", generator=g).bfloat16())
            ads.append(mux.Adapter((torch.randn(r, KK, device="cuda", generator=g) / KK ** 0.5).bfloat16(),
                                   B, r, 2.0))
        return W, ads

    W1, a1 = make(K, N)
    W2, a2 = make(N, K)
    X = torch.randn(R, K, device="cuda", generator=g).bfloat16()
    dY = torch.randn(R, K, device="cuda", generator=g).bfloat16()
    mk = lambda A, B, r, s: mux.Adapter(A, B, r, s)  # noqa: E731
    be = tp.MuxBackend()
    W1p, a1p = tp.shard_column(W1, a1, 1, 0, mk)
    W2p, a2p = tp.shard_row(W2, a2, 1, 0, mk)
    up = tp.ColumnParallelMuxLinear(be, W1p, a1p, 32, fused_rs=True)
    down = tp.RowParallelMuxLinear(be, W2p, a2p, 32, fused_rs=True)
    for _ in range(2):   # twice: the receive slots and flags are reused (seq 1, 2)
        h = up.forward(seg_off, st, X)
        y = down.forward(seg_off, st, h)
        dh, dA2, dB2 = down.backward(seg_off, st, dY)
        dx, dA1, dB1 = up.backward(seg_off, st, dh)
    torch.cuda.synchronize()
    got = [y.clone(), dx.clone()] + [t.clone() for t in dA1 + dB1 + dA2 + dB2]
    H, Hs1 = mux.linear_fwd(seg_off, st, a1, X, W1, 32)
    Y, Hs2 = mux.linear_fwd(seg_off, st, a2, H, W2, 32)
    dH = mux.linear_bwd(seg_off, st, a2, dY, H, W2, Hs2, 32)
    dX = mux.linear_bwd(seg_off, st, a1, dH, X, W1, Hs1, 32)
    torch.cuda.synchronize()
    ref = [Y, dX] + [a.dA for a in a1] + [a.dB for a in a1] + [a.dA for a in a2] + [a.dB for a in a2]
    for a_, b_ in zip(got, ref):
        assert torch.equal(_bits(a_), _bits(b_))


def test_tp_fused_ag_world1_double_forward(pg):
    """fused_ag holds the gather buffer from the forward until the backward re-read X.  A second
    forward before that backward must raise (pushing again would wait forever for this rank's own
    release and trap the context); release_ag() makes a forward-only re-call legal; the chain
    with the all-gather fused equals direct binding calls, bit for bit."""
    g = torch.Generator(device="cuda").manual_seed(31)
    R, K, N = 512, 256, 384
    seg_off = torch.tensor([0, 192, 320, 512], dtype=torch.int32, device="cuda")
    st = [0, 1, 2]
    ranks = [16, 8, 32]
    W = (torch.randn(N, K, device="cuda", generator=g) / K ** 0.5).bfloat16()
    ads = []
    for r in ranks:
        B = mux.make_B_storage(N, r)
        B.copy_(torch.randn(N, r, device="cuda", generator=g).bfloat16())
        ads.append(mux.Adapter((torch.randn(r, K, device="cuda", generator=g) / K ** 0.5).bfloat16(), B, r, 2.0))
    X = torch.randn(R, K, device="cuda", generator=g).bfloat16()
    dY = torch.randn(R, N, device="cuda", generator=g).bfloat16()
    mk = lambda A, B, r, s: mux.Adapter(A, B, r, s)  # noqa: E731
    Wp, ap = tp.shard_column(W, ads, 1, 0, mk)
    up = tp.ColumnParallelMuxLinear(tp.MuxBackend(), Wp, ap, 32, fused_ag=True)
    up.forward(seg_off, st, X)
    with pytest.raises(RuntimeError, match="before the backward"):
        up.forward(seg_off, st, X)
    up.release_ag()                      # forward-only use: give the gather back, then call again
    y = up.forward(seg_off, st, X).clone()
    dx, dA, dB = up.backward(seg_off, st, dY)
    torch.cuda.synchronize()
    got = [y, dx.clone()] + [t.clone() for t in dA + dB]
    Y, Hs = mux.linear_fwd(seg_off, st, ads, X, W, 32)
    dX = mux.linear_bwd(seg_off, st, ads, dY, X, W, Hs, 32)
    torch.cuda.synchronize()
    ref = [Y, dX] + [a.dA for a in ads] + [a.dB for a in ads]
    for a_, b_ in zip(got, ref):
        assert torch.equal(_bits(a_), _bits(b_))
