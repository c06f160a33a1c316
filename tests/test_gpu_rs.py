"""Fused GEMM -> reduce-scatter (mux_linear_fwd_rs / mux_linear_bwd_dx_rs +
mux_rs_reduce) on ONE GPU with `world` simulated ranks:
every rank's receive buffer and flag block live on cuda:0, so the epilogue's
stores to "peer" slots, the ready/ack handshake and the owner-side reduction
run exactly as they would over NVLink, minus the link.

Checks, over three consecutive calls (so every receive slot is reused and the
ack handshake is exercised):
* the reduced rows equal the fp32 sum, in ascending rank order, of the
  per-rank bf16 partials computed by the plain fused kernels on the same
  shards — bit for bit (same kernel, same tiles, same summation order);
* and the full-problem fp64 oracle within the north_star tolerance.
Row-parallel forward (W split on K) and column-parallel dX (W split on N)."""
import numpy as np
import pytest

pytestmark = pytest.mark.gpu

torch = pytest.importorskip("torch")
if not torch.cuda.is_available():
    pytest.skip("needs a CUDA device", allow_module_level=True)

from paper_2603_02885_b200 import mux  # noqa: E402
from oracle import linear as olin  # noqa: E402
from gpu_harness import TOL, rel_err  # noqa: E402


def _bits(t):
    return t.view(torch.int16)


def _adapters(g, ranks, K, N):
    ads = []
    for r in ranks:
        B = mux.make_B_storage(N, r)
        B.copy_(torch.randn(N, r, device="cuda", generator=g).bfloat16())
        ads.append(mux.Adapter((torch.randn(r, K, device="cuda", generator=g) / K ** 0.5).bfloat16(), B, r, 2.0))
    return ads


@pytest.mark.parametrize("world", [2, 4])
def test_row_parallel_fwd_rs(world):
    g = torch.Generator(device="cuda").manual_seed(100 + world)
    rows_per_rank = 256
    R, K, N = world * rows_per_rank, 128 * world, 384
    seg_off = torch.tensor([0, 192, 448, R], dtype=torch.int32, device="cuda")
    st, ranks = [0, 1, 2], [16, 8, 4]
    W = (torch.randn(N, K, device="cuda", generator=g) / K ** 0.5).bfloat16()
    full_ads = _adapters(g, ranks, K, N)
    k = K // world
    Wp = [W[:, p * k:(p + 1) * k].contiguous() for p in range(world)]
    ads_p = [[mux.Adapter(a.A[:, p * k:(p + 1) * k].contiguous(), a.B, a.rank, a.scale) for a in full_ads]
             for p in range(world)]
    recv = [torch.zeros(world * rows_per_rank * N, dtype=torch.bfloat16, device="cuda") for _ in range(world)]
    flags = [torch.zeros(mux.rs_flags_elems(world), dtype=torch.int64, device="cuda") for _ in range(world)]
    ws = [torch.zeros(mux.linear_workspace_size(3, R, k, N, 16), dtype=torch.uint8, device="cuda")
          for _ in range(world)]
    outs = [torch.empty(rows_per_rank, N, dtype=torch.bfloat16, device="cuda") for _ in range(world)]
    for seq in (1, 2, 3):
        X = torch.randn(R, K, device="cuda", generator=g).bfloat16()
        Xp = [X[:, p * k:(p + 1) * k].contiguous() for p in range(world)]
        for p in range(world):
            rs = mux.make_rs(world, p, rows_per_rank, seq, recv, flags)
            mux.linear_fwd_rs(rs, seg_off, st, ads_p[p], Xp[p], Wp[p], 16, workspace=ws[p])
        for p in range(world):
            mux.rs_reduce(mux.make_rs(world, p, rows_per_rank, seq, recv, flags), outs[p])
        # reference 1: plain fused kernels per shard, summed in fp32 in rank order
        parts = [mux.linear_fwd(seg_off, st, ads_p[p], Xp[p], Wp[p], 16)[0] for p in range(world)]
        acc = parts[0].float()
        for p in range(1, world):
            acc = acc + parts[p].float()
        torch.cuda.synchronize()
        ref = acc.bfloat16()
        for p in range(world):
            assert torch.equal(_bits(outs[p]), _bits(ref[p * rows_per_rank:(p + 1) * rows_per_rank])), (seq, p)
        # reference 2: the fp64 oracle of the whole (unsharded) layer
        Yo, _ = olin.linear_fwd(seg_off.cpu().numpy(), st, [a.A.float().cpu().numpy() for a in full_ads],
                                [a.B.float().cpu().numpy() for a in full_ads], ranks, [2.0] * 3,
                                X.float().cpu().numpy(), W.float().cpu().numpy(), 16)
        got = torch.cat(outs).float().cpu().numpy()
        assert rel_err(got, Yo) <= TOL


@pytest.mark.parametrize("world", [2, 4])
def test_column_parallel_dx_rs(world):
    g = torch.Generator(device="cuda").manual_seed(200 + world)
    rows_per_rank = 256
    R, K, N = world * rows_per_rank, 320, 128 * world
    seg_off = torch.tensor([0, 64, 320, R], dtype=torch.int32, device="cuda")
    st, ranks = [0, 1, 2], [8, 16, 32]
    W = (torch.randn(N, K, device="cuda", generator=g) / K ** 0.5).bfloat16()
    full_ads = _adapters(g, ranks, K, N)
    n = N // world
    Wp = [W[p * n:(p + 1) * n].contiguous() for p in range(world)]
    recv = [torch.zeros(world * rows_per_rank * K, dtype=torch.bfloat16, device="cuda") for _ in range(world)]
    flags = [torch.zeros(mux.rs_flags_elems(world), dtype=torch.int64, device="cuda") for _ in range(world)]
    outs = [torch.empty(rows_per_rank, K, dtype=torch.bfloat16, device="cuda") for _ in range(world)]
    X = torch.randn(R, K, device="cuda", generator=g).bfloat16()
    for seq in (1, 2, 3):
        dY = torch.randn(R, N, device="cuda", generator=g).bfloat16()
        ads_p, ws, Hs_p = [], [], []
        for p in range(world):
            ap = [mux.Adapter(a.A, a.B[p * n:(p + 1) * n], a.rank, a.scale) for a in full_ads]
            ads_p.append(ap)
            ws.append(torch.zeros(mux.linear_workspace_size(3, R, K, n, 32), dtype=torch.uint8, device="cuda"))
            Hs_p.append(mux.linear_fwd(seg_off, st, ap, X, Wp[p], 32)[1])
        dYp = [dY[:, p * n:(p + 1) * n].contiguous() for p in range(world)]
        for p in range(world):
            rs = mux.make_rs(world, p, rows_per_rank, seq, recv, flags)
            mux.linear_bwd_dx_rs(rs, seg_off, st, ads_p[p], dYp[p], X, Wp[p], Hs_p[p], 32, ws[p])
            mux.linear_bwd(seg_off, st, ads_p[p], dYp[p], X, Wp[p], Hs_p[p], 32, workspace=ws[p],
                           part=mux.BWD_GRADS)
        for p in range(world):
            mux.rs_reduce(mux.make_rs(world, p, rows_per_rank, seq, recv, flags), outs[p])
        parts = [mux.linear_bwd(seg_off, st, [mux.Adapter(a.A, a.B, a.rank, a.scale) for a in ads_p[p]], dYp[p], X,
                                Wp[p], Hs_p[p], 32) for p in range(world)]
        acc = parts[0].float()
        for p in range(1, world):
            acc = acc + parts[p].float()
        torch.cuda.synchronize()
        ref = acc.bfloat16()
        for p in range(world):
            assert torch.equal(_bits(outs[p]), _bits(ref[p * rows_per_rank:(p + 1) * rows_per_rank])), (seq, p)
        dXo, _, _ = olin.linear_bwd(seg_off.cpu().numpy(), st, [a.A.float().cpu().numpy() for a in full_ads],
                                    [a.B.float().cpu().numpy() for a in full_ads], ranks, [2.0] * 3,
                                    dY.float().cpu().numpy(), X.float().cpu().numpy(), W.float().cpu().numpy(), 32)
        got = torch.cat(outs).float().cpu().numpy()
        assert rel_err(got, dXo) <= TOL


def test_rs_rejects_bad_layout():
    recv = [torch.zeros(2 * 256 * 128, dtype=torch.bfloat16, device="cuda") for _ in range(2)]
    flags = [torch.zeros(mux.rs_flags_elems(2), dtype=torch.int64, device="cuda") for _ in range(2)]
    X = torch.zeros(512, 128, dtype=torch.bfloat16, device="cuda")
    W = torch.zeros(128, 128, dtype=torch.bfloat16, device="cuda")
    so = torch.tensor([0, 512], dtype=torch.int32, device="cuda")
    ads = [mux.Adapter(None, None, 0, 0.0)]
    with pytest.raises((mux.MuxError, ValueError)):   # rows_per_rank not a multiple of 256
        mux.linear_fwd_rs(mux.make_rs(2, 0, 128, 1, recv, flags), so, [0], ads, X[:256], W, 16)
    with pytest.raises((mux.MuxError, ValueError)):   # world * rows_per_rank != max_rows
        mux.linear_fwd_rs(mux.make_rs(2, 0, 256, 1, recv, flags), so, [0], ads, X[:256], W, 16)
    with pytest.raises((mux.MuxError, ValueError)):   # seq 0
        mux.linear_fwd_rs(mux.make_rs(2, 0, 256, 0, recv, flags), so, [0], ads, X, W, 16)


@pytest.mark.parametrize("world", [2, 4])
def test_all_gather_fused_gemm(world):
    """mux_ag_push (copy engines, on a copy stream) + mux_linear_fwd_ag / mux_linear_bwd_ag (the
    producer waits per row block for its owner's rows) + mux_ag_release, world simulated ranks on
    one GPU, three calls reusing the gather buffers: every rank's result == the plain kernels on the
    full input, bit for bit (the gather buffer holds exactly the full input)."""
    g = torch.Generator(device="cuda").manual_seed(300 + world)
    rows_per_rank = 256
    R, K, N = world * rows_per_rank, 192, 320
    seg_off = torch.tensor([0, 128, 320, R], dtype=torch.int32, device="cuda")
    st, ranks = [0, 1, 2], [16, 4, 8]
    W = (torch.randn(N, K, device="cuda", generator=g) / K ** 0.5).bfloat16()
    ads = _adapters(g, ranks, K, N)
    gx = [torch.zeros(R * K, dtype=torch.bfloat16, device="cuda") for _ in range(world)]    # gather X
    gd = [torch.zeros(R * N, dtype=torch.bfloat16, device="cuda") for _ in range(world)]    # gather dY
    fx = [torch.zeros(mux.rs_flags_elems(world), dtype=torch.int64, device="cuda") for _ in range(world)]
    fd = [torch.zeros(mux.rs_flags_elems(world), dtype=torch.int64, device="cuda") for _ in range(world)]
    copy = torch.cuda.Stream()
    for seq in (1, 2, 3):
        X = torch.randn(R, K, device="cuda", generator=g).bfloat16()
        dY = torch.randn(R, N, device="cuda", generator=g).bfloat16()
        agx = [mux.make_ag(world, p, rows_per_rank, seq, gx, fx) for p in range(world)]
        agd = [mux.make_ag(world, p, rows_per_rank, seq, gd, fd) for p in range(world)]
        ev = torch.cuda.Event()
        ev.record()
        copy.wait_event(ev)   # the inputs of this call are ready
        for p in range(world):
            mux.ag_push(agx[p], X[p * rows_per_rank:(p + 1) * rows_per_rank], stream=copy)
            mux.ag_push(agd[p], dY[p * rows_per_rank:(p + 1) * rows_per_rank], stream=copy)
        outs = []
        for p in range(world):
            pads = [mux.Adapter(a.A, a.B, a.rank, a.scale) for a in ads]
            Y, Hs = mux.linear_fwd_ag(agx[p], seg_off, st, pads, K, W, 16)
            dX = mux.linear_bwd_ag(agd[p], seg_off, st, pads, gx[p].view(R, K), W, Hs, 16)
            mux.ag_release(agx[p])
            mux.ag_release(agd[p])
            outs.append((Y, dX, pads))
        Yr, Hsr = mux.linear_fwd(seg_off, st, ads, X, W, 16)
        dXr = mux.linear_bwd(seg_off, st, ads, dY, X, W, Hsr, 16)
        torch.cuda.synchronize()
        for p, (Y, dX, pads) in enumerate(outs):
            assert torch.equal(_bits(Y), _bits(Yr)), (seq, p)
            assert torch.equal(_bits(dX), _bits(dXr)), (seq, p)
            for a, b in zip(pads, ads):
                assert torch.equal(a.dA, b.dA) and torch.equal(a.dB, b.dB)
    torch.cuda.current_stream().wait_stream(copy)
