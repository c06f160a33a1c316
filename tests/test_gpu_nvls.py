"""In-switch collectives (NVLink SHARP; libmux mux_nvls_*, csrc/nvls.cu; NEXT-1 P:799-802) on the
GPU at world size 1 — the only world this box has: a 1-device multicast object, so
multimem.ld_reduce returns the rank's own copy and multimem.st writes it; the counters advance by
one per call.  Checks the mechanics bit for bit (buffer mapping, the multimem instructions, the
ready/done/consumed counters over several calls with slot reuse) and the tensor-parallel layers and
decoder block with every collective on NVLS equal to the NCCL path, bit for bit."""
import os

import pytest

pytestmark = pytest.mark.gpu

torch = pytest.importorskip("torch")
if not torch.cuda.is_available():
    pytest.skip("needs a CUDA device", allow_module_level=True)

import torch.distributed as dist  # noqa: E402

from paper_2603_02885_b200 import mux, tp, tp_block  # noqa: E402
from paper_2603_02885_b200.block import LINEARS, BlockShape  # noqa: E402
from paper_2603_02885_b200.nvls import NvlsBuffer, NvlsUnavailable  # noqa: E402


def _multicast_or_skip():
    """Boxes whose process cannot create a CUDA multicast object (the GPU reports multicast support,
    but cuMulticastCreate returns CUDA_ERROR_INVALID_VALUE without NVSwitch fabric access, as in the
    single-GPU sandbox this suite was developed on; tools/probe/mc_probe.cu) skip with that reason."""
    try:
        NvlsBuffer(None, 256, 64)
    except NvlsUnavailable as e:
        pytest.skip(f"NVLS multicast unavailable on this box: {e}")


@pytest.fixture(scope="module")
def pg():
    os.environ.setdefault("MASTER_ADDR", "127.0.0.1")
    os.environ.setdefault("MASTER_PORT", "29551")
    if not dist.is_initialized():
        dist.init_process_group("nccl", rank=0, world_size=1, device_id=torch.device("cuda", 0))
    yield
    dist.destroy_process_group()


@pytest.fixture(autouse=True)
def _needs_multicast(pg):
    _multicast_or_skip()


def _bits(t):
    return t.view(torch.int16)


def test_nvls_buffer_rs_ag_counters(pg):
    g = torch.Generator(device="cuda").manual_seed(1)
    rows, cols = 512, 384
    rsb = NvlsBuffer(None, rows, cols)
    agb = NvlsBuffer(None, rows, cols)
    flags = torch.as_tensor(__import__("paper_2603_02885_b200.nvls", fromlist=["_Cai"])._Cai(
        rsb.uc_flags_ptr, (8,), "<i8"), device="cuda")
    for call in range(1, 4):
        part = torch.randn(rows, cols, device="cuda", generator=g).bfloat16()
        rsb.uc.copy_(part)
        out = torch.empty(rows, cols, dtype=torch.bfloat16, device="cuda")
        rsb.reduce_scatter(out, ctas=8)
        src = torch.randn(rows, cols, device="cuda", generator=g).bfloat16()
        got = agb.all_gather(src, ctas=4)
        torch.cuda.synchronize()
        assert torch.equal(_bits(out), _bits(part))
        assert torch.equal(_bits(got), _bits(src))
        agb.release()
        torch.cuda.synchronize()
        assert flags[0].item() == call and flags[1].item() == call    # ready / done, world 1
    # a strided output (row stride 512) and a strided source
    wide = torch.zeros(rows, 512, dtype=torch.bfloat16, device="cuda")
    rsb.uc.copy_(part)
    rsb.reduce_scatter(wide[:, :cols])
    torch.cuda.synchronize()
    assert torch.equal(_bits(wide[:, :cols]), _bits(part)) and not wide[:, cols:].any()


def _make(K, N, ranks, g):
    W = (torch.randn(N, K, device="cuda", generator=g) / K ** 0.5).bfloat16()
    ads = []
    for r in ranks:
        B = mux.make_B_storage(N, r)
        B.copy_(torch.randn(N, r, device="cuda", generator=g).bfloat16())
        ads.append(mux.Adapter((torch.randn(r, K, device="cuda", generator=g) / K ** 0.5).bfloat16(), B, r, 2.0))
    return W, ads


def test_tp_layers_nvls_world1_equal_direct(pg):
    g = torch.Generator(device="cuda").manual_seed(3)
    R, K, N = 512, 256, 384
    seg_off = torch.tensor([0, 192, 320, 512], dtype=torch.int32, device="cuda")
    st, ranks = [0, 1, 2], [16, 8, 32]
    W1, a1 = _make(K, N, ranks, g)
    W2, a2 = _make(N, K, ranks, g)
    X = torch.randn(R, K, device="cuda", generator=g).bfloat16()
    dY = torch.randn(R, K, device="cuda", generator=g).bfloat16()
    mk = lambda A, B, r, s: mux.Adapter(A, B, r, s)  # noqa: E731
    nv = tp.NvlsCollectives(None, ctas=8)
    be = tp.MuxBackend()
    up = tp.ColumnParallelMuxLinear(be, *tp.shard_column(W1, a1, 1, 0, mk), 32, nvls=nv)
    down = tp.RowParallelMuxLinear(be, *tp.shard_row(W2, a2, 1, 0, mk), 32, nvls=nv)
    for _ in range(3):     # buffers and counters reused
        y = down.forward(seg_off, st, up.forward(seg_off, st, X)).clone()
        dh, dA2, dB2 = down.backward(seg_off, st, dY)
        dx, dA1, dB1 = up.backward(seg_off, st, dh)
    torch.cuda.synchronize()
    got = [y, dx.clone()] + [t.clone() for t in dA1 + dB1 + dA2 + dB2]
    H, Hs1 = mux.linear_fwd(seg_off, st, a1, X, W1, 32)
    Y, Hs2 = mux.linear_fwd(seg_off, st, a2, H, W2, 32)
    dH = mux.linear_bwd(seg_off, st, a2, dY, H, W2, Hs2, 32)
    dX = mux.linear_bwd(seg_off, st, a1, dH, X, W1, Hs1, 32)
    torch.cuda.synchronize()
    ref = [Y, dX] + [a.dA for a in a1] + [a.dB for a in a1] + [a.dA for a in a2] + [a.dB for a in a2]
    for a_, b_ in zip(got, ref):
        assert torch.equal(a_.view(torch.int16) if a_.dtype == torch.bfloat16 else a_,
                           b_.view(torch.int16) if b_.dtype == torch.bfloat16 else b_)
    with pytest.raises(RuntimeError, match="before the backward"):
        up.forward(seg_off, st, X)
        up.forward(seg_off, st, X)


def test_tp_block_nvls_world1_equals_nccl(pg):
    g = torch.Generator(device="cuda").manual_seed(9)
    shape = BlockShape(hidden=256, ffn=384, heads=2, kv_heads=2)
    lens = [100, 30, 200, 64, 50]
    R = int(mux.pack_bound_rows(sum(lens), len(lens), 64))
    pk = mux.pack_chunks([0, 2, 3, 5], lens, None, 0, 64, max_rows=R, max_chunks=R // 64)
    rs = mux.row_start(torch.tensor(lens, dtype=torch.int32, device="cuda"), pk["seq_row"], R)
    dims = shape.linear_dims()
    ranks = [4, 16, 8]
    W, ads = {}, {}
    for n in LINEARS:
        W[n], ads[n] = _make(dims[n][0], dims[n][1], ranks, g)
    for i in (1, 2):
        W[f"norm{i}"] = (1 + 0.1 * torch.randn(256, device="cuda", generator=g)).bfloat16()
    x = mux.pack_apply(pk["row_src"], torch.randn(sum(lens), 256, device="cuda", generator=g).bfloat16(), R)
    dy = mux.pack_apply(pk["row_src"], torch.randn(sum(lens), 256, device="cuda", generator=g).bfloat16(), R)
    mk = lambda A, B, r, s: mux.Adapter(A, B, r, s)  # noqa: E731
    tshape = tp_block.TPBlockShape(hidden=256, ffn=384, heads=2, kv_heads=2, p=1)
    outs = []
    for nv in (None, tp.NvlsCollectives(None, ctas=8)):
        Wp, ap = tp_block.shard_block(W, {n: [mux.Adapter(a.A, a.B, a.rank, a.scale) for a in ads[n]]
                                          for n in LINEARS}, 1, 0, mk)
        blk = tp_block.TPDecoderBlock(tp.MuxBackend(), tshape, Wp, ap, 16, nvls=nv)
        for _ in range(2):
            y = blk.forward(x, pk["seg_off"], [0, 1, 2], rs).clone()
            dx = blk.backward(dy).clone()
        torch.cuda.synchronize()
        grads = [t.clone() for n in LINEARS for lst in blk.adapter_grads()[n] for t in lst]
        outs.append([y, dx] + grads)
    for a_, b_ in zip(*outs):
        assert torch.equal(a_.view(torch.int16) if a_.dtype == torch.bfloat16 else a_,
                           b_.view(torch.int16) if b_.dtype == torch.bfloat16 else b_)
