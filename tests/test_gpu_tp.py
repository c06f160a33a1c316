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

from paper_2603_02885_b200 import mux, tp  # noqa: E402


def _bits(t):
    return t.view(torch.int16) if t.dtype == torch.bfloat16 else t


def test_tp_world1_equals_direct():
    os.environ.setdefault("MASTER_ADDR", "127.0.0.1")
    os.environ.setdefault("MASTER_PORT", "29533")
    if not dist.is_initialized():
        dist.init_process_group("nccl", rank=0, world_size=1, device_id=torch.device("cuda", 0))
    try:
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
        up = tp.ColumnParallelMuxLinear(be, W1p, a1p, 32)
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
    finally:
        dist.destroy_process_group()
