"""Two processes, one GPU: tensor parallelism with the reduce-scatter fused
into the GEMM epilogue (tp.py fused_rs=True) and, optionally, the all-gather
pushed by the copy engines and consumed inside the GEMM (fused_ag=True),
across real process boundaries.
Both ranks live on cuda:0 (the box has one GPU), so the "peer" stores go
through CUDA IPC mappings of the other process's buffers instead of NVLink,
and the ready/ack flags are exchanged between processes exactly as between
GPUs.  torch symmetric memory refuses two ranks on one device, so the receive
buffers and flags are mapped with CUDA IPC handles (torch.multiprocessing
shares CUDA tensors between processes) through FusedRs's exchange hook.  The
process group is gloo (NCCL refuses two ranks on one device); the
all-gathers and all-reduces of the layer classes run on it.

The gathered result of a column-parallel -> row-parallel chain (fwd + bwd,
with dA/dB) must match the single-process direct calls within the
north_star tolerance (the sharded reduction sums two bf16 partials)."""
import os
import socket

import numpy as np
import pytest

pytestmark = pytest.mark.gpu

torch = pytest.importorskip("torch")
if not torch.cuda.is_available():
    pytest.skip("needs a CUDA device", allow_module_level=True)

import torch.multiprocessing as mp  # noqa: E402

R, K, N = 512, 256, 384
SEG = [0, 192, 320, 512]
RANKS = [16, 8, 32]


def _problem():
    from paper_2603_02885_b200 import mux
    g = torch.Generator(device="cuda").manual_seed(31)

    def make(KK, NN):
        W = (torch.randn(NN, KK, device="cuda", generator=g) / KK ** 0.5).bfloat16()
        ads = []
        for r in RANKS:
            B = mux.make_B_storage(NN, r)
            B.copy_(torch.randn(NN, r, device="cuda", generator=g).bfloat16())
            ads.append(mux.Adapter((torch.randn(r, KK, device="cuda", generator=g) / KK ** 0.5).bfloat16(),
                                   B, r, 2.0))
        return W, ads

    W1, a1 = make(K, N)
    W2, a2 = make(N, K)
    X = torch.randn(R, K, device="cuda", generator=g).bfloat16()
    dY = torch.randn(R, K, device="cuda", generator=g).bfloat16()
    return W1, a1, W2, a2, X, dY


def _worker(rank, world, port, q, boxes, fused_ag, shared_shrink=False):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    import torch.distributed as dist
    torch.cuda.set_device(0)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        from paper_2603_02885_b200 import mux, tp
        W1, a1, W2, a2, X, dY = _problem()
        seg_off = torch.tensor(SEG, dtype=torch.int32, device="cuda")
        st = [0, 1, 2]
        mk = lambda A, B, r, s: mux.Adapter(A, B, r, s)  # noqa: E731
        be = tp.MuxBackend()
        keep = []

        def exchange(recv, flags):
            # hand this rank's buffers to every other rank (CUDA IPC), collect theirs
            for d in range(world):
                if d != rank:
                    boxes[d].put((rank, recv, flags))
            got = {rank: (recv, flags)}
            for _ in range(world - 1):
                src, rv, fl = boxes[rank].get(timeout=120)
                got[src] = (rv, fl)
            keep.append(got)
            return [got[d][0].data_ptr() for d in range(world)], [got[d][1].data_ptr() for d in range(world)]
        be.rs_exchange = exchange
        W1p, a1p = tp.shard_column(W1, a1, world, rank, mk)
        W2p, a2p = tp.shard_row(W2, a2, world, rank, mk)
        up = tp.ColumnParallelMuxLinear(be, W1p, a1p, 32, fused_rs=True, fused_ag=fused_ag,
                                        shared_shrink=shared_shrink)
        down = tp.RowParallelMuxLinear(be, W2p, a2p, 32, fused_rs=True, fused_ag=fused_ag)
        rows = R // world
        for _ in range(2):   # twice: receive slots and flags reused
            h = up.forward(seg_off, st, X[rank * rows:(rank + 1) * rows].contiguous())
            y = down.forward(seg_off, st, h)
            dh, dA2, dB2 = down.backward(seg_off, st, dY[rank * rows:(rank + 1) * rows].contiguous())
            dx, dA1, dB1 = up.backward(seg_off, st, dh)
        torch.cuda.synchronize()
        q.put((rank, y.float().cpu().numpy(), dx.float().cpu().numpy(),
               [t.cpu().numpy() for t in dA1], [t.cpu().numpy() for t in dB1],
               [t.cpu().numpy() for t in dA2], [t.cpu().numpy() for t in dB2], None))
    except Exception as e:  # noqa: BLE001
        q.put((rank, None, None, None, None, None, None, repr(e)))
    finally:
        dist.destroy_process_group()


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


@pytest.mark.parametrize("fused_ag,shared_shrink", [(False, False), (True, False), (False, True)])
def test_fused_rs_two_processes_one_gpu(fused_ag, shared_shrink):
    """shared_shrink: each process shrinks its own 256 rows (mux_linear_shrink), the Hs rows are
    all-gathered over the process group, and the column GEMM runs with the shrink given."""
    from paper_2603_02885_b200 import mux
    from gpu_harness import TOL, rel_err
    world = 2
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    boxes = [ctx.Queue() for _ in range(world)]
    procs = [ctx.Process(target=_worker, args=(r, world, port, q, boxes, fused_ag, shared_shrink))
             for r in range(world)]
    for p in procs:
        p.start()
    res = sorted([q.get(timeout=300) for _ in range(world)], key=lambda x: x[0])
    for p in procs:
        p.join(timeout=60)
    errs = [r[7] for r in res if r[7]]
    assert not errs, errs
    for p in procs:
        assert p.exitcode == 0
    # single-process reference
    W1, a1, W2, a2, X, dY = _problem()
    seg_off = torch.tensor(SEG, dtype=torch.int32, device="cuda")
    st = [0, 1, 2]
    H, Hs1 = mux.linear_fwd(seg_off, st, a1, X, W1, 32)
    Y, Hs2 = mux.linear_fwd(seg_off, st, a2, H, W2, 32)
    dH = mux.linear_bwd(seg_off, st, a2, dY, H, W2, Hs2, 32)
    dX = mux.linear_bwd(seg_off, st, a1, dH, X, W1, Hs1, 32)
    torch.cuda.synchronize()
    y = np.concatenate([r[1] for r in res])
    dx = np.concatenate([r[2] for r in res])
    assert rel_err(y, Y.float().cpu().numpy()) <= TOL
    assert rel_err(dx, dX.float().cpu().numpy()) <= TOL
    n = N // world
    for t in range(3):
        assert rel_err(res[0][3][t], a1[t].dA.cpu().numpy()) <= TOL                       # column dA: all-reduced
        assert rel_err(np.concatenate([r[4][t] for r in res]), a1[t].dB.cpu().numpy()) <= TOL   # column dB: N-sharded
        assert rel_err(np.concatenate([r[5][t] for r in res], axis=1), a2[t].dA.cpu().numpy()) <= TOL  # row dA
        assert rel_err(res[0][6][t], a2[t].dB.cpu().numpy()) <= TOL                       # row dB: all-reduced
    del n
