"""Tensor-parallel decoder block (tp_block.py) on the GPU at world size 1 (NCCL, collectives are
identities): the forward equals the single-GPU DecoderBlock (block.py) bit for bit; the backward
differs only in where the q/k/v (and gate/up) input-gradient partials are summed (bf16 adds before
the reduce-scatter vs fp32 inside RMSNorm's backward), so dx is within the north_star tolerance of
it and the adapter gradients are equal.  And bench.py's N > 1 command line end to end: two ranks
sharing this GPU over gloo (test-only backend) print one line with n_gpus 2 and mode tp, for the
config-2 layer stack and the config-4 decoder block."""
import json
import os
import subprocess
import sys

import pytest

pytestmark = pytest.mark.gpu

torch = pytest.importorskip("torch")
if not torch.cuda.is_available():
    pytest.skip("needs a CUDA device", allow_module_level=True)

import torch.distributed as dist  # noqa: E402

from paper_2603_02885_b200 import mux, tp, tp_block  # noqa: E402
from paper_2603_02885_b200.block import LINEARS, BlockShape, DecoderBlock  # noqa: E402

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


@pytest.fixture(scope="module")
def pg():
    os.environ.setdefault("MASTER_ADDR", "127.0.0.1")
    os.environ.setdefault("MASTER_PORT", "29541")
    if not dist.is_initialized():
        dist.init_process_group("nccl", rank=0, world_size=1, device_id=torch.device("cuda", 0))
    yield
    dist.destroy_process_group()


def _rel(a, b):
    return float((a.float() - b.float()).abs().max() / b.float().abs().max().clamp_min(1e-30))


@pytest.mark.parametrize("fused,shared_shrink", [(False, False), (True, False), (True, True)])
def test_tp_block_world1_matches_block(pg, fused, shared_shrink):
    """fused: q|k|v and gate|up as one column-sliced GEMM each (include/mux.h "Fused projections");
    the output columns of a slice get the same backbone sum and the same adapter product (plus exact
    zeros where a tile straddles two slices), so the forward is still the DecoderBlock's bit for bit."""
    g = torch.Generator(device="cuda").manual_seed(17)
    shape = BlockShape(hidden=256, ffn=384, heads=2, kv_heads=1)
    lens = [100, 30, 200, 64, 1, 50]
    task_off = [0, 2, 3, 6]
    ranks = [4, 8, 16]
    M = 3
    R = int(mux.pack_bound_rows(sum(lens), len(lens), 64))
    pk = mux.pack_chunks(task_off, lens, None, 0, 64, max_rows=R, max_chunks=R // 64)
    sl = torch.tensor(lens, dtype=torch.int32, device="cuda")
    rs = mux.row_start(sl, pk["seq_row"], R)
    dims = shape.linear_dims()
    W = {n: (torch.randn(dims[n][1], dims[n][0], device="cuda", generator=g) * dims[n][0] ** -0.5
             * (0.5 if n in ("q", "k") else 1.0)).bfloat16() for n in LINEARS}
    for i in (1, 2):
        W[f"norm{i}"] = (1 + 0.1 * torch.randn(256, device="cuda", generator=g)).bfloat16()

    def adapters():
        out = {}
        for n in LINEARS:
            K, N = dims[n]
            out[n] = []
            for r in ranks:
                B = mux.make_B_storage(N, r)
                B.copy_(torch.randn(N, r, device="cuda", generator=g).bfloat16())
                out[n].append(mux.Adapter((torch.randn(r, K, device="cuda", generator=g) * K ** -0.5).bfloat16(),
                                          B, r, 2.0))
        return out
    ads = adapters()
    ads2 = {n: [mux.Adapter(a.A, a.B, a.rank, a.scale) for a in ads[n]] for n in LINEARS}
    Xtok = torch.randn(sum(lens), 256, device="cuda", generator=g).bfloat16()
    x = mux.pack_apply(pk["row_src"], Xtok, R)
    dy = mux.pack_apply(pk["row_src"], torch.randn(sum(lens), 256, device="cuda", generator=g).bfloat16(), R)
    st = list(range(M))

    ref = DecoderBlock(shape, W, ads, 16)
    y_ref = ref.forward(x, pk["seg_off"], st, rs).clone()
    dx_ref = ref.backward(dy).clone()
    torch.cuda.synchronize()

    mk = lambda A, B, r, s: mux.Adapter(A, B, r, s)  # noqa: E731
    col_off = None
    if fused:
        Wp, ap, col_off = tp_block.shard_block_fused(W, ads2, 1, 0, mk)
    else:
        Wp, ap = tp_block.shard_block(W, ads2, 1, 0, mk)
    tshape = tp_block.TPBlockShape(hidden=256, ffn=384, heads=2, kv_heads=1, p=1)
    blk = tp_block.TPDecoderBlock(tp.MuxBackend(), tshape, Wp, ap, 16, col_off=col_off, shared_shrink=shared_shrink)
    for _ in range(2):   # twice: cached buffers are reused
        y = blk.forward(x, pk["seg_off"], st, rs)
        dx = blk.backward(dy)
    torch.cuda.synchronize()
    # rows >= seg_off[M] belong to no segment: the linears leave them unwritten (mux.h), so the block's
    # output there is whatever the buffers held; compare the packed rows
    n = int(mux.read_info(pk["info"])["total_rows"])
    assert torch.equal(y[:n].view(torch.int16), y_ref[:n].view(torch.int16))
    assert _rel(dx[:n], dx_ref[:n]) <= 2e-2
    got = blk.adapter_grads()
    for n in LINEARS:
        for t in range(M):
            assert _rel(got[n][0][t], ads[n][t].dA) <= 2e-2, n
            assert _rel(got[n][1][t], ads[n][t].dB) <= 2e-2, n


def _bench(args, timeout=900):
    env = dict(os.environ, MUX_BENCH_DIST_BACKEND="gloo")
    env.pop("WORLD_SIZE", None)
    r = subprocess.run([sys.executable, os.path.join(ROOT, "bench.py")] + args, capture_output=True, text=True,
                       timeout=timeout, env=env, cwd=ROOT)
    assert r.returncode == 0, r.stderr[-3000:]
    lines = [ln for ln in r.stdout.splitlines() if ln.startswith("{")]
    assert len(lines) == 1, r.stdout[-2000:]
    return json.loads(lines[0])


@pytest.mark.parametrize("config", ["2", "2crc", "4"])
def test_bench_gpus2_runs_tp(config):
    extra = ["--chain", "crc"] if config == "2crc" else []
    line = _bench(["--gpus", "2", "--steps", "2", "--warmup", "3", "--config", config[0], "--no-replicas"] + extra)
    assert line["n_gpus"] == 2 and line["mode"] == "tp" and line["scaling"] == "strong"
    assert line["value"] > 0 and line["e2e"]["value"] > 0
    assert line["roofline"]["achieved"] > 0 and line["gpu_launches"] > 0
    # a physically possible rate: every packed row computed (a pack overflow would skip rows)
    assert line["roofline"]["frac_of_burst"] < 1.05 and line["frac_of_peak_per_gpu"]["measured_burst"] < 1.05
    assert line["config"]["dist_backend"] == "gloo"
