"""GPU parity: mux_linear_fwd / mux_linear_bwd (through the C ABI) vs the fp64 oracle.

Bar (north_star): max|gpu - oracle| / max|oracle| <= 2e-2 per tensor; integer
inputs bit-exact.  Shapes span several 128x256 tiles, ragged tails, 64-row
segments straddling 128-row tiles (two tasks in one tile), ranks 4..64 and 0,
empty segments, a task owning two segments, NaN isolation.
"""
import numpy as np
import pytest

pytestmark = pytest.mark.gpu

torch = pytest.importorskip("torch")
if not torch.cuda.is_available():
    pytest.skip("needs a CUDA device", allow_module_level=True)

from gpu_harness import Problem, compare, bf16_to_f64, TOL  # noqa: E402


def _run(prob, rows=None, exact=False, bwd=True):
    gpu = prob.run_gpu(bwd=bwd)
    ref = prob.run_oracle(bwd=bwd, rows=rows)
    return compare(prob, gpu, ref, rows=rows, exact=exact)


def test_config1_shape():
    """Config 1: d=256->256, 2 tasks rank 8, 64 tokens each."""
    errs = _run(Problem(256, 256, [64, 64], [8, 8], seed=11))
    print(errs)


def test_integer_exact_single_task():
    _run(Problem(256, 256, [128], [16], variant="int", scales=[2.0], seed=12), exact=True)


def test_integer_exact_straddle():
    """64-row segments: tiles 0 and 1 each hold two tasks (lane-masked adapter MMAs)."""
    p = Problem(512, 768, [64, 128, 64, 192], [8, 16, 32, 64], variant="int",
                scales=[1.0, 2.0, 1.0, 2.0], seed=13)
    _run(p, exact=True)


def test_multi_tile_ragged():
    """Several N tiles with a ragged tail (N = 640 = 2.5 tiles), K not a multiple of 256."""
    _run(Problem(320, 640, [192, 64, 256], [16, 4, 64], seed=14))


def test_dims_multiple_of_8_not_64():
    """K, N multiples of 8 only (e.g. an 8-way TP shard of 11008 = 1376):
    partial 64-wide k-blocks read TMA zero fill, partial output boxes clip."""
    _run(Problem(264, 200, [64, 128], [8, 16], seed=22))
    _run(Problem(1376, 328, [128, 64], [16, 4], variant="int", scales=[2.0, 1.0], seed=23), exact=True)


def test_heterogeneous_ranks_and_rank0():
    _run(Problem(256, 512, [128, 64, 64, 128], [4, 0, 48, 8], r_cap=48, seed=15))


def test_empty_segment_and_shared_task():
    """An empty segment (Q16) and task 0 owning two segments."""
    p = Problem(256, 256, [128, 0, 64, 64], [16, 32], seg_task=[0, 1, 1, 0], seed=16)
    errs = _run(p)
    print(errs)


def test_empty_task_grads_are_zero():
    p = Problem(256, 256, [128, 0], [16, 8], seg_task=[0, 1], seed=17)
    gpu = p.run_gpu()
    assert np.all(gpu["dA"][1] == 0) and np.all(gpu["dB"][1] == 0)


def test_zero_B_backbone():
    _run(Problem(256, 512, [128, 128], [16, 16], variant="zeroB", seed=18))


def test_max_rows_larger_than_rows():
    """max_rows > seg_off[S]: rows beyond are never written."""
    p = Problem(256, 256, [64, 64], [8, 8], seed=19, max_rows=384)
    _run(p)


def test_nan_isolation():
    """NaN in task 1's X rows and in task 2's B never reach other tasks."""
    p = Problem(256, 512, [64, 64, 128], [8, 16, 8], seed=20)
    p.X[70, 5] = np.uint16(0x7FC0)               # row of segment 1 (task 1), shares tile 0 with task 0
    p.B[2][3, 2] = np.uint16(0x7FC0)             # task 2's B
    gpu = p.run_gpu()
    Y = bf16_to_f64(gpu["Y"])
    dX = bf16_to_f64(gpu["dX"])
    assert np.all(np.isfinite(Y[:64])), "task 0 rows poisoned"
    assert np.all(np.isfinite(dX[:64]))
    assert np.all(np.isfinite(gpu["dA"][0])) and np.all(np.isfinite(gpu["dB"][0]))
    assert np.isnan(Y[70]).any()
    assert np.isnan(Y[128:]).any()               # task 2 (bad B) is itself affected


@pytest.mark.parametrize("K,N", [(4096, 4096), (4096, 11008), (11008, 4096)])
def test_config2_linears_sampled(K, N):
    """Config-2 shapes at a reduced token count (full K/N; 4 tasks r=16), with
    Y/dX compared on a sampled row set; Hs, dA, dB on every row."""
    lens = [256, 192, 320, 256]
    p = Problem(K, N, lens, [16] * 4, seed=21)
    rng = np.random.default_rng(0)
    rows = np.unique(np.concatenate([np.arange(0, 8), np.arange(p.R - 8, p.R),
                                     rng.integers(0, p.R, 48)])).astype(np.int64)
    errs = _run(p, rows=rows)
    print(errs)


def test_bwd_parts_overlapped_equal_combined():
    """mux_linear_bwd_part: the dX GEMM on one stream and the adapter gradients on a
    second stream (after an event) == mux_linear_bwd, bit for bit."""
    import torch
    from paper_2603_02885_b200 import mux
    g = torch.Generator(device="cuda").manual_seed(5)
    R, K, N = 1024, 512, 768
    seg_off = torch.tensor([0, 256, 640, 1024], dtype=torch.int32, device="cuda")
    st = [0, 1, 2]
    ranks = [16, 4, 32]
    W = (torch.randn(N, K, device="cuda", generator=g) / K ** 0.5).bfloat16()
    X = torch.randn(R, K, device="cuda", generator=g).bfloat16()
    dY = torch.randn(R, N, device="cuda", generator=g).bfloat16()

    def adapters():
        out = []
        gg = torch.Generator(device="cuda").manual_seed(9)
        for r in ranks:
            B = mux.make_B_storage(N, r)
            B.copy_(torch.randn(N, r, device="cuda", generator=gg).bfloat16())
            out.append(mux.Adapter((torch.randn(r, K, device="cuda", generator=gg) / K ** 0.5).bfloat16(), B, r, 2.0))
        return out

    a1, a2 = adapters(), adapters()
    _, Hs = mux.linear_fwd(seg_off, st, a1, X, W, 32)
    dX1 = mux.linear_bwd(seg_off, st, a1, dY, X, W, Hs, 32)
    ws = torch.zeros(mux.linear_workspace_size(3, R, K, N, 32), dtype=torch.uint8, device="cuda")
    side = torch.cuda.Stream()
    ev = torch.cuda.Event()
    dX2 = mux.linear_bwd(seg_off, st, a2, dY, X, W, Hs, 32, workspace=ws, part=mux.BWD_DX)
    ev.record()
    side.wait_event(ev)
    mux.linear_bwd(seg_off, st, a2, dY, X, W, Hs, 32, dX=dX2, workspace=ws, part=mux.BWD_GRADS, stream=side)
    torch.cuda.current_stream().wait_stream(side)
    torch.cuda.synchronize()
    assert torch.equal(dX1.view(torch.int16), dX2.view(torch.int16))
    for x, y in zip(a1, a2):
        assert torch.equal(x.dA, y.dA) and torch.equal(x.dB, y.dB)
    with pytest.raises(mux.MuxError):
        mux.linear_bwd(seg_off, st, a2, dY, X, W, Hs, 32, dX=dX2, workspace=ws, part=3)


@pytest.mark.parametrize("case", range(16))
def test_fuzz_random_problems(case):
    """Seeded random problems across the ABI's legal space: K, N multiples of 8 (not of 64),
    1-12 segments of multiples of 64 rows (empty ones included), tasks owning several segments,
    ranks 0-64 (r_cap the smallest legal), integer-valued inputs half of the time (then bit-exact)."""
    rng = np.random.default_rng(1000 + case)
    K = int(rng.integers(1, 48)) * 8
    N = int(rng.integers(1, 48)) * 8
    S = int(rng.integers(1, 13))
    seg_lens = [int(rng.integers(0, 7)) * 64 for _ in range(S)]
    if sum(seg_lens) == 0:
        seg_lens[0] = 64
    T = int(rng.integers(1, min(S, 6) + 1))
    ranks = [int(rng.choice([0, 1, 4, 8, 16, 17, 32, 48, 64])) for _ in range(T)]
    if max(ranks) == 0:
        ranks[0] = 8
    seg_task = [int(rng.integers(0, T)) for _ in range(S)]
    variant = "int" if case % 2 else "normal"
    scales = [float(rng.choice([1.0, 2.0])) for _ in range(T)] if variant == "int" else \
        [float(rng.uniform(0.25, 4.0)) for _ in range(T)]
    prob = Problem(K, N, seg_lens, ranks, seg_task=seg_task, scales=scales, variant=variant, seed=3000 + case)
    errs = compare(prob, prob.run_gpu(), prob.run_oracle(), exact=(variant == "int"))
    assert max(errs.values()) <= TOL, errs


def test_debug_build_traps_on_bad_segment_offsets():
    """A -DMUX_DEBUG_CHECKS build checks the device-side preconditions the host cannot see
    (seg_off non-decreasing multiples of 64 <= max_rows) and traps; a valid call passes."""
    import subprocess
    import sys
    import os
    from paper_2603_02885_b200 import build as mbuild
    lib = mbuild.build(defines=("MUX_DEBUG_CHECKS",), out="libmux_debug.so")
    code = f"""
import torch, sys
sys.path.insert(0, {os.path.dirname(os.path.dirname(os.path.abspath(__file__)))!r})
from paper_2603_02885_b200 import mux
mux.LIB_PATH = {lib!r}
mux._lib = None
X = torch.randn(256, 64, device='cuda').bfloat16()
W = torch.randn(64, 64, device='cuda').bfloat16()
ads = [mux.Adapter(None, None, 0, 0.0), mux.Adapter(None, None, 0, 0.0)]
mux.linear_fwd(torch.tensor([0, 128, 256], dtype=torch.int32, device='cuda'), [0, 1], ads, X, W, 16)
torch.cuda.synchronize()
print('valid ok', flush=True)
mux.linear_fwd(torch.tensor([0, 100, 256], dtype=torch.int32, device='cuda'), [0, 1], ads, X, W, 16)
torch.cuda.synchronize()
print('not trapped', flush=True)
"""
    r = subprocess.run([sys.executable, "-c", code], capture_output=True, text=True, timeout=300)
    out = r.stdout + r.stderr
    assert "valid ok" in out, out
    assert "not trapped" not in out and r.returncode != 0, out
    assert "bad seg_off[1] = 100" in out, out


def test_maximum_segments_and_adapters():
    """The ABI's maxima: 64 segments (MUX_MAX_SEGMENTS) over 64 adapters (MUX_MAX_ADAPTERS), ranks
    cycling 1..64 (r_cap 64), some segments empty, several 64-row segments per 256-row pair tile;
    integer inputs, so Y, dX, Hs and every dA_t / dB_t must be bit-exact."""
    rng = np.random.default_rng(77)
    seg_lens = [int(rng.choice([0, 64, 64, 128])) for _ in range(64)]
    ranks = [1 + (t * 7) % 64 for t in range(64)]
    scales = [1.0 if t % 2 else 2.0 for t in range(64)]
    p = Problem(256, 192, seg_lens, ranks, seg_task=list(range(64)), scales=scales, variant="int", seed=78)
    _run(p, exact=True)


def test_all_segments_empty():
    """Degenerate call: every segment empty (seg_off[S] = 0).  Nothing is computed, no row is
    written, and every adapter's dA/dB is written as exact zeros (Q16)."""
    from paper_2603_02885_b200 import mux
    K, N, R = 256, 192, 128
    seg_off = torch.zeros(3, dtype=torch.int32, device="cuda")
    X = torch.randn(R, K, device="cuda").bfloat16()
    W = torch.randn(N, K, device="cuda").bfloat16()
    dY = torch.randn(R, N, device="cuda").bfloat16()
    ads = []
    for r in (8, 16):
        B = mux.make_B_storage(N, r)
        B.copy_(torch.randn(N, r, device="cuda").bfloat16())
        ads.append(mux.Adapter(torch.randn(r, K, device="cuda").bfloat16(), B, r, 2.0,
                               torch.full((r, K), 7.0, device="cuda"), torch.full((N, r), 7.0, device="cuda")))
    Y = torch.full((R, N), 3.0, device="cuda").bfloat16()
    Y, Hs = mux.linear_fwd(seg_off, [0, 1], ads, X, W, 16, Y=Y)
    dX = torch.full((R, K), 5.0, device="cuda").bfloat16()
    mux.linear_bwd(seg_off, [0, 1], ads, dY, X, W, Hs, 16, dX=dX)
    torch.cuda.synchronize()
    assert torch.all(Y == 3.0) and torch.all(dX == 5.0)
    for a in ads:
        assert torch.all(a.dA == 0) and torch.all(a.dB == 0)


def test_shrink_and_fwd_with_given_hs_bit_identical():
    """mux_linear_shrink over the whole range and over 256-row sub-ranges reproduces mux_linear_fwd's
    Hs bit for bit (rows outside a sub-range untouched), and mux_linear_fwd_hs fed that Hs
    reproduces Y bit for bit (the tensor-parallel shared-shrink path)."""
    from paper_2603_02885_b200 import mux
    from gpu_harness import to_dev_bf16
    p = Problem(320, 640, [192, 64, 256, 128, 128], [16, 4, 64, 8, 0], seg_task=[0, 1, 2, 3, 4], seed=91,
                r_cap=64, max_rows=1024)
    seg_off = torch.from_numpy(p.seg_off).cuda()
    X, W = to_dev_bf16(p.X), to_dev_bf16(p.W)
    ads = p.gpu_adapters()
    Y, Hs = mux.linear_fwd(seg_off, p.seg_task, ads, X, W, p.r_cap)
    Hs_full = mux.linear_shrink(seg_off, p.seg_task, ads, X, p.N, p.r_cap)
    Y2 = mux.linear_fwd_hs(seg_off, p.seg_task, ads, X, W, Hs, p.r_cap)
    torch.cuda.synchronize()
    R = p.R
    assert torch.equal(Hs_full[:R].view(torch.int16), Hs[:R].view(torch.int16))
    assert torch.equal(Y2[:R].view(torch.int16), Y[:R].view(torch.int16))
    for lo, hi in ((0, 256), (256, 512), (512, 1024), (256, 1024)):
        part = torch.full((p.max_rows, p.r_cap), float("nan"), device="cuda").bfloat16()
        mux.linear_shrink(seg_off, p.seg_task, ads, X, p.N, p.r_cap, lo, hi, Hs=part)
        torch.cuda.synchronize()
        a, b = max(lo, 0), min(hi, R)
        if b > a:
            assert torch.equal(part[a:b].view(torch.int16), Hs[a:b].view(torch.int16)), (lo, hi)
        outside = torch.cat([part[:lo], part[max(hi, lo):]])
        assert torch.isnan(outside.float()).all(), (lo, hi)
    with pytest.raises(mux.MuxError):
        mux.linear_shrink(seg_off, p.seg_task, ads, X, p.N, p.r_cap, 100, 356)


def test_more_row_blocks_than_the_group_table():
    """> 128 pair row blocks (64 segments, 36 608 rows): the GEMM computes the tile task groups on the
    fly instead of from its per-launch shared-memory table (gemm.cu kGroupTab); integer inputs
    bit-exact, 64-row-granular segments straddling tiles across the whole range, 16 tasks."""
    segs = [64 * (5 + (i * 5) % 9) for i in range(64)]
    ranks = [(4, 8, 16, 32)[t % 4] for t in range(16)]
    p = Problem(128, 128, segs, ranks, variant="int", seg_task=[s % 16 for s in range(64)], seed=31)
    assert p.R > 128 * 256
    _run(p, exact=True)


def test_shrink_bwd_and_bwd_with_given_gs_bit_identical():
    """MUX_OP_SHRINK_BWD over the whole range, fed back as the given Gs of the backward (no shrink tiles;
    the row-parallel shared-shrink path, tp.py), reproduces mux_linear_bwd's dX, dA and dB bit for bit;
    over a 256-row sub-range it writes exactly those rows."""
    from paper_2603_02885_b200 import mux
    from gpu_harness import to_dev_bf16
    p = Problem(320, 640, [192, 64, 256, 128, 128], [16, 4, 64, 8, 0], seg_task=[0, 1, 2, 3, 4], seed=93,
                r_cap=64, max_rows=1024)
    seg_off = torch.from_numpy(p.seg_off).cuda()
    X, W, dY = to_dev_bf16(p.X), to_dev_bf16(p.W), to_dev_bf16(p.dY)
    ads = p.gpu_adapters()
    _, Hs = mux.linear_fwd(seg_off, p.seg_task, ads, X, W, p.r_cap)
    dX = mux.linear_bwd(seg_off, p.seg_task, ads, dY, X, W, Hs, p.r_cap)
    ref = {"dX": dX.clone(), "dA": [None if a.dA is None else a.dA.clone() for a in ads],
           "dB": [None if a.dB is None else a.dB.clone() for a in ads]}
    Gs = mux.linear_shrink_bwd(seg_off, p.seg_task, ads, dY, p.K, p.r_cap)
    dX2 = mux.linear_bwd_gs(seg_off, p.seg_task, ads, dY, X, W, Hs, Gs, p.r_cap)
    torch.cuda.synchronize()
    R = p.R
    assert torch.equal(dX2[:R].view(torch.int16), ref["dX"][:R].view(torch.int16))
    for t, a in enumerate(ads):
        if a.rank:
            assert torch.equal(a.dA, ref["dA"][t]) and torch.equal(a.dB, ref["dB"][t]), t
    part = torch.full((p.max_rows, p.r_cap), float("nan"), device="cuda").bfloat16()
    mux.linear_shrink_bwd(seg_off, p.seg_task, ads, dY, p.K, p.r_cap, 256, 512, Gs=part)
    torch.cuda.synchronize()
    assert torch.equal(part[256:512].view(torch.int16), Gs[256:512].view(torch.int16))
    assert torch.isnan(torch.cat([part[:256], part[512:]]).float()).all()
