"""GPU parity of the carrier shrink (gemm.cu tile_at_carry): the shrink
Hs = s_t X A_t^T (bwd: Gs = s_t dY B_t) computed on the first main tiles of each row block
from the same staged A tiles, instead of side tiles that re-read X / dY.  Every case runs the
fused forward + backward twice — carriers (MUX_CARRY=2: also at these short reductions, where
the default keeps side tiles) and side tiles (MUX_CARRY=0) — against the fp64 oracle: integer inputs bit-exact, and both schedules must
give the same bits (the main product and each shrink element accumulate in the same order).
Covers one carrier per row block (2 task groups at r_cap 16), several carriers in one wave
(4 groups of 64-row segments, r_cap 32), the device-side fallback to side tiles when several
carriers per row block would not fit one wave, rank-0 and rank < r_cap adapters."""
import os

import numpy as np
import pytest

pytestmark = pytest.mark.gpu

torch = pytest.importorskip("torch")
if not torch.cuda.is_available():
    pytest.skip("needs a CUDA device", allow_module_level=True)

from gpu_harness import Problem, bf16_to_f64, compare  # noqa: E402


def _run_env(p, carry):
    old = os.environ.get("MUX_CARRY")
    os.environ["MUX_CARRY"] = carry
    try:
        return p.run_gpu()
    finally:
        if old is None:
            del os.environ["MUX_CARRY"]
        else:
            os.environ["MUX_CARRY"] = old


def _both(p, exact, rows=None, carry="2"):
    # MUX_CARRY=2: carriers also at reductions <= 2048, where the default keeps side tiles
    # (3: and one carrier per row block even when the carriers span several waves)
    g1 = _run_env(p, carry)
    g0 = _run_env(p, "0")
    ref = p.run_oracle(rows=rows)
    e1 = compare(p, g1, ref, rows=rows, exact=exact)
    compare(p, g0, ref, rows=rows, exact=exact)
    for k in ("Y", "Hs", "dX"):
        assert np.array_equal(g1[k], g0[k]), f"{k}: carrier and side-tile schedules differ"
    for t, r in enumerate(p.ranks):
        if r:
            assert np.array_equal(g1["dA"][t], g0["dA"][t]) and np.array_equal(g1["dB"][t], g0["dB"][t]), t
    return e1


def test_one_carrier_per_row_block_int():
    """4 tasks rank 16 (config-2 structure at K = N = 1024): row blocks hold <= 2 task groups, one
    carrier each (r_cap 16 stacks two groups); fwd and bwd (dX: 4 column tiles)."""
    p = Problem(1024, 1024, [448, 320, 1216, 576], [16, 16, 16, 16], variant="int", seed=301)
    _both(p, exact=True)


def test_four_groups_several_carriers_one_wave_int():
    """64-row segments: every row block holds 4 task groups; r_cap 32 (ranks 4/8/32/16, a rank-4
    adapter's second 8-row slab is all zero fill) -> 4 carriers per row block, all in one wave."""
    segs = [64] * 24
    p = Problem(1024, 1280, segs, [4, 8, 32, 16], seg_task=[s % 4 for s in range(24)], variant="int",
                scales=[1.0, 2.0, 0.5, 1.0], seed=302)
    _both(p, exact=True)


def test_two_carriers_r16_with_rank0_int():
    """r_cap 16 with up to 4 groups per row block -> 2 carriers; a rank-0 task's rows get Hs = 0
    from carrier 0 and never take part in a shrink MMA."""
    segs = [64, 64, 64, 64, 64, 64, 128, 192, 64, 256]
    p = Problem(768, 1024, segs, [16, 0, 8, 16, 4], seg_task=[0, 2, 3, 4, 1, 0, 2, 3, 1, 4], variant="int",
                seed=303)
    _both(p, exact=True)


def test_fallback_to_side_tiles_int():
    """A row block with 4 groups at r_cap 32 (4 carriers) and 31 row blocks: 124 carriers do not fit
    one wave of CTA pairs, so the launch runs side tiles (same results)."""
    segs = [64, 64, 64, 64] + [128] * 60
    p = Problem(1024, 1024, segs, [32, 16, 8, 4], seg_task=[s % 4 for s in range(64)], variant="int",
                seed=304)
    _both(p, exact=True)


def test_normal_values_config2_like():
    """Floating-point inputs, 4 tasks rank 16, 4096 x 4096, 3 072 rows: sampled rows of Y / dX and all
    of Hs, dA, dB within the north_star tolerance; carrier and side-tile schedules bit-identical."""
    p = Problem(4096, 4096, [768, 704, 896, 704], [16, 16, 16, 16], seed=305)
    rng = np.random.default_rng(3)
    rows = np.unique(np.concatenate([np.arange(0, 32), np.arange(p.R - 32, p.R),
                                     rng.integers(0, p.R, size=96)])).astype(np.int64)
    errs = _both(p, exact=False, rows=rows)
    print(errs)


def test_fallback_more_row_blocks_than_pairs():
    """One carrier per row block but 76 row blocks on 74 CTA pairs: a carrier would be some cluster's
    second item (it would wait for the previous tile's epilogue), so the launch runs side tiles.
    Sampled rows of Y / dX, all of Hs / dA / dB; both schedules bit-identical."""
    p = Problem(1024, 1024, [4864, 4864, 4864, 4864], [16, 16, 8, 16], seed=306)
    rng = np.random.default_rng(4)
    rows = np.unique(np.concatenate([np.arange(0, 16), np.arange(p.R - 16, p.R),
                                     rng.integers(0, p.R, size=64)])).astype(np.int64)
    _both(p, exact=False, rows=rows)


def test_one_carrier_spanning_waves():
    """MUX_CARRY=3: one carrier per row block with 76 row blocks on 74 CTA pairs (some carriers are
    their cluster's second item and first wait for the previous tile's epilogue to drain the other
    accumulator); integer inputs bit-exact and bit-identical to side tiles."""
    p = Problem(1024, 2048, [4864, 4864, 4864, 4864], [16, 16, 8, 16], variant="int", seed=307)
    rng = np.random.default_rng(5)
    rows = np.unique(np.concatenate([np.arange(0, 16), np.arange(p.R - 16, p.R),
                                     rng.integers(0, p.R, size=64)])).astype(np.int64)
    _both(p, exact=True, rows=rows, carry="3")


def test_nan_isolation_with_carriers():
    """P:500 with the stacked shrink: a carrier's N = 32 MMA multiplies every row of its row block by
    every carried group's adapter rows (the other groups' columns are discarded per row), so NaN in
    task 1's X rows and in task 2's A / B must still never reach task 0 (3 groups in row block 0 ->
    2 carriers at r_cap 16), forward and backward, and both schedules must agree bit for bit."""
    p = Problem(1024, 1024, [64, 64, 128, 256, 512], [8, 16, 8], seg_task=[0, 1, 2, 0, 1], seed=308)
    p.X[70, 5] = np.uint16(0x7FC0)       # task 1's row, in row block 0 with tasks 0 and 2
    p.A[2][1, 7] = np.uint16(0x7FC0)     # task 2's A: its stacked shrink columns become NaN
    p.B[2][3, 2] = np.uint16(0x7FC0)     # task 2's B: its Gs and expand
    outs = [_run_env(p, c) for c in ("2", "0")]
    for g in outs:
        Y, Hs, dX = (bf16_to_f64(g[k]) for k in ("Y", "Hs", "dX"))
        t0 = np.r_[0:64, 256:512]        # task 0's rows (segments 0 and 3)
        assert np.all(np.isfinite(Y[t0])) and np.all(np.isfinite(Hs[t0])) and np.all(np.isfinite(dX[t0]))
        assert np.all(np.isfinite(g["dA"][0])) and np.all(np.isfinite(g["dB"][0]))
        assert np.isnan(Y[70]).any() and np.isnan(Y[128:256]).any()
    for k in ("Y", "Hs", "dX"):  # same values (NaN payloads may differ)
        assert np.array_equal(bf16_to_f64(outs[0][k]), bf16_to_f64(outs[1][k]), equal_nan=True), k


def test_workspace_shared_across_row_counts():
    """One workspace shared by calls with different max_rows (the contract allows it): small calls'
    Gs / Hs scratch must never land on a larger call's row-block flags (with a flag region sized by
    max_rows it did, and the 16-task call below waited on garbage counters until the watchdog
    trapped).  Results equal those with a fresh workspace, bit for bit."""
    from paper_2603_02885_b200 import mux
    g = torch.Generator(device="cuda").manual_seed(9)
    K = N = 4096
    per, m = 1024, 16
    W = (torch.randn(N, K, device="cuda", generator=g) / K ** 0.5).bfloat16()
    ads = []
    for _ in range(m):
        B = mux.make_B_storage(N, 16)
        B.copy_(torch.randn(N, 16, device="cuda", generator=g).bfloat16())
        ads.append(mux.Adapter((torch.randn(16, K, device="cuda", generator=g) / K ** 0.5).bfloat16(), B, 16, 2.0))
    X = torch.randn(m * per, K, device="cuda", generator=g).bfloat16()
    dY = torch.randn(m * per, N, device="cuda", generator=g).bfloat16()
    ws = torch.zeros(mux.linear_workspace_size(m, m * per, K, N, 16), dtype=torch.uint8, device="cuda")

    def call(rows, tasks, workspace):
        so = torch.tensor([i * per for i in range(tasks + 1)], dtype=torch.int32, device="cuda")
        Y, Hs = mux.linear_fwd(so, list(range(tasks)), ads[:tasks], X[:rows], W, 16, workspace=workspace)
        dX = mux.linear_bwd(so, list(range(tasks)), ads[:tasks], dY[:rows], X[:rows], W, Hs, 16, workspace=workspace)
        torch.cuda.synchronize()
        return Y.clone(), Hs.clone(), dX.clone()

    for rows, tasks in ((per, 1), (2 * per, 2), (m * per, m), (per, 1), (m * per, m)):
        got = call(rows, tasks, ws)
        fresh = call(rows, tasks, torch.zeros_like(ws))
        for a, b in zip(got, fresh):
            assert torch.equal(a.view(torch.int16), b.view(torch.int16)), (rows, tasks)


@pytest.mark.parametrize("seed", range(8))
def test_carrier_fuzz_int(seed):
    """Random problems (widths 768-2048, 1-8 tasks of ranks 0/4/8/16/32, 64-row-granular segments,
    several segments per task): integer inputs bit-exact vs the oracle under carriers (forced) and
    side tiles, both schedules bit-identical."""
    rng = np.random.default_rng(1000 + seed)
    K = int(rng.choice([768, 1024, 1280, 2048]))
    N = int(rng.choice([768, 1024, 1536, 2048]))
    T = int(rng.integers(1, 9))
    ranks = [int(r) for r in rng.choice([0, 4, 8, 16, 32], size=T)]
    if max(ranks) == 0:
        ranks[0] = 16
    S = int(rng.integers(T, min(2 * T, 12) + 1))
    segs = [64 * int(x) for x in rng.integers(1, 9, size=S)]
    seg_task = [s % T for s in range(S)]
    rng.shuffle(seg_task)
    p = Problem(K, N, segs, ranks, seg_task=seg_task, variant="int", seed=2000 + seed)
    _both(p, exact=True)
