"""GPU parity of fused projections with one adapter per column slice (include/mux.h "Fused
projections"; P:296 names attaching adapters to the fused qkv projection as the obstacle to running
per-projection LoRA on one fused backbone op).  The fused call (mux_linear, op FWD / BWD) is compared
element by element with the fp64 oracle's definition (oracle/linear.py linear_*_sliced: one
independent LoRA linear per slice).  Bars: north_star 2e-2 (max|gpu - oracle| / max|oracle| per
tensor); integer-valued inputs bit-exact; one slice = the plain entry points bit for bit."""
import numpy as np
import pytest

pytestmark = pytest.mark.gpu

torch = pytest.importorskip("torch")
if not torch.cuda.is_available():
    pytest.skip("needs a CUDA device", allow_module_level=True)

from synth import gen  # noqa: E402
from oracle import linear as olin  # noqa: E402
from paper_2603_02885_b200 import mux  # noqa: E402
from gpu_harness import TOL, Problem, bf16_to_f64, from_dev_bf16, rel_err, to_dev_bf16  # noqa: E402


class SlicedProblem:
    def __init__(self, K, col_off, seg_lens, ranks, scales=None, seg_task=None, variant="normal", seed=5,
                 r_cap=None):
        self.K, self.col_off = K, list(col_off)
        self.N = col_off[-1]
        self.S = len(col_off) - 1
        self.seg_off = np.concatenate([[0], np.cumsum(seg_lens)]).astype(np.int32)
        self.R = int(self.seg_off[-1])
        self.max_rows = max(self.R, 1)
        self.T = len(ranks)
        self.seg_task = list(seg_task) if seg_task is not None else [s % self.T for s in range(len(seg_lens))]
        self.ranks = [list(r) for r in ranks]
        self.scales = scales or [[2.0 - 0.5 * (s % 2) for s in range(self.S)] for _ in range(self.T)]
        mr = max(max(r) for r in ranks)
        self.r_cap = r_cap or max(16, -(-mr // 16) * 16)
        st = gen.Stream(seed)
        ns = [col_off[s + 1] - col_off[s] for s in range(self.S)]
        if variant == "int":
            self.X = gen.int_bf16(seed, st.take(), (self.max_rows, K), -4, 4)
            self.W = gen.int_bf16(seed, st.take(), (self.N, K), -4, 4)
            self.dY = gen.int_bf16(seed, st.take(), (self.max_rows, self.N), -4, 4)
            self.A = [[gen.sparse_int_bf16(seed, st.take(), (r, K), 8, 1, -2, 2) for r in rt] for rt in ranks]
            self.B = [[gen.sparse_int_bf16(seed, st.take(), (ns[s], r), 8, 0, -2, 2) for s, r in enumerate(rt)]
                      for rt in ranks]
            self.scales = [[float(1 + (t + s) % 2) for s in range(self.S)] for t in range(self.T)]
        else:
            self.X = gen.normal_bf16(seed, st.take(), (self.max_rows, K), 1.0)
            self.W = gen.normal_bf16(seed, st.take(), (self.N, K), 1.0 / np.sqrt(K))
            self.dY = gen.normal_bf16(seed, st.take(), (self.max_rows, self.N), 1.0)
            self.A = [[gen.normal_bf16(seed, st.take(), (r, K), 1.0 / np.sqrt(K)) for r in rt] for rt in ranks]
            self.B = [[gen.normal_bf16(seed, st.take(), (ns[s], r), 1.0 / np.sqrt(max(r, 1)))
                       for s, r in enumerate(rt)] for rt in ranks]

    def adapters(self):
        ads = []
        for t in range(self.T):
            row = []
            for s in range(self.S):
                r = self.ranks[t][s]
                if r == 0:
                    row.append(mux.Adapter(None, None, 0, self.scales[t][s]))
                    continue
                B = mux.make_B_storage(self.col_off[s + 1] - self.col_off[s], r)
                B.copy_(to_dev_bf16(self.B[t][s]))
                row.append(mux.Adapter(to_dev_bf16(self.A[t][s]), B, r, self.scales[t][s]))
            ads.append(row)
        return ads

    def run_gpu(self):
        seg_off = torch.from_numpy(self.seg_off).cuda()
        X, W, dY = to_dev_bf16(self.X), to_dev_bf16(self.W), to_dev_bf16(self.dY)
        ads = self.adapters()
        Y, Hs = mux.linear_fwd_sliced(seg_off, self.seg_task, ads, X, W, self.col_off, self.r_cap)
        dX = mux.linear_bwd_sliced(seg_off, self.seg_task, ads, dY, X, W, Hs, self.col_off, self.r_cap)
        torch.cuda.synchronize()
        return {"Y": from_dev_bf16(Y)[:self.R], "Hs": from_dev_bf16(Hs)[:self.R], "dX": from_dev_bf16(dX)[:self.R],
                "dA": [[None if a.rank == 0 else a.dA.cpu().numpy() for a in row] for row in ads],
                "dB": [[None if a.rank == 0 else a.dB.cpu().numpy() for a in row] for row in ads]}

    def run_oracle(self):
        Y, Hs = olin.linear_fwd_sliced(self.seg_off, self.seg_task, self.col_off, self.A, self.B, self.ranks,
                                       self.scales, self.X, self.W, self.r_cap)
        dX, Gs, grads = olin.linear_bwd_sliced(self.seg_off, self.seg_task, self.col_off, self.A, self.B,
                                               self.ranks, self.scales, self.dY, self.X, self.W, self.r_cap)
        return {"Y": Y, "Hs": Hs, "dX": dX, "grads": grads}


def check(prob, exact=False, tol=TOL):
    g = prob.run_gpu()
    r = prob.run_oracle()
    errs = {}
    for name in ("Y", "Hs", "dX"):
        if exact:
            assert np.array_equal(g[name], gen.bf16_bits_from_f64(r[name])), f"{name}: not bit-exact"
        errs[name] = rel_err(bf16_to_f64(g[name]), r[name])
    for t in range(prob.T):
        for s in range(prob.S):
            if prob.ranks[t][s] == 0:
                continue
            dA, dB = r["grads"][t][s]
            if exact:
                assert np.array_equal(g["dA"][t][s].astype(np.float64), dA), f"dA[{t}][{s}] not exact"
                assert np.array_equal(g["dB"][t][s].astype(np.float64), dB), f"dB[{t}][{s}] not exact"
            errs[f"dA{t}.{s}"] = rel_err(g["dA"][t][s], dA)
            errs[f"dB{t}.{s}"] = rel_err(g["dB"][t][s], dB)
    bad = {k: v for k, v in errs.items() if not v <= tol}
    assert not bad, f"tolerance {tol} exceeded: {bad} (all {errs})"
    return errs


# q|k|v-like: three slices on 256-column tile boundaries except the middle one (a tile straddles
# slices 1 and 2), heterogeneous ranks incl. a rank-0 slice and a task without any adapter, segments
# that straddle 256-row tiles, a task owning two segments
QKV = dict(K=512, col_off=[0, 256, 384, 640], seg_lens=[192, 320, 128, 64, 256],
           ranks=[[16, 8, 0], [4, 32, 16], [0, 0, 0]])


def test_sliced_qkv_normal():
    check(SlicedProblem(**QKV))


def test_sliced_qkv_integer_bit_exact():
    check(SlicedProblem(**QKV, variant="int"), exact=True)


def test_sliced_tp8_gate_up_widths():
    """gate|up at an 8-way tensor-parallel shard of LLaMA-7B: 1376 = 11008 / 8 columns each, not a
    multiple of 64 (slice boundaries inside a 64-column box; B rows outside a slice are zero fill,
    including negative TMA coordinates)."""
    p = SlicedProblem(K=256, col_off=[0, 1376, 2752], seg_lens=[128, 192, 64], ranks=[[16, 8], [8, 16]],
                      variant="int", seed=9)
    check(p, exact=True)


def test_sliced_four_slices_max_slots():
    """MUX_MAX_SLICES slices and 24 tasks x 4 = 96 adapter slots (the parameter-block limit)."""
    T = 24
    ranks = [[(4, 8, 16, 0)[(t + s) % 4] for s in range(4)] for t in range(T)]
    p = SlicedProblem(K=256, col_off=[0, 64, 192, 200, 328], seg_lens=[64] * T, ranks=ranks, seed=13)
    check(p)


def test_sliced_one_slice_equals_plain_call():
    """num_slices = 1 through mux_linear is the plain entry points bit for bit."""
    prob = Problem(512, 384, [128, 256, 64], [16, 8, 32], seed=21)
    ref = prob.run_gpu()
    seg_off = torch.from_numpy(prob.seg_off).cuda()
    X, W, dY = to_dev_bf16(prob.X), to_dev_bf16(prob.W), to_dev_bf16(prob.dY)
    ads = [[a] for a in prob.gpu_adapters()]
    Y, Hs = mux.linear_fwd_sliced(seg_off, prob.seg_task, ads, X, W, [0, prob.N], prob.r_cap)
    dX = mux.linear_bwd_sliced(seg_off, prob.seg_task, ads, dY, X, W, Hs, [0, prob.N], prob.r_cap)
    torch.cuda.synchronize()
    assert np.array_equal(from_dev_bf16(Y)[:prob.R], ref["Y"])
    assert np.array_equal(from_dev_bf16(Hs)[:prob.R], ref["Hs"])
    assert np.array_equal(from_dev_bf16(dX)[:prob.R], ref["dX"])
    for t, row in enumerate(ads):
        assert np.array_equal(row[0].dA.cpu().numpy(), ref["dA"][t])
        assert np.array_equal(row[0].dB.cpu().numpy(), ref["dB"][t])


def test_sliced_llama7b_qkv_full_size_sampled():
    """The fused q|k|v shape of SURVEY 8(a) a5 (4096 -> 3 x 4096), 4 tasks (config 2 ranks 16, one
    task with mixed ranks), ~2.3k rows: Y / dX on sampled rows, Hs / dA / dB on all rows."""
    K = 4096
    col_off = [0, 4096, 8192, 12288]
    ranks = [[16, 16, 16], [16, 16, 16], [8, 64, 32], [16, 0, 16]]
    p = SlicedProblem(K=K, col_off=col_off, seg_lens=[576, 640, 512, 576], ranks=ranks, seed=17, r_cap=64)
    seg_off = torch.from_numpy(p.seg_off).cuda()
    X, W, dY = to_dev_bf16(p.X), to_dev_bf16(p.W), to_dev_bf16(p.dY)
    ads = p.adapters()
    Y, Hs = mux.linear_fwd_sliced(seg_off, p.seg_task, ads, X, W, col_off, p.r_cap)
    dX = mux.linear_bwd_sliced(seg_off, p.seg_task, ads, dY, X, W, Hs, col_off, p.r_cap)
    torch.cuda.synchronize()
    rows = np.unique(np.concatenate([np.arange(0, p.R, 97), p.seg_off[1:-1] - 1, p.seg_off[:-1]]))
    Yo, Hso = olin.linear_fwd_sliced(p.seg_off, p.seg_task, col_off, p.A, p.B, p.ranks, p.scales, p.X, p.W,
                                     p.r_cap, rows=rows)
    dXo, _, grads = olin.linear_bwd_sliced(p.seg_off, p.seg_task, col_off, p.A, p.B, p.ranks, p.scales, p.dY,
                                           p.X, p.W, p.r_cap, rows=rows)
    errs = {"Y": rel_err(bf16_to_f64(from_dev_bf16(Y)[rows]), Yo),
            "Hs": rel_err(bf16_to_f64(from_dev_bf16(Hs)[:p.R]), Hso),
            "dX": rel_err(bf16_to_f64(from_dev_bf16(dX)[rows]), dXo)}
    for t in range(p.T):
        for s in range(3):
            if p.ranks[t][s]:
                errs[f"dA{t}.{s}"] = rel_err(ads[t][s].dA.cpu().numpy(), grads[t][s][0])
                errs[f"dB{t}.{s}"] = rel_err(ads[t][s].dB.cpu().numpy(), grads[t][s][1])
    assert max(errs.values()) <= TOL, errs


def test_sliced_nan_stays_in_its_task():
    """A NaN in one task's slice-1 A never reaches another task's rows."""
    p = SlicedProblem(**QKV, seed=3)
    bad = np.array(p.A[1][1])
    bad[0, 3] = 0x7FC0  # bf16 NaN bits
    p.A[1][1] = bad
    g = p.run_gpu()
    Y = bf16_to_f64(g["Y"])
    dX = bf16_to_f64(g["dX"])
    for s, t in enumerate(p.seg_task):
        rows = slice(p.seg_off[s], p.seg_off[s + 1])
        if t != 1:
            assert np.isfinite(Y[rows]).all() and np.isfinite(dX[rows]).all(), f"segment {s} (task {t})"
    for t in (0,):
        for s in range(3):
            if p.ranks[t][s]:
                assert np.isfinite(g["dA"][t][s]).all() and np.isfinite(g["dB"][t][s]).all()


@pytest.mark.parametrize("case", range(12))
def test_sliced_fuzz_integer_bit_exact(case):
    """Random fused projections: 1-4 slices of random widths (multiples of 8, some below one 64-column
    box), 1-6 tasks with random ranks per slice (0 allowed), random 64-row segments (a task may own
    several), K a multiple of 8; integer inputs, every output bit-exact against the oracle."""
    rng = np.random.default_rng(4000 + case)
    S = int(rng.integers(1, 5))
    widths = [int(8 * rng.integers(1, 48)) for _ in range(S)]
    col_off = [0]
    for w in widths:
        col_off.append(col_off[-1] + w)
    T = int(rng.integers(1, 7))
    ranks = [[int(rng.choice([0, 4, 8, 16, 24, 32, 48, 64])) for _ in range(S)] for _ in range(T)]
    if all(r == 0 for row in ranks for r in row):
        ranks[0][0] = 16
    nseg = int(rng.integers(1, 9))
    seg_lens = [64 * int(rng.integers(0, 6)) for _ in range(nseg)]
    if sum(seg_lens) == 0:
        seg_lens[0] = 64
    seg_task = [int(rng.integers(0, T)) for _ in range(nseg)]
    K = int(8 * rng.integers(2, 80))
    p = SlicedProblem(K=K, col_off=col_off, seg_lens=seg_lens, ranks=ranks, seg_task=seg_task, variant="int",
                      seed=5000 + case)
    check(p, exact=True)
