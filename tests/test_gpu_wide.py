"""The fused GEMM's wide pair tiles (gemm.cu kTileN = 512: one 512-column TMEM accumulator filled
by two N = 256 MMAs per k-step, each CTA staging 256 B rows; MUX_TILE_N=512 forces them) compute
exactly what the standard tiles do: integer inputs bit-exact against the fp64 oracle for forward
and backward (Y, Hs, dX, dA, dB) over ragged shapes (N not a multiple of 512, K not a multiple of
64), straddling tasks, heterogeneous ranks, and fused projections whose slices straddle the two MMA
halves; normal inputs within the north_star tolerance."""
import os

import pytest

pytestmark = pytest.mark.gpu

torch = pytest.importorskip("torch")
if not torch.cuda.is_available():
    pytest.skip("needs a CUDA device", allow_module_level=True)

from gpu_harness import TOL, Problem, compare  # noqa: E402


@pytest.fixture
def wide():
    old = os.environ.get("MUX_TILE_N")
    os.environ["MUX_TILE_N"] = "512"
    yield
    if old is None:
        os.environ.pop("MUX_TILE_N", None)
    else:
        os.environ["MUX_TILE_N"] = old


CASES = [
    # K, N, segment rows, ranks
    (512, 1024, [256, 512], [16, 8]),
    (1376, 1800, [128, 64, 320, 192], [16, 4, 48, 64]),   # N = 3.5 wide tiles, ragged K
    (2048, 768, [64, 192, 256], [32, 8, 16]),             # 1.5 wide tiles per row block
    (256, 4096, [704], [64]),
]


@pytest.mark.parametrize("case", range(len(CASES)))
def test_wide_integer_bit_exact(wide, case):
    K, N, segs, ranks = CASES[case]
    p = Problem(K, N, segs, ranks, variant="int", scales=[float(1 + t % 2) for t in range(len(ranks))],
                seed=1200 + case)
    compare(p, p.run_gpu(), p.run_oracle(), exact=True)


@pytest.mark.parametrize("case", range(len(CASES)))
def test_wide_normal_within_tolerance(wide, case):
    K, N, segs, ranks = CASES[case]
    p = Problem(K, N, segs, ranks, seed=1300 + case)
    errs = compare(p, p.run_gpu(), p.run_oracle())
    assert max(errs.values()) <= TOL, errs


def test_wide_sliced_integer_bit_exact(wide):
    """q|k|v-like slices of 320, 448 and 256 columns: slice boundaries inside both MMA halves."""
    from test_gpu_sliced import SlicedProblem, check
    p = SlicedProblem(K=512, col_off=[0, 320, 768, 1024], seg_lens=[192, 320, 128], ranks=[[16, 8, 0], [4, 32, 16]],
                      variant="int", seed=1400)
    check(p, exact=True)
