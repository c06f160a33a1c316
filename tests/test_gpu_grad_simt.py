"""GPU parity of the CUDA-core adapter-gradient kernel (csrc/grad_simt.cu).

The default build routes dA/dB to the tcgen05 kernel (grad.cu) unless every
rank is <= MUX_GRAD_SIMT_MAX_RANK; a variant build with the threshold at 64
routes every call to the CUDA-core kernel, so the same problems exercise all of
its (columns x ranks x token-group) layouts: ranks 1..64 (including
non-multiples of 4 and 16), empty segments, a task owning two segments, ragged
K/N tails, integer inputs (bit-exact: every fp32 partial sum is an integer
below 2^24) and the fp64 oracle at the north_star tolerance.
"""
import contextlib

import numpy as np
import pytest

pytestmark = pytest.mark.gpu

torch = pytest.importorskip("torch")
if not torch.cuda.is_available():
    pytest.skip("needs a CUDA device", allow_module_level=True)

from gpu_harness import Problem, compare, TOL  # noqa: E402


@contextlib.contextmanager
def simt_lib():
    from paper_2603_02885_b200 import build as mbuild, mux
    path = mbuild.build(defines=("MUX_GRAD_SIMT_MAX_RANK=64",), out="libmux_gsimt.so")
    saved = (mux.LIB_PATH, mux._lib)
    mux.LIB_PATH, mux._lib = path, None
    try:
        yield mux
    finally:
        mux.LIB_PATH, mux._lib = saved


CASES = [
    dict(K=256, N=256, seg_lens=[64, 64], ranks=[4, 4]),
    dict(K=320, N=640, seg_lens=[192, 64, 256], ranks=[8, 4, 8]),
    dict(K=512, N=384, seg_lens=[128, 64, 192], ranks=[16, 12, 1]),
    dict(K=264, N=200, seg_lens=[64, 128], ranks=[32, 17]),
    dict(K=384, N=512, seg_lens=[128, 0, 64, 128], ranks=[64, 48], seg_task=[0, 1, 1, 0]),
]


@pytest.mark.parametrize("variant", ["normal", "int"])
@pytest.mark.parametrize("case", range(len(CASES)))
def test_simt_grads_vs_oracle(case, variant):
    c = dict(CASES[case])
    ranks = c.pop("ranks")
    scales = [1.0 if t % 2 else 2.0 for t in range(len(ranks))]
    prob = Problem(c["K"], c["N"], c["seg_lens"], ranks, seg_task=c.get("seg_task"), scales=scales,
                   variant=variant, seed=4100 + case)
    ref = prob.run_oracle()
    with simt_lib():
        gpu = prob.run_gpu()
    errs = compare(prob, gpu, ref, exact=(variant == "int"))
    assert max(errs.values()) <= TOL, errs


def test_simt_matches_tensor_core_kernel():
    """Same problem through both kernels: the fp32 gradients agree to fp32 summation-order noise."""
    prob = Problem(1024, 768, [256, 192, 320], [4, 8, 16], seed=4200)
    tc = prob.run_gpu()
    with simt_lib():
        si = prob.run_gpu()
    for t in range(3):
        for name in ("dA", "dB"):
            a, b = tc[name][t].astype(np.float64), si[name][t].astype(np.float64)
            assert np.max(np.abs(a - b)) <= 1e-5 * np.max(np.abs(a)), (name, t)
