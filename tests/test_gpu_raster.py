"""The fused GEMM's column-band raster (MUX_RASTER=n: bands of output-column blocks with the band's
W tiles L2-resident, each row block's shrink tile right before its main tiles in the first band)
computes exactly what the row-band raster does: on integer inputs every output is bit-exact
against the fp64 oracle under both rasters, over shapes whose column-block count is and is not a
multiple of the band, forward and backward (dX, Gs, dA, dB)."""
import os

import pytest

pytestmark = pytest.mark.gpu

torch = pytest.importorskip("torch")
if not torch.cuda.is_available():
    pytest.skip("needs a CUDA device", allow_module_level=True)

from gpu_harness import Problem, compare  # noqa: E402


@pytest.fixture
def raster():
    old = os.environ.get("MUX_RASTER")

    def set_(m):
        os.environ["MUX_RASTER"] = m
    yield set_
    if old is None:
        os.environ.pop("MUX_RASTER", None)
    else:
        os.environ["MUX_RASTER"] = old


@pytest.mark.parametrize("mode", ["m", "n", "a"])
@pytest.mark.parametrize("K,N,segs", [
    (2048, 1536, [384, 640, 192, 320]),      # 6 column blocks: one band
    (24576, 2304, [256, 256, 128, 64]),      # long reduction: bands of 4 column blocks (9 = 4 + 4 + 1)
    (1024, 4096, [256, 1024, 704]),
])
def test_raster_integer_bit_exact(raster, mode, K, N, segs):
    raster(mode)
    p = Problem(K, N, segs, [16, 8, 32, 4][:len(segs)], variant="int", seed=K + N)
    compare(p, p.run_gpu(), p.run_oracle(), exact=True)
