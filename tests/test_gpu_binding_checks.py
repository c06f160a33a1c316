"""The binding's host-side checks (mux.py _check_linear): everything the C ABI cannot see through
raw pointers — dtype, shape (W must be [N, K] with K = X's columns; adapters [r, K] / [N, r]),
contiguity, device — raises ValueError before any launch instead of reading out of bounds."""
import pytest

pytestmark = pytest.mark.gpu

torch = pytest.importorskip("torch")
if not torch.cuda.is_available():
    pytest.skip("needs a CUDA device", allow_module_level=True)

from paper_2603_02885_b200 import mux  # noqa: E402


def _setup(R=256, K=128, N=192, ranks=(16, 8)):
    g = torch.Generator(device="cuda").manual_seed(5)
    X = torch.randn(R, K, device="cuda", generator=g).bfloat16()
    W = torch.randn(N, K, device="cuda", generator=g).bfloat16()
    ads = []
    for r in ranks:
        B = mux.make_B_storage(N, r)
        B.copy_(torch.randn(N, r, device="cuda", generator=g).bfloat16())
        ads.append(mux.Adapter(torch.randn(r, K, device="cuda", generator=g).bfloat16(), B, r, 2.0))
    seg_off = torch.tensor([0, 128, R], dtype=torch.int32, device="cuda")
    return X, W, ads, seg_off


def test_valid_call_passes():
    X, W, ads, so = _setup()
    Y, Hs = mux.linear_fwd(so, [0, 1], ads, X, W, 16)
    dX = mux.linear_bwd(so, [0, 1], ads, torch.randn_like(Y), X, W, Hs, 16)
    torch.cuda.synchronize()
    assert Y.shape == (256, 192) and dX.shape == (256, 128)


@pytest.mark.parametrize("case", ["W_K", "W_T", "X_f32", "X_noncontig", "A_shape", "B_shape", "Y_shape",
                                  "Hs_rcap", "seg_off_len", "seg_off_dtype", "X_cpu"])
def test_fwd_mismatch_raises(case):
    X, W, ads, so = _setup()
    kw = {}
    st = [0, 1]
    if case == "W_K":
        W = torch.randn(192, 256, device="cuda").bfloat16()          # K = 256 != X's 128
    elif case == "W_T":
        W = W.t().contiguous()                                         # [K, N] instead of [N, K]
    elif case == "X_f32":
        X = X.float()
    elif case == "X_noncontig":
        X = torch.randn(256, 256, device="cuda").bfloat16()[:, :128]
    elif case == "A_shape":
        ads[0].A = torch.randn(16, 64, device="cuda").bfloat16()
    elif case == "B_shape":
        ads[1].B = torch.zeros(96, 8, device="cuda").bfloat16()
    elif case == "Y_shape":
        kw["Y"] = torch.empty(256, 128, dtype=torch.bfloat16, device="cuda")
    elif case == "Hs_rcap":
        kw["Hs"] = torch.empty(256, 32, dtype=torch.bfloat16, device="cuda")
    elif case == "seg_off_len":
        so = so[:2]
    elif case == "seg_off_dtype":
        so = so.long()
    elif case == "X_cpu":
        X = X.cpu()
    with pytest.raises(ValueError):
        mux.linear_fwd(so, st, ads, X, W, 16, **kw)


def test_bwd_mismatch_raises():
    X, W, ads, so = _setup()
    Y, Hs = mux.linear_fwd(so, [0, 1], ads, X, W, 16)
    with pytest.raises(ValueError):      # dY with K columns instead of N
        mux.linear_bwd(so, [0, 1], ads, torch.randn_like(X), X, W, Hs, 16)
    with pytest.raises(ValueError):      # fp32 gradient buffer of the wrong shape
        ads[0].dA = torch.empty(16, 64, device="cuda")
        mux.linear_bwd(so, [0, 1], ads, torch.randn_like(Y), X, W, Hs, 16)
    with pytest.raises(ValueError):      # W [K, N]
        ads[0].dA = None
        mux.linear_bwd(so, [0, 1], ads, torch.randn_like(Y), X, W.t().contiguous(), Hs, 16)
