"""MuxLoRALinear (autograd glue) == direct binding calls, bit for bit: the
forward output, dX and every adapter's dA/dB (cast to the parameter dtype) —
and an optimizer step updates the padded B storage in place."""
import pytest

pytestmark = pytest.mark.gpu

torch = pytest.importorskip("torch")
if not torch.cuda.is_available():
    pytest.skip("needs a CUDA device", allow_module_level=True)

from paper_2603_02885_b200 import mux, MuxLoRALinear  # noqa: E402


def test_autograd_matches_binding():
    torch.manual_seed(0)
    R, K, N = 384, 256, 320
    W = (torch.randn(N, K, device="cuda") / K ** 0.5).bfloat16()
    lin = MuxLoRALinear(W, ranks=[16, 4, 32], scales=[2.0, 1.0, 0.5], init_B_zero=False)
    seg_off = torch.tensor([0, 128, 192, 384], dtype=torch.int32, device="cuda")
    st = [0, 1, 2]
    X = torch.randn(R, K, device="cuda").bfloat16().requires_grad_(True)
    G = torch.randn(R, N, device="cuda").bfloat16()
    Y = lin(X, seg_off, st)
    Y.backward(G)
    torch.cuda.synchronize()

    ads = [mux.Adapter(lin.A[t].data, lin.B[t].data, r, lin.scales[t]) for t, r in enumerate(lin.ranks)]
    Y2, Hs2 = mux.linear_fwd(seg_off, st, ads, X.detach(), W, lin.r_cap)
    dX2 = mux.linear_bwd(seg_off, st, ads, G, X.detach(), W, Hs2, lin.r_cap)
    torch.cuda.synchronize()
    assert torch.equal(Y.view(torch.int16), Y2.view(torch.int16))
    assert torch.equal(X.grad.view(torch.int16), dX2.view(torch.int16))
    for t in range(3):
        assert torch.equal(lin.A[t].grad, ads[t].dA.to(torch.bfloat16))
        assert torch.equal(lin.B[t].grad, ads[t].dB.to(torch.bfloat16))
    # an optimizer step writes through the [N, r] view into the padded storage
    opt = torch.optim.SGD(lin.parameters(), lr=0.1)
    before = lin.B[1].detach().clone()
    opt.step()
    assert lin.B[1].stride(0) == 8 and not torch.equal(lin.B[1].detach(), before)
    Y3 = lin(X, seg_off, st)
    assert not torch.equal(Y3.view(torch.int16), Y.view(torch.int16))


def test_call_from_fresh_thread():
    """The ABI encodes TMA descriptors with a driver call; a thread that has
    made no CUDA runtime call yet (PyTorch's autograd worker is one) must work."""
    import threading
    torch.manual_seed(1)
    R, K, N = 256, 128, 192
    W = (torch.randn(N, K, device="cuda") / K ** 0.5).bfloat16()
    X = torch.randn(R, K, device="cuda").bfloat16()
    seg_off = torch.tensor([0, 256], dtype=torch.int32, device="cuda")
    B = mux.make_B_storage(N, 8)
    B.copy_(torch.randn(N, 8, device="cuda").bfloat16())
    ads = [mux.Adapter((torch.randn(8, K, device="cuda") / K ** 0.5).bfloat16(), B, 8, 2.0)]
    ref, _ = mux.linear_fwd(seg_off, [0], ads, X, W, 16)
    out = {}

    def run():
        Y = torch.empty_like(ref)   # a fresh output buffer: its descriptor is not cached yet
        out["Y"], _ = mux.linear_fwd(seg_off, [0], ads, X, W, 16, Y=Y)
        torch.cuda.synchronize()

    th = threading.Thread(target=run)
    th.start()
    th.join()
    torch.cuda.synchronize()
    assert torch.equal(out["Y"].view(torch.int16), ref.view(torch.int16))
