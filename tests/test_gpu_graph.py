"""The whole hot path (pack -> Dispatch -> fused fwd -> bwd) is enqueue-only
(no host reads of device data), so it can be captured in a CUDA graph and
replayed; replays reuse the same workspaces (epoch-tagged flags) and must
reproduce the eager results bit for bit, also after the inputs change in
place between replays."""
import numpy as np
import pytest

pytestmark = pytest.mark.gpu

torch = pytest.importorskip("torch")
if not torch.cuda.is_available():
    pytest.skip("needs a CUDA device", allow_module_level=True)

from paper_2603_02885_b200 import mux  # noqa: E402


def _setup(seed):
    g = torch.Generator(device="cuda").manual_seed(seed)
    off = torch.tensor([0, 3, 5, 6], dtype=torch.int32, device="cuda")
    lens = torch.tensor([100, 40, 64, 130, 30, 77], dtype=torch.int32, device="cuda")
    T = int(lens.sum())
    K, N = 512, 768
    max_rows = mux.pack_bound_rows(T, 6, 64)
    pk = mux.alloc_pack_outputs(3, 6, max_rows, max_rows // 64)
    Xtok = torch.randn(T, K, device="cuda", generator=g).bfloat16()
    dYtok = torch.randn(T, N, device="cuda", generator=g).bfloat16()
    W = (torch.randn(N, K, device="cuda", generator=g) / K ** 0.5).bfloat16()
    ads = []
    for t, r in enumerate([16, 4, 48]):
        B = mux.make_B_storage(N, r)
        B.copy_(torch.randn(N, r, device="cuda", generator=g).bfloat16())
        ads.append(mux.Adapter((torch.randn(r, K, device="cuda", generator=g) / K ** 0.5).bfloat16(), B, r, 2.0,
                               torch.empty(r, K, device="cuda"), torch.empty(N, r, device="cuda")))
    bufs = {"X": torch.empty(max_rows, K, dtype=torch.bfloat16, device="cuda"),
            "dY": torch.empty(max_rows, N, dtype=torch.bfloat16, device="cuda"),
            "Y": torch.empty(max_rows, N, dtype=torch.bfloat16, device="cuda"),
            "Hs": torch.empty(max_rows, 48, dtype=torch.bfloat16, device="cuda"),
            "dX": torch.empty(max_rows, K, dtype=torch.bfloat16, device="cuda"),
            "ws": torch.zeros(mux.linear_workspace_size(3, max_rows, K, N, 48), dtype=torch.uint8, device="cuda")}
    return off, lens, pk, Xtok, dYtok, W, ads, bufs, max_rows


def _step(off, lens, pk, Xtok, dYtok, W, ads, b, max_rows):
    mux.pack_chunks(off, lens, None, 0, 64, max_rows=max_rows, max_chunks=max_rows // 64, out=pk)
    mux.pack_apply(pk["row_src"], Xtok, max_rows, out=b["X"])
    mux.pack_apply(pk["row_src"], dYtok, max_rows, out=b["dY"])
    mux.linear_fwd(pk["seg_off"], [0, 1, 2], ads, b["X"], W, 48, Y=b["Y"], Hs=b["Hs"], workspace=b["ws"])
    mux.linear_bwd(pk["seg_off"], [0, 1, 2], ads, b["dY"], b["X"], W, b["Hs"], 48, dX=b["dX"], workspace=b["ws"])


def _snapshot(b, ads, R):
    return ([b[k][:R].clone() for k in ("Y", "Hs", "dX")] + [a.dA.clone() for a in ads] +
            [a.dB.clone() for a in ads])


def test_graph_capture_and_replay_bitexact():
    off, lens, pk, Xtok, dYtok, W, ads, b, max_rows = _setup(5)
    R = mux.read_info(mux.pack_chunks(off, lens, None, 0, 64, max_rows=max_rows,
                                      max_chunks=max_rows // 64)["info"])["total_rows"]
    s = torch.cuda.Stream()
    s.wait_stream(torch.cuda.current_stream())
    with torch.cuda.stream(s):
        _step(off, lens, pk, Xtok, dYtok, W, ads, b, max_rows)
    torch.cuda.current_stream().wait_stream(s)
    torch.cuda.synchronize()
    eager = _snapshot(b, ads, R)

    graph = torch.cuda.CUDAGraph()
    with torch.cuda.graph(graph):
        _step(off, lens, pk, Xtok, dYtok, W, ads, b, max_rows)
    for _ in range(3):
        for k in ("Y", "Hs", "dX"):
            b[k].fill_(float("nan"))
        graph.replay()
        torch.cuda.synchronize()
        got = _snapshot(b, ads, R)
        for e, g_ in zip(eager, got):
            assert torch.equal(e.view(torch.int16) if e.dtype == torch.bfloat16 else e,
                               g_.view(torch.int16) if g_.dtype == torch.bfloat16 else g_)

    # new inputs written in place -> the replay computes the new result (eager on a fresh workspace agrees)
    Xtok.mul_(-0.5)
    graph.replay()
    torch.cuda.synchronize()
    got = _snapshot(b, ads, R)
    b2 = dict(b)
    b2["ws"] = torch.zeros_like(b["ws"])
    _step(off, lens, pk, Xtok, dYtok, W, ads, b2, max_rows)
    torch.cuda.synchronize()
    ref = _snapshot(b2, ads, R)
    for e, g_ in zip(ref, got):
        assert torch.equal(e.view(torch.int16) if e.dtype == torch.bfloat16 else e,
                           g_.view(torch.int16) if g_.dtype == torch.bfloat16 else g_)
    assert not torch.equal(got[0], eager[0])
