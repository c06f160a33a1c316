"""GPU parity of the decoder-block ops (NEXT-3) through the C ABI vs the fp64
oracle (oracle/block.py): row map (bit-exact), RMSNorm, SwiGLU, RoPE and
causal attention inside packed sequences (fwd + bwd, MHA and grouped KV).
Layouts come from the GPU pack kernel (checked bit-exact against the pack
oracle first); inputs are seeded bf16 from synth.gen.  Tolerance (north_star):
max|gpu - oracle| / max|oracle| <= 2e-2 per tensor."""
import numpy as np
import pytest

pytestmark = pytest.mark.gpu

torch = pytest.importorskip("torch")
if not torch.cuda.is_available():
    pytest.skip("needs a CUDA device", allow_module_level=True)

from synth import gen  # noqa: E402
from oracle import block as ob  # noqa: E402
from oracle import pack as opk  # noqa: E402
from paper_2603_02885_b200 import mux  # noqa: E402
from gpu_harness import TOL, bf16_to_f64, from_dev_bf16, rel_err, to_dev_bf16  # noqa: E402


def _f64(t):
    return bf16_to_f64(from_dev_bf16(t))


def _layout(task_lens, chunk_size=0, seed=0):
    """GPU pack of the given per-task lengths -> (row_start device, row_start oracle, max_rows)."""
    off = np.concatenate([[0], np.cumsum([len(x) for x in task_lens])]).astype(np.int32)
    lens = np.concatenate(task_lens).astype(np.int32)
    ref = opk.pack_chunks(off, lens, None, chunk_size, 64)
    R = ref["info"]["total_rows"]
    max_rows = R + 64
    o = mux.pack_chunks(off, lens, None, chunk_size, 64, max_rows=max_rows, max_chunks=max_rows // 64)
    sl = torch.tensor(lens, dtype=torch.int32, device="cuda")
    rs_dev = mux.row_start(sl, o["seq_row"], max_rows)
    ref = opk.pack_chunks(off, lens, None, chunk_size, 64, max_rows=max_rows, max_chunks=max_rows // 64)
    rs_ref = ob.row_seq_start(ref["seq_row"], lens, max_rows)
    return rs_dev, rs_ref, max_rows


def test_row_start_bit_exact():
    lens = [gen.seq_lengths(3, 10 + t, 5, 1, 300) for t in range(4)]
    rs_dev, rs_ref, _ = _layout(lens)
    torch.cuda.synchronize()
    assert np.array_equal(rs_dev.cpu().numpy().astype(np.int64), rs_ref)


@pytest.mark.parametrize("rows,dim", [(37, 4096), (300, 1024), (5, 8)])
def test_rmsnorm(rows, dim):
    st = gen.Stream(7)
    xb = gen.normal_bf16(7, st.take(), (rows, dim), 2.0)
    wb = gen.normal_bf16(7, st.take(), (dim,), 1.0)
    dyb = gen.normal_bf16(7, st.take(), (rows, dim), 1.0)
    x, w, dy = to_dev_bf16(xb), to_dev_bf16(wb), to_dev_bf16(dyb)
    y = mux.rmsnorm_fwd(x, w, 1e-5)
    dx = mux.rmsnorm_bwd(dy, x, w, 1e-5)
    torch.cuda.synchronize()
    X, Wt, DY = bf16_to_f64(xb), bf16_to_f64(wb), bf16_to_f64(dyb)
    assert rel_err(_f64(y), ob.rmsnorm_fwd(X, Wt, 1e-5)) <= TOL
    assert rel_err(_f64(dx), ob.rmsnorm_bwd(DY, X, Wt, 1e-5)) <= TOL
    # fused residual stream: xs = x + res (bf16, written), y = RMSNorm(xs); gradient sums + residual
    rb = gen.normal_bf16(7, st.take(), (rows, dim), 1.0)
    d2b, d3b, gb = (gen.normal_bf16(7, st.take(), (rows, dim), 1.0) for _ in range(3))
    res, d2, d3, gres = to_dev_bf16(rb), to_dev_bf16(d2b), to_dev_bf16(d3b), to_dev_bf16(gb)
    y2, xs = mux.rmsnorm_fwd(x, w, 1e-5, res=res)
    dx2 = mux.rmsnorm_bwd(dy, xs, w, 1e-5, dy2=d2, dy3=d3, resid=gres)
    torch.cuda.synchronize()
    XS = X + bf16_to_f64(rb)
    assert rel_err(_f64(xs), XS) <= TOL
    assert rel_err(_f64(y2), ob.rmsnorm_fwd(XS, Wt, 1e-5)) <= TOL
    ref = ob.rmsnorm_bwd(DY + bf16_to_f64(d2b) + bf16_to_f64(d3b), _f64(xs), Wt, 1e-5) + bf16_to_f64(gb)
    assert rel_err(_f64(dx2), ref) <= TOL


def test_swiglu_on_fused_gate_up():
    rows, F = 129, 1376
    st = gen.Stream(8)
    gub = gen.normal_bf16(8, st.take(), (rows, 2 * F), 2.0)      # [gate | up] as one projection output
    dhb = gen.normal_bf16(8, st.take(), (rows, F), 1.0)
    gu, dh = to_dev_bf16(gub), to_dev_bf16(dhb)
    g, u = gu[:, :F], gu[:, F:]
    h = mux.swiglu_fwd(g, u)
    dgu = torch.empty_like(gu)
    mux.swiglu_bwd(dh, g, u, dg=dgu[:, :F], du=dgu[:, F:])
    torch.cuda.synchronize()
    G, U, DH = bf16_to_f64(gub[:, :F]), bf16_to_f64(gub[:, F:]), bf16_to_f64(dhb)
    assert rel_err(_f64(h), ob.swiglu_fwd(G, U)) <= TOL
    rdg, rdu = ob.swiglu_bwd(DH, G, U)
    got = _f64(dgu)
    assert rel_err(got[:, :F], rdg) <= TOL
    assert rel_err(got[:, F:], rdu) <= TOL


def test_rope_inplace_on_qkv_slice():
    lens = [gen.seq_lengths(4, 20 + t, 6, 1, 400) for t in range(3)]
    rs_dev, rs_ref, R = _layout(lens)
    H, d = 4, 128
    st = gen.Stream(9)
    qkvb = gen.normal_bf16(9, st.take(), (R, 3 * H * d), 1.0)
    qkv = to_dev_bf16(qkvb)
    q = qkv[:, :H * d]
    mux.rope_(q, rs_dev, H, d)
    torch.cuda.synchronize()
    got = _f64(qkv)
    Q = bf16_to_f64(qkvb[:, :H * d]).reshape(R, H, d)
    ref = ob.rope_fwd(Q, rs_ref).reshape(R, H * d)
    assert rel_err(got[:, :H * d], ref) <= TOL
    assert np.array_equal(from_dev_bf16(qkv)[:, H * d:], qkvb[:, H * d:])   # k, v untouched
    pads = rs_ref < 0
    assert np.array_equal(from_dev_bf16(qkv)[pads, :H * d], qkvb[pads, :H * d])
    mux.rope_(q, rs_dev, H, d, inverse=True)                                 # backward = inverse rotation
    torch.cuda.synchronize()
    assert rel_err(_f64(qkv)[:, :H * d], bf16_to_f64(qkvb[:, :H * d])) <= TOL


def _attn_case(task_lens, H, Hkv, seed, chunk_size=0, scale=None):
    rs_dev, rs_ref, R = _layout(task_lens, chunk_size)
    d = 128
    scale = scale or 1.0 / np.sqrt(d)
    st = gen.Stream(seed)
    qb = gen.normal_bf16(seed, st.take(), (R, H * d), 1.0)
    kb = gen.normal_bf16(seed, st.take(), (R, Hkv * d), 1.0)
    vb = gen.normal_bf16(seed, st.take(), (R, Hkv * d), 1.0)
    dob = gen.normal_bf16(seed, st.take(), (R, H * d), 1.0)
    q, k, v, dO = (to_dev_bf16(b) for b in (qb, kb, vb, dob))
    o, lse = mux.attn_fwd(q, k, v, rs_dev, H, Hkv, scale)
    dq, dk, dv = mux.attn_bwd(dO, q, k, v, o, lse, rs_dev, H, Hkv, scale)
    torch.cuda.synchronize()
    G = H // Hkv
    Q = bf16_to_f64(qb).reshape(R, H, d)
    K = np.repeat(bf16_to_f64(kb).reshape(R, Hkv, d), G, axis=1)
    V = np.repeat(bf16_to_f64(vb).reshape(R, Hkv, d), G, axis=1)
    DO = bf16_to_f64(dob).reshape(R, H, d)
    ro, rlse = ob.attention_fwd(Q, K, V, rs_ref, scale)
    # the backward's reference uses the GPU's bf16 O only through D = rowsum(dO * O): the oracle
    # recomputes its own P, so it is independent of the kernel
    rdq, rdk, rdv = ob.attention_bwd(DO, Q, K, V, rs_ref, scale)
    rdk = rdk.reshape(R, Hkv, G, d).sum(axis=2)
    rdv = rdv.reshape(R, Hkv, G, d).sum(axis=2)
    valid = rs_ref >= 0
    errs = {
        "o": rel_err(_f64(o).reshape(R, H, d), ro),
        "lse": float(np.max(np.abs(lse.cpu().numpy()[valid] - rlse[valid]))),
        "dq": rel_err(_f64(dq).reshape(R, H, d), rdq),
        "dk": rel_err(_f64(dk).reshape(R, Hkv, d), rdk),
        "dv": rel_err(_f64(dv).reshape(R, Hkv, d), rdv),
    }
    lse_np = lse.cpu().numpy()
    assert np.isneginf(lse_np[~valid]).all()
    assert (from_dev_bf16(o)[~valid] == 0).all()
    assert (from_dev_bf16(dq)[~valid] == 0).all() and (from_dev_bf16(dk)[~valid] == 0).all()
    return errs


@pytest.mark.parametrize("name,task_lens,H,Hkv", [
    ("short+long", [np.array([1, 5, 64, 65, 130], np.int32), np.array([512, 3], np.int32)], 4, 4),
    ("gqa", [np.array([200, 90, 33], np.int32), np.array([257, 64, 1], np.int32)], 8, 2),
    ("mixed", [gen.seq_lengths(5, 30 + t, 4, 1, 512) for t in range(4)], 2, 1),
])
def test_attention_fwd_bwd(name, task_lens, H, Hkv):
    errs = _attn_case(task_lens, H, Hkv, seed=11)
    print(name, errs)
    assert errs["o"] <= TOL and errs["dq"] <= TOL and errs["dk"] <= TOL and errs["dv"] <= TOL, errs
    assert errs["lse"] <= 2e-2, errs


def test_attention_chunk_128_layout():
    """P:1128's explicit chunk 128: chunks and sequences straddle the 64-row kernel tiles differently."""
    errs = _attn_case([np.array([100, 120, 64], np.int32), np.array([300], np.int32)], 2, 2, seed=12,
                      chunk_size=128)
    assert max(errs["o"], errs["dq"], errs["dk"], errs["dv"]) <= TOL, errs


def test_attention_deterministic():
    lens = [np.array([300, 77], np.int32), np.array([128], np.int32)]
    rs_dev, _, R = _layout(lens)
    st = gen.Stream(13)
    q, k, v, dO = (to_dev_bf16(gen.normal_bf16(13, st.take(), (R, 256), 1.0)) for _ in range(4))
    outs = []
    for _ in range(2):
        o, lse = mux.attn_fwd(q, k, v, rs_dev, 2, 2, 0.088)
        dq, dk, dv = mux.attn_bwd(dO, q, k, v, o, lse, rs_dev, 2, 2, 0.088)
        torch.cuda.synchronize()
        outs.append([t.clone() for t in (o, lse, dq, dk, dv)])
    for a, b in zip(*outs):
        assert torch.equal(a.view(torch.int32) if a.dtype == torch.float32 else a.view(torch.int16),
                           b.view(torch.int32) if b.dtype == torch.float32 else b.view(torch.int16))
