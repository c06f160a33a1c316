"""GPU parity at BASELINE.json's full sizes, in bench.py's launch configuration:
the real packed row layout of each config (mux_pack_chunks on the GPU, checked
bit-exact against the oracle pack), full K/N, all tasks/ranks, pad rows zero.
Y and dX are compared on a row sample the oracle computes one by one (first
and last 32 rows of every segment + 64 seeded rows); Hs, dA_t
and dB_t on every row.  Bar: max|gpu-oracle|/max|oracle| <= 2e-2."""
import numpy as np
import pytest

pytestmark = pytest.mark.gpu

torch = pytest.importorskip("torch")
if not torch.cuda.is_available():
    pytest.skip("needs a CUDA device", allow_module_level=True)

import synth  # noqa: E402
from synth import gen  # noqa: E402
from oracle import pack as opk  # noqa: E402
from oracle import linear as olin  # noqa: E402
from paper_2603_02885_b200 import mux  # noqa: E402
from gpu_harness import to_dev_bf16, from_dev_bf16, bf16_to_f64, rel_err, TOL  # noqa: E402


def _row_sample(seg_off, seed):
    rows = []
    for s in range(len(seg_off) - 1):
        a, b = int(seg_off[s]), int(seg_off[s + 1])
        rows += list(range(a, min(a + 32, b))) + list(range(max(b - 32, a), b))
    rng = np.random.default_rng(seed)
    rows += list(rng.integers(0, int(seg_off[-1]), 64))
    return np.unique(np.array(rows, np.int64))


CASES = [("2", 0), ("2", 1), ("2", 2), ("3a", 2), ("3b", 0), ("3c", 1), ("4", 0), ("4", 4), ("4", 6),
         ("5", 0), ("5", 1)]


@pytest.mark.parametrize("cid,li", CASES)
def test_full_size_linear(cid, li):
    _full_size(cid, li)


# tensor-parallel shards at TP 8: each rank's local linear is itself a multiplexed
# linear on a slice; these exercise the narrow-tile path (config 5 k: N = 1024/8 = 128), the
# short-reduction schedule (config 5 o: K = 8192/8 = 1024; config 4 q's dX: N = 512) at full rows
TP_CASES = [("5", 1, 8, "col", 3), ("5", 3, 8, "row", 5), ("4", 0, 8, "col", 0), ("4", 6, 8, "row", 7)]


@pytest.mark.parametrize("cid,li,p,kind,part", TP_CASES)
def test_full_size_tp_shard(cid, li, p, kind, part):
    _full_size(cid, li, (p, kind, part))


def _full_size(cid, li, shard=None):
    wl = synth.workload(cid)
    off, lens = wl.csr()
    L = wl.linears[li]
    ref = opk.pack_chunks(off, lens, wl.pack_capacity, wl.chunk_size, wl.chunk_min)
    R = ref["info"]["total_rows"]
    max_rows = int(mux.pack_bound_rows(wl.valid_tokens, wl.num_seqs, 64))
    ref = opk.pack_chunks(off, lens, wl.pack_capacity, wl.chunk_size, wl.chunk_min, max_rows=max_rows,
                          max_chunks=max_rows // 64)
    o = mux.pack_chunks(list(off), list(lens), wl.pack_capacity, wl.chunk_size, wl.chunk_min,
                        max_rows=max_rows, max_chunks=max_rows // 64)
    torch.cuda.synchronize()
    assert np.array_equal(o["seg_off"].cpu().numpy(), ref["seg_off"])
    assert np.array_equal(o["row_src"].cpu().numpy(), ref["row_src"])

    # token-major inputs -> packed rows (GPU: mux_pack_apply; oracle: numpy placement)
    Xtok = synth.token_input(wl, li, "X", L.K)
    dYtok = synth.token_input(wl, li, "dY", L.N)
    W = synth.weight(wl, li)
    A, B = zip(*[synth.adapter(wl, li, t) for t in range(wl.num_tasks)])
    K, N = L.K, L.N
    if shard is not None:  # Megatron shard of this rank: column = N slice, row = K slice
        p, kind, part = shard
        c = np.ascontiguousarray
        if kind == "col":
            N //= p
            n0 = part * N
            W, dYtok = c(W[n0:n0 + N]), c(dYtok[:, n0:n0 + N])
            B = tuple(c(b[n0:n0 + N]) for b in B)
        else:
            K //= p
            k0 = part * K
            W, Xtok = c(W[:, k0:k0 + K]), c(Xtok[:, k0:k0 + K])
            A = tuple(c(a[:, k0:k0 + K]) for a in A)
    X = mux.pack_apply(o["row_src"], to_dev_bf16(Xtok), max_rows)
    dY = mux.pack_apply(o["row_src"], to_dev_bf16(dYtok), max_rows)
    rs = ref["row_src"][:R]
    Xp = np.zeros((R, K), np.uint16)
    Xp[rs >= 0] = Xtok[rs[rs >= 0]]
    dYp = np.zeros((R, N), np.uint16)
    dYp[rs >= 0] = dYtok[rs[rs >= 0]]
    assert np.array_equal(from_dev_bf16(X)[:R], Xp)
    r_cap = 16 * -(-max(wl.ranks) // 16)
    ads = []
    for t, r in enumerate(wl.ranks):
        Bs = mux.make_B_storage(N, r)
        Bs.copy_(to_dev_bf16(B[t]))
        ads.append(mux.Adapter(to_dev_bf16(A[t]), Bs, r, wl.scales[t]))
    seg_task = list(range(wl.num_tasks))
    Wd = to_dev_bf16(W)
    Y, Hs = mux.linear_fwd(o["seg_off"], seg_task, ads, X, Wd, r_cap)
    dX = mux.linear_bwd(o["seg_off"], seg_task, ads, dY, X, Wd, Hs, r_cap)
    torch.cuda.synchronize()

    rows = _row_sample(ref["seg_off"], 99)
    Yr, Hsr = olin.linear_fwd(ref["seg_off"], seg_task, list(A), list(B), wl.ranks, wl.scales, Xp, W, r_cap,
                              rows=rows)
    dXr, _, grads = olin.linear_bwd(ref["seg_off"], seg_task, list(A), list(B), wl.ranks, wl.scales, dYp, Xp, W,
                                    r_cap, rows=rows)
    errs = {"Y": rel_err(bf16_to_f64(from_dev_bf16(Y)[rows]), Yr),
            "dX": rel_err(bf16_to_f64(from_dev_bf16(dX)[rows]), dXr),
            "Hs": rel_err(bf16_to_f64(from_dev_bf16(Hs)[:R]), Hsr)}
    for t in range(wl.num_tasks):
        errs[f"dA{t}"] = rel_err(ads[t].dA.cpu().numpy(), grads[t][0])
        errs[f"dB{t}"] = rel_err(ads[t].dB.cpu().numpy(), grads[t][1])
    # pad rows of Y are exactly zero (X pad rows are zero, R10)
    pad = np.where(rs < 0)[0]
    if len(pad):
        assert np.all(bf16_to_f64(from_dev_bf16(Y)[pad]) == 0.0)
    worst = max(errs.values())
    print(cid, L.name, shard, R, "worst", worst)
    assert worst <= TOL, errs
