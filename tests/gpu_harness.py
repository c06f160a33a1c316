"""Shared helpers for the `-m gpu` parity tests: build one multiplexed linear
problem from the seeded generator, run it through the C ABI (binding in
paper_2603_02885_b200.mux) and through the fp64 oracle, and compare.

Tolerance (north_star): max|gpu - oracle| / max|oracle| <= 2e-2 per tensor
(Y, dX, Hs, and per task dA_t, dB_t).  Integer-valued inputs: exact.
"""
from __future__ import annotations

import numpy as np
import torch

import synth
from synth import gen
from oracle import linear as olin

TOL = 2e-2


def to_dev_bf16(bits: np.ndarray) -> torch.Tensor:
    t = torch.from_numpy(np.ascontiguousarray(bits).view(np.int16)).view(torch.bfloat16)
    return t.cuda()


def from_dev_bf16(t: torch.Tensor) -> np.ndarray:
    return t.contiguous().view(torch.int16).cpu().numpy().view(np.uint16)


def bf16_to_f64(bits: np.ndarray) -> np.ndarray:
    return gen.bf16_bits_to_f32(bits).astype(np.float64)


def rel_err(gpu: np.ndarray, ref: np.ndarray) -> float:
    gpu = np.asarray(gpu, dtype=np.float64)
    ref = np.asarray(ref, dtype=np.float64)
    m = float(np.max(np.abs(ref))) if ref.size else 0.0
    d = float(np.max(np.abs(gpu - ref))) if ref.size else 0.0
    return d / m if m > 0 else d


class Problem:
    """One multiplexed linear call: segments, adapters, X, W, dY (bf16 bits)."""

    def __init__(self, K, N, seg_lens, ranks, seg_task=None, scales=None, variant="normal", seed=1,
                 r_cap=None, max_rows=None, pad_rows=None):
        self.K, self.N = K, N
        self.seg_off = np.concatenate([[0], np.cumsum(seg_lens)]).astype(np.int32)
        self.R = int(self.seg_off[-1])
        self.max_rows = max_rows or max(self.R, 1)
        S = len(seg_lens)
        self.seg_task = list(seg_task) if seg_task is not None else [s % len(ranks) for s in range(S)]
        self.ranks = list(ranks)
        self.scales = list(scales) if scales is not None else [2.0] * len(ranks)
        self.r_cap = r_cap or max(16, -(-max(max(ranks), 1) // 16) * 16)
        st = gen.Stream(seed)
        if variant == "int":
            self.X = gen.int_bf16(seed, st.take(), (self.max_rows, K), -4, 4)
            self.W = gen.int_bf16(seed, st.take(), (N, K), -4, 4)
            self.dY = gen.int_bf16(seed, st.take(), (self.max_rows, N), -4, 4)
            self.A = [gen.sparse_int_bf16(seed, st.take(), (r, K), 8, 1, -2, 2) for r in ranks]
            self.B = [gen.sparse_int_bf16(seed, st.take(), (N, r), 8, 0, -2, 2) for r in ranks]
        else:
            self.X = gen.normal_bf16(seed, st.take(), (self.max_rows, K), 1.0)
            self.W = gen.normal_bf16(seed, st.take(), (N, K), 1.0 / np.sqrt(K))
            self.dY = gen.normal_bf16(seed, st.take(), (self.max_rows, N), 1.0)
            self.A = [gen.normal_bf16(seed, st.take(), (r, K), 1.0 / np.sqrt(K)) for r in ranks]
            self.B = [gen.normal_bf16(seed, st.take(), (N, r), 1.0 / np.sqrt(max(r, 1))) for r in ranks]
            if variant == "zeroB":
                self.B = [np.zeros_like(b) for b in self.B]
        if pad_rows is not None:       # rows that are chunk padding: X = 0 there
            self.X[pad_rows] = 0

    # ---------------------------------------------------------------- GPU
    def gpu_adapters(self):
        from paper_2603_02885_b200 import mux
        ads = []
        for t, r in enumerate(self.ranks):
            if r == 0:
                ads.append(mux.Adapter(None, None, 0, self.scales[t]))
                continue
            A = to_dev_bf16(self.A[t])
            B = mux.make_B_storage(self.N, r)
            B.copy_(to_dev_bf16(self.B[t]))
            ads.append(mux.Adapter(A, B, r, self.scales[t]))
        return ads

    def run_gpu(self, bwd=True, want_dx=True):
        from paper_2603_02885_b200 import mux
        seg_off = torch.from_numpy(self.seg_off).cuda()
        X, W, dY = to_dev_bf16(self.X), to_dev_bf16(self.W), to_dev_bf16(self.dY)
        ads = self.gpu_adapters()
        Y, Hs = mux.linear_fwd(seg_off, self.seg_task, ads, X, W, self.r_cap)
        out = {"Y": Y, "Hs": Hs}
        if bwd:
            dX = mux.linear_bwd(seg_off, self.seg_task, ads, dY, X, W, Hs, self.r_cap, want_dx=want_dx)
            out["dX"] = dX
            out["dA"] = [a.dA for a in ads]
            out["dB"] = [a.dB for a in ads]
        torch.cuda.synchronize()
        res = {"Y": from_dev_bf16(out["Y"])[: self.R], "Hs": from_dev_bf16(out["Hs"])[: self.R]}
        if bwd:
            res["dX"] = from_dev_bf16(out["dX"])[: self.R] if out["dX"] is not None else None
            res["dA"] = [None if a is None else a.cpu().numpy() for a in out["dA"]]
            res["dB"] = [None if b is None else b.cpu().numpy() for b in out["dB"]]
        return res

    # ---------------------------------------------------------------- oracle
    def run_oracle(self, bwd=True, rows=None):
        Y, Hs = olin.linear_fwd(self.seg_off, self.seg_task, self.A, self.B, self.ranks, self.scales,
                                self.X, self.W, self.r_cap, rows=rows)
        out = {"Y": Y, "Hs": Hs}
        if bwd:
            dX, Gs, grads = olin.linear_bwd(self.seg_off, self.seg_task, self.A, self.B, self.ranks,
                                            self.scales, self.dY, self.X, self.W, self.r_cap, rows=rows)
            out.update(dX=dX, Gs=Gs, dA=[g[0] for g in grads], dB=[g[1] for g in grads])
        return out


def compare(prob: Problem, gpu: dict, ref: dict, rows=None, tol=TOL, exact=False):
    """Returns {name: rel_err}; asserts all within tol (or exact)."""
    errs = {}
    sel = slice(None) if rows is None else rows
    for name in ("Y", "dX"):
        if name not in gpu or gpu[name] is None:
            continue
        g = bf16_to_f64(gpu[name][sel])
        r = ref[name]
        if exact:
            rb = gen.bf16_bits_from_f64(r)
            assert np.array_equal(gpu[name][sel], rb), f"{name}: not bit-exact"
        errs[name] = rel_err(g, r)
    g = bf16_to_f64(gpu["Hs"])
    errs["Hs"] = rel_err(g, ref["Hs"])
    if exact:
        assert np.array_equal(gpu["Hs"], gen.bf16_bits_from_f64(ref["Hs"])), "Hs: not bit-exact"
    if "dA" in gpu:
        for t, r in enumerate(prob.ranks):
            if r == 0:
                continue
            errs[f"dA{t}"] = rel_err(gpu["dA"][t], ref["dA"][t])
            errs[f"dB{t}"] = rel_err(gpu["dB"][t], ref["dB"][t])
            if exact:
                assert np.array_equal(gpu["dA"][t].astype(np.float64), ref["dA"][t]), f"dA{t} not exact"
                assert np.array_equal(gpu["dB"][t].astype(np.float64), ref["dB"][t]), f"dB{t} not exact"
    bad = {k: v for k, v in errs.items() if not (v <= tol)}
    assert not bad, f"tolerance {tol} exceeded: {bad} (all: {errs})"
    return errs
