"""fp64 oracle backends injected as each rank's local kernels in the CPU (gloo)
tensor-parallel tests: `OracleBackend` (the multiplexed linear, oracle/linear.c)
and `OracleOps` (+ RMSNorm, RoPE, attention, SwiGLU, add from oracle/block.py).
Test infrastructure only."""
import numpy as np
import torch

from oracle import block as ob
from oracle import linear as olin


class OracleBackend:
    """fp64 oracle as the per-rank local linear (torch fp64 CPU tensors in/out).  col_off: a fused
    projection (adapters[t][s], oracle linear_*_sliced)."""

    @staticmethod
    def _tabs(ads, col_off):
        if col_off is None:
            return ([a.A.numpy() for a in ads], [a.B.numpy() for a in ads], [a.rank for a in ads],
                    [a.scale for a in ads])
        return ([[a.A.numpy() for a in row] for row in ads], [[a.B.numpy() for a in row] for row in ads],
                [[a.rank for a in row] for row in ads], [[a.scale for a in row] for row in ads])

    def fwd(self, seg_off, seg_task, ads, X, W, r_cap, Y=None, col_off=None):
        A, B, rk, sc = self._tabs(ads, col_off)
        if col_off is None:
            Yn, Hs = olin.linear_fwd(seg_off.numpy(), seg_task, A, B, rk, sc, X.numpy(), W.numpy(), r_cap)
        else:
            Yn, Hs = olin.linear_fwd_sliced(seg_off.numpy(), seg_task, col_off, A, B, rk, sc, X.numpy(), W.numpy(),
                                            r_cap)
        return torch.from_numpy(Yn), torch.from_numpy(Hs)

    def shrink(self, seg_off, seg_task, ads, X, W, r_cap, row_begin, row_end, col_off=None):
        # rows outside the range are NaN: only the all-gathered own rows may reach the forward
        _, Hs = self.fwd(seg_off, seg_task, ads, X, W, r_cap, col_off=col_off)
        Hs = Hs.clone()
        Hs[:row_begin] = float("nan")
        Hs[row_end:] = float("nan")
        return Hs

    def fwd_hs(self, seg_off, seg_task, ads, X, W, Hs, r_cap, col_off=None):
        # Eq. 1 with the given (gathered) shrink: Y = X W^T + Hs B_t^T on each segment's rows
        # (per slice s: Hs columns [s r_cap, s r_cap + rank) times B_{t,s} into the slice's columns)
        Y = X.numpy() @ W.numpy().T
        so, Hn = seg_off.numpy(), Hs.numpy()
        co = [0, W.shape[0]] if col_off is None else col_off
        for s, t in enumerate(seg_task):
            row = [ads[t]] if col_off is None else ads[t]
            for c, a in enumerate(row):
                if a.rank:
                    Y[so[s]:so[s + 1], co[c]:co[c + 1]] += (Hn[so[s]:so[s + 1], c * r_cap:c * r_cap + a.rank]
                                                            @ a.B.numpy().T)
        return torch.from_numpy(Y)

    def shrink_bwd(self, seg_off, seg_task, ads, dY, W, r_cap, row_begin, row_end, col_off=None):
        # Gs = s dY B_t of the oracle; rows outside the range are NaN: only the all-gathered own rows may
        # reach the backward
        A, B, rk, sc = self._tabs(ads, col_off)
        N = W.shape[0]
        K = W.shape[1]
        dYn = np.ascontiguousarray(dY.numpy())
        Xz = np.zeros((dYn.shape[0], K))
        if col_off is None:
            _, Gs, _ = olin.linear_bwd(seg_off.numpy(), seg_task, A, B, rk, sc, dYn, Xz, W.numpy(), r_cap)
        else:
            _, Gs, _ = olin.linear_bwd_sliced(seg_off.numpy(), seg_task, col_off, A, B, rk, sc, dYn, Xz, W.numpy(),
                                              r_cap)
        Gs = torch.from_numpy(Gs.copy())
        Gs[:row_begin] = float("nan")
        Gs[row_end:] = float("nan")
        return Gs

    def bwd(self, seg_off, seg_task, ads, dY, X, W, Hs, r_cap, dX=None, col_off=None, Gs=None):
        # the oracle recomputes H from X (fp64), which equals the saved Hs / s
        A, B, rk, sc = self._tabs(ads, col_off)
        dYn = np.ascontiguousarray(dY.numpy())
        if Gs is not None:   # the given (gathered) Gs: dX = dY W + Gs A_t, dA_t = Gs^T X on each segment
            return self._bwd_gs(seg_off, seg_task, ads, dYn, X, W, Gs, r_cap, dX, col_off, A, B, rk, sc)
        if col_off is None:
            dXn, Gs, grads = olin.linear_bwd(seg_off.numpy(), seg_task, A, B, rk, sc, dYn, X.numpy(), W.numpy(),
                                             r_cap)
            dA, dB = [torch.from_numpy(g[0]) for g in grads], [torch.from_numpy(g[1]) for g in grads]
        else:
            dXn, Gs, grads = olin.linear_bwd_sliced(seg_off.numpy(), seg_task, col_off, A, B, rk, sc, dYn,
                                                    X.numpy(), W.numpy(), r_cap)
            dA = [[torch.from_numpy(g[0]) for g in row] for row in grads]
            dB = [[torch.from_numpy(g[1]) for g in row] for row in grads]
        out = torch.from_numpy(dXn)
        if dX is not None:
            dX.copy_(out)
            out = dX
        return out, dA, dB

    def _bwd_gs(self, seg_off, seg_task, ads, dYn, X, W, Gs, r_cap, dX, col_off, A, B, rk, sc):
        # dB_t (needs H, not Gs) from the oracle; dX and dA_t from the given Gs
        if col_off is None:
            _, _, grads = olin.linear_bwd(seg_off.numpy(), seg_task, A, B, rk, sc, dYn, X.numpy(), W.numpy(), r_cap)
            rows_ads = [[a] for a in ads]
        else:
            _, _, grads = olin.linear_bwd_sliced(seg_off.numpy(), seg_task, col_off, A, B, rk, sc, dYn, X.numpy(),
                                                 W.numpy(), r_cap)
            rows_ads = ads
        so, Gn, Xn = seg_off.numpy(), Gs.numpy(), X.numpy()
        dXn = dYn @ W.numpy()
        dAs = [[np.zeros_like(np.asarray(a.A.numpy(), dtype=np.float64)) if a.rank else None for a in row]
               for row in rows_ads]
        for s_, t in enumerate(seg_task):
            lo, hi = so[s_], so[s_ + 1]
            for c, a in enumerate(rows_ads[t]):
                if a.rank:
                    g = Gn[lo:hi, c * r_cap:c * r_cap + a.rank]
                    dXn[lo:hi] += g @ a.A.numpy()
                    dAs[t][c] += g.T @ Xn[lo:hi]
        if col_off is None:
            dA = [torch.from_numpy(row[0]) if row[0] is not None else None for row in dAs]
            dB = [torch.from_numpy(g[1]) for g in grads]
        else:
            dA = [[torch.from_numpy(x) if x is not None else None for x in row] for row in dAs]
            dB = [[torch.from_numpy(g[1]) for g in row] for row in grads]
        out = torch.from_numpy(dXn)
        if dX is not None:
            dX.copy_(out)
            out = dX
        return out, dA, dB


class OracleOps:
    """fp64 oracle as each rank's local kernels (torch fp64 CPU tensors in and out)."""

    def __init__(self, head_dim):
        self.d = head_dim
        self.lin = OracleBackend()

    def fwd(self, *a, **kw):
        return self.lin.fwd(*a, **kw)

    def bwd(self, *a, **kw):
        return self.lin.bwd(*a, **kw)

    def shrink(self, *a, **kw):
        return self.lin.shrink(*a, **kw)

    def fwd_hs(self, *a, **kw):
        return self.lin.fwd_hs(*a, **kw)

    def shrink_bwd(self, *a, **kw):
        return self.lin.shrink_bwd(*a, **kw)

    def rmsnorm_fwd(self, x, w, eps, res=None):
        if res is None:
            return torch.from_numpy(ob.rmsnorm_fwd(x.numpy(), w.numpy(), eps))
        xs = x.numpy() + res.numpy()
        return torch.from_numpy(ob.rmsnorm_fwd(xs, w.numpy(), eps)), torch.from_numpy(xs)

    def rmsnorm_bwd(self, dy, x, w, eps, resid=None):
        dx = ob.rmsnorm_bwd(dy.numpy(), x.numpy(), w.numpy(), eps)
        return torch.from_numpy(dx + (0 if resid is None else resid.numpy()))

    def rope(self, x, row_start, heads, head_dim, base, inverse=False):
        # in place, like mux_rope (x may be a column view of a fused projection's output)
        R = x.shape[0]
        f = ob.rope_bwd if inverse else ob.rope_fwd
        y = f(np.ascontiguousarray(x.numpy()).reshape(R, heads, head_dim), row_start.numpy(), base).reshape(R, -1)
        x.copy_(torch.from_numpy(y))
        return x

    def empty(self, rows, cols, like):
        return torch.empty(rows, cols, dtype=like.dtype)

    @staticmethod
    def _into(out, vals):
        if out is None:
            return vals
        for o, v in zip(out, vals):
            o.copy_(v)
        return out

    def attn_fwd(self, q, k, v, row_start, heads, kv_heads, scale):
        q, k, v = (t.contiguous() for t in (q, k, v))
        R, d, G = q.shape[0], self.d, heads // kv_heads
        Kf = np.repeat(k.numpy().reshape(R, kv_heads, d), G, axis=1)
        Vf = np.repeat(v.numpy().reshape(R, kv_heads, d), G, axis=1)
        o, lse = ob.attention_fwd(q.numpy().reshape(R, heads, d), Kf, Vf, row_start.numpy(), scale)
        return torch.from_numpy(o.reshape(R, heads * d)), torch.from_numpy(lse)

    def attn_bwd(self, dO, q, k, v, o, lse, row_start, heads, kv_heads, scale, out=None):
        q, k, v = (t.contiguous() for t in (q, k, v))
        R, d, G = q.shape[0], self.d, heads // kv_heads
        Kf = np.repeat(k.numpy().reshape(R, kv_heads, d), G, axis=1)
        Vf = np.repeat(v.numpy().reshape(R, kv_heads, d), G, axis=1)
        dq, dk, dv = ob.attention_bwd(dO.numpy().reshape(R, heads, d), q.numpy().reshape(R, heads, d), Kf, Vf,
                                      row_start.numpy(), scale)
        dk = dk.reshape(R, kv_heads, G, d).sum(axis=2).reshape(R, kv_heads * d)
        dv = dv.reshape(R, kv_heads, G, d).sum(axis=2).reshape(R, kv_heads * d)
        return self._into(out, (torch.from_numpy(dq.reshape(R, heads * d)), torch.from_numpy(dk),
                                torch.from_numpy(dv)))

    def swiglu_fwd(self, g, u):
        return torch.from_numpy(ob.swiglu_fwd(np.ascontiguousarray(g.numpy()), np.ascontiguousarray(u.numpy())))

    def swiglu_bwd(self, dh, g, u, out=None):
        dg, du = ob.swiglu_bwd(dh.numpy(), np.ascontiguousarray(g.numpy()), np.ascontiguousarray(u.numpy()))
        return self._into(out, (torch.from_numpy(dg), torch.from_numpy(du)))

    def add(self, a, b, out=None):
        return a + b
