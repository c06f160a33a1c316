"""fp64 oracle backends injected as each rank's local kernels in the CPU (gloo)
tensor-parallel tests: `OracleBackend` (the multiplexed linear, oracle/linear.c)
and `OracleOps` (+ RMSNorm, RoPE, attention, SwiGLU, add from oracle/block.py).
Test infrastructure only."""
import numpy as np
import torch

from oracle import block as ob
from oracle import linear as olin


class OracleBackend:
    """fp64 oracle as the per-rank local linear (torch fp64 CPU tensors in/out)."""

    def fwd(self, seg_off, seg_task, ads, X, W, r_cap):
        Y, Hs = olin.linear_fwd(seg_off.numpy(), seg_task, [a.A.numpy() for a in ads],
                                [a.B.numpy() for a in ads], [a.rank for a in ads], [a.scale for a in ads],
                                X.numpy(), W.numpy(), r_cap)
        return torch.from_numpy(Y), torch.from_numpy(Hs)

    def shrink(self, seg_off, seg_task, ads, X, W, r_cap, row_begin, row_end):
        # rows outside the range are NaN: only the all-gathered own rows may reach the forward
        _, Hs = self.fwd(seg_off, seg_task, ads, X, W, r_cap)
        Hs = Hs.clone()
        Hs[:row_begin] = float("nan")
        Hs[row_end:] = float("nan")
        return Hs

    def fwd_hs(self, seg_off, seg_task, ads, X, W, Hs, r_cap):
        # Eq. 1 with the given (gathered) shrink: Y = X W^T + Hs B_t^T on each segment's rows
        Y = X.numpy() @ W.numpy().T
        so, Hn = seg_off.numpy(), Hs.numpy()
        for s, t in enumerate(seg_task):
            a = ads[t]
            if a.rank:
                Y[so[s]:so[s + 1]] += Hn[so[s]:so[s + 1], :a.rank] @ a.B.numpy().T
        return torch.from_numpy(Y)

    def bwd(self, seg_off, seg_task, ads, dY, X, W, Hs, r_cap):
        # the oracle recomputes H from X (fp64), which equals the saved Hs / s
        dX, Gs, grads = olin.linear_bwd(seg_off.numpy(), seg_task, [a.A.numpy() for a in ads],
                                        [a.B.numpy() for a in ads], [a.rank for a in ads],
                                        [a.scale for a in ads], dY.numpy(), X.numpy(), W.numpy(), r_cap)
        return (torch.from_numpy(dX), [torch.from_numpy(g[0]) for g in grads],
                [torch.from_numpy(g[1]) for g in grads])


class OracleOps:
    """fp64 oracle as each rank's local kernels (torch fp64 CPU tensors in and out)."""

    def __init__(self, head_dim):
        self.d = head_dim
        self.lin = OracleBackend()

    def fwd(self, *a):
        return self.lin.fwd(*a)

    def bwd(self, *a):
        return self.lin.bwd(*a)

    def rmsnorm_fwd(self, x, w, eps, res=None):
        if res is None:
            return torch.from_numpy(ob.rmsnorm_fwd(x.numpy(), w.numpy(), eps))
        xs = x.numpy() + res.numpy()
        return torch.from_numpy(ob.rmsnorm_fwd(xs, w.numpy(), eps)), torch.from_numpy(xs)

    def rmsnorm_bwd(self, dy, x, w, eps, resid=None):
        dx = ob.rmsnorm_bwd(dy.numpy(), x.numpy(), w.numpy(), eps)
        return torch.from_numpy(dx + (0 if resid is None else resid.numpy()))

    def rope(self, x, row_start, heads, head_dim, base, inverse=False):
        R = x.shape[0]
        f = ob.rope_bwd if inverse else ob.rope_fwd
        return torch.from_numpy(f(x.numpy().reshape(R, heads, head_dim), row_start.numpy(), base).reshape(R, -1))

    def attn_fwd(self, q, k, v, row_start, heads, kv_heads, scale):
        R, d, G = q.shape[0], self.d, heads // kv_heads
        Kf = np.repeat(k.numpy().reshape(R, kv_heads, d), G, axis=1)
        Vf = np.repeat(v.numpy().reshape(R, kv_heads, d), G, axis=1)
        o, lse = ob.attention_fwd(q.numpy().reshape(R, heads, d), Kf, Vf, row_start.numpy(), scale)
        return torch.from_numpy(o.reshape(R, heads * d)), torch.from_numpy(lse)

    def attn_bwd(self, dO, q, k, v, o, lse, row_start, heads, kv_heads, scale):
        R, d, G = q.shape[0], self.d, heads // kv_heads
        Kf = np.repeat(k.numpy().reshape(R, kv_heads, d), G, axis=1)
        Vf = np.repeat(v.numpy().reshape(R, kv_heads, d), G, axis=1)
        dq, dk, dv = ob.attention_bwd(dO.numpy().reshape(R, heads, d), q.numpy().reshape(R, heads, d), Kf, Vf,
                                      row_start.numpy(), scale)
        dk = dk.reshape(R, kv_heads, G, d).sum(axis=2).reshape(R, kv_heads * d)
        dv = dv.reshape(R, kv_heads, G, d).sum(axis=2).reshape(R, kv_heads * d)
        return torch.from_numpy(dq.reshape(R, heads * d)), torch.from_numpy(dk), torch.from_numpy(dv)

    def swiglu_fwd(self, g, u):
        return torch.from_numpy(ob.swiglu_fwd(g.numpy(), u.numpy()))

    def swiglu_bwd(self, dh, g, u):
        dg, du = ob.swiglu_bwd(dh.numpy(), g.numpy(), u.numpy())
        return torch.from_numpy(dg), torch.from_numpy(du)

    def add(self, a, b, out=None):
        return a + b
