"""A LLaMA decoder block whose seven linears (q, k, v, o, gate, up, down) are
multiplexed LoRA linears: one hTask's
packed rows go through the whole block, forward and backward, with every
step a libmux kernel (thin glue; no arithmetic here):

  h1 = RMSNorm(x);  q, k, v = mux_linear(h1);  RoPE(q, k)
  a  = causal attention inside packed sequences (chunk KV reuse)
  x2 = x + mux_linear_o(a);  h2 = RMSNorm(x2)
  y  = x2 + mux_linear_down(SwiGLU(mux_linear_gate(h2), mux_linear_up(h2)))

The backbone (linears, norms) is frozen: backward returns dx and
writes every adapter's dA/dB.  Attention, RMSNorm and SwiGLU are not BaseOps
("Attention is excluded"): they carry no adapters.
"""
from __future__ import annotations

from dataclasses import dataclass
from typing import Dict, List, Sequence

import torch

from . import mux

LINEARS = ("q", "k", "v", "o", "gate", "up", "down")
# fused projections (include/mux.h "Fused projections"): one column-sliced GEMM each, every task
# keeping its own adapter on every slice
FUSED = {"qkv": ("q", "k", "v"), "gate_up": ("gate", "up")}


@dataclass
class BlockShape:
    hidden: int = 4096
    ffn: int = 11008
    heads: int = 32
    kv_heads: int = 32
    head_dim: int = 128
    eps: float = 1e-5
    rope_base: float = 10000.0

    def linear_dims(self) -> Dict[str, tuple]:
        """(K, N) of each linear."""
        H, F, kv = self.hidden, self.ffn, self.kv_heads * self.head_dim
        return {"q": (H, self.heads * self.head_dim), "k": (H, kv), "v": (H, kv),
                "o": (self.heads * self.head_dim, H), "gate": (H, F), "up": (H, F), "down": (F, H)}


class DecoderBlock:
    """weights: {"q".."down": W [N, K] bf16, "norm1", "norm2": [hidden] bf16};
    adapters: {"q".."down": [mux.Adapter per task]} (dA/dB allocated here)."""

    def __init__(self, shape: BlockShape, weights: Dict[str, torch.Tensor], adapters: Dict[str, List[mux.Adapter]],
                 r_cap: int, fused: bool = False):
        """fused: q|k|v and gate|up run as one column-sliced GEMM each (their W concatenated once here;
        the adapters keep their per-linear objects, so dA/dB land where they do unfused)."""
        self.s, self.w, self.ads, self.r_cap = shape, dict(weights), dict(adapters), r_cap
        self.fused = fused
        self.col_off = {}
        dims = shape.linear_dims()
        for name in LINEARS:
            K, N = dims[name]
            assert tuple(weights[name].shape) == (N, K), (name, weights[name].shape)
            for a in adapters[name]:
                if a.rank and a.dA is None:
                    a.dA = torch.empty(a.rank, K, dtype=torch.float32, device=weights[name].device)
                if a.rank and a.dB is None:
                    a.dB = torch.empty(N, a.rank, dtype=torch.float32, device=weights[name].device)
        if fused:
            for f, parts in FUSED.items():
                self.w[f] = torch.cat([weights[n] for n in parts], 0).contiguous()
                self.ads[f] = [[adapters[n][t] for n in parts] for t in range(len(adapters[parts[0]]))]
                off = [0]
                for n in parts:
                    off.append(off[-1] + weights[n].shape[0])
                self.col_off[f] = off
        self._buf: Dict[str, torch.Tensor] = {}
        self._rows = -1
        self.overlap_grads = True
        self._side = torch.cuda.Stream(device=weights["q"].device)
        self._events: Dict[str, torch.cuda.Event] = {}

    def _b(self, name, cols, dtype=torch.bfloat16):
        t = self._buf.get(name)
        if t is None or t.shape[0] != self._rows or t.shape[1] != cols or t.dtype != dtype:
            t = torch.empty(self._rows, cols, dtype=dtype, device=self.w["q"].device)
            self._buf[name] = t
        return t

    def _ws(self, name, n_segs):
        N, K = self.w[name].shape
        S = len(self.col_off[name]) - 1 if name in self.col_off else 1
        need = mux.linear_workspace_size(n_segs, self._rows, K, N, self.r_cap * S)
        t = self._buf.get("ws_" + name)
        if t is None or t.numel() < need:
            t = torch.zeros(need, dtype=torch.uint8, device=self.w["q"].device)
            self._buf["ws_" + name] = t
        return t

    def _lin_fwd(self, name, X):
        N = self.w[name].shape[0]
        co = self.col_off.get(name)
        Y, Hs = self._b(name + ".y", N), self._b(name + ".hs", self.r_cap * (1 if co is None else len(co) - 1))
        ws = self._ws(name, len(self.seg_task))
        if co is not None:
            mux.linear_fwd_sliced(self.seg_off, self.seg_task, self.ads[name], X, self.w[name], co, self.r_cap, Y=Y,
                                  Hs=Hs, workspace=ws)
        else:
            mux.linear_fwd(self.seg_off, self.seg_task, self.ads[name], X, self.w[name], self.r_cap, Y=Y, Hs=Hs,
                           workspace=ws)
        return Y

    def _lin_bwd(self, name, dY, X, out):
        """dX GEMM on the caller's stream; the adapter gradients (HBM-bound) on a side stream, where
        they fill the tail of the next tensor-bound GEMM (joined at the end of backward())."""
        ws = self._ws(name, len(self.seg_task))
        co = self.col_off.get(name)
        if co is not None:
            def call(**kw):
                mux.linear_bwd_sliced(self.seg_off, self.seg_task, self.ads[name], dY, X, self.w[name],
                                      self._buf[name + ".hs"], co, self.r_cap, workspace=ws, **kw)
        else:
            def call(**kw):
                mux.linear_bwd(self.seg_off, self.seg_task, self.ads[name], dY, X, self.w[name],
                               self._buf[name + ".hs"], self.r_cap, workspace=ws, **kw)
        if not self.overlap_grads:
            call(dX=out)
            return out
        main = torch.cuda.current_stream()
        call(dX=out, part=mux.BWD_DX)
        ev = self._events.setdefault(name, torch.cuda.Event())
        ev.record(main)
        self._side.wait_event(ev)
        call(dX=out, part=mux.BWD_GRADS, stream=self._side)
        return out

    def forward(self, x: torch.Tensor, seg_off: torch.Tensor, seg_task: Sequence[int], row_start: torch.Tensor):
        s = self.s
        self._rows = x.shape[0]
        self.seg_off, self.seg_task, self.row_start = seg_off, list(seg_task), row_start
        self.x = x
        h1 = mux.rmsnorm_fwd(x, self.w["norm1"], s.eps, y=self._b("h1", s.hidden))
        nq, nk = s.heads * s.head_dim, s.kv_heads * s.head_dim
        if self.fused:     # q, k, v: column views of one GEMM's output
            qkv = self._lin_fwd("qkv", h1)
            q, k, v = qkv[:, :nq], qkv[:, nq:nq + nk], qkv[:, nq + nk:]
        else:
            q, k, v = self._lin_fwd("q", h1), self._lin_fwd("k", h1), self._lin_fwd("v", h1)
        mux.rope_(q, row_start, s.heads, s.head_dim, s.rope_base)
        mux.rope_(k, row_start, s.kv_heads, s.head_dim, s.rope_base)
        a, lse = mux.attn_fwd(q, k, v, row_start, s.heads, s.kv_heads, s.head_dim ** -0.5,
                              o=self._b("a", s.heads * s.head_dim), lse=self._b("lse", s.heads, torch.float32))
        o = self._lin_fwd("o", a)
        # residual add fused into the second RMSNorm: x2 = x + o, h2 = RMSNorm(x2)
        h2, x2 = mux.rmsnorm_fwd(o, self.w["norm2"], s.eps, y=self._b("h2", s.hidden), res=x,
                                 xsum=self._b("x2", s.hidden))
        if self.fused:
            gu = self._lin_fwd("gate_up", h2)
            g, u = gu[:, :s.ffn], gu[:, s.ffn:]
        else:
            g, u = self._lin_fwd("gate", h2), self._lin_fwd("up", h2)
        m = mux.swiglu_fwd(g, u, h=self._b("m", s.ffn))
        d = self._lin_fwd("down", m)
        self.saved = dict(h1=h1, q=q, k=k, v=v, a=a, lse=lse, x2=x2, h2=h2, g=g, u=u, m=m)
        return mux.add(x2, d, y=self._b("y", s.hidden))

    def backward(self, dy: torch.Tensor) -> torch.Tensor:
        s, sv = self.s, self.saved
        dm = self._lin_bwd("down", dy, sv["m"], self._b("dm", s.ffn))
        if self.fused:     # dgate|dup side by side: one dX GEMM, no partial to sum
            dgu = self._b("dgu", 2 * s.ffn)
            mux.swiglu_bwd(dm, sv["g"], sv["u"], dg=dgu[:, :s.ffn], du=dgu[:, s.ffn:])
            dh2 = self._lin_bwd("gate_up", dgu, sv["h2"], self._b("dh2", s.hidden))
            dh2u = None
        else:
            dg, du = mux.swiglu_bwd(dm, sv["g"], sv["u"], dg=self._b("dg", s.ffn), du=self._b("du", s.ffn))
            dh2 = self._lin_bwd("gate", dg, sv["h2"], self._b("dh2", s.hidden))
            dh2u = self._lin_bwd("up", du, sv["h2"], self._b("dh2u", s.hidden))
        # dx2 = RMSNorm'(x2)^T (dh2 + dh2u) + dy (residual): sum and residual fused into the norm
        dx2 = mux.rmsnorm_bwd(dh2, sv["x2"], self.w["norm2"], s.eps, dx=self._b("dx2", s.hidden), dy2=dh2u,
                              resid=dy)
        da = self._lin_bwd("o", dx2, sv["a"], self._b("da", s.heads * s.head_dim))
        need = mux.attn_workspace_size(self._rows, s.heads)
        ws = self._buf.get("attn_ws")
        if ws is None or ws.numel() < need:
            ws = self._buf["attn_ws"] = torch.empty(need, dtype=torch.uint8, device=dy.device)
        nq, nk = s.heads * s.head_dim, s.kv_heads * s.head_dim
        if self.fused:     # dq|dk|dv written side by side into the fused projection's dY
            dqkv = self._b("dqkv", nq + 2 * nk)
            outs = dict(dq=dqkv[:, :nq], dk=dqkv[:, nq:nq + nk], dv=dqkv[:, nq + nk:])
        else:
            outs = dict(dq=self._b("dq", nq), dk=self._b("dk", nk), dv=self._b("dv", nk))
        dq, dk, dv = mux.attn_bwd(da, sv["q"], sv["k"], sv["v"], sv["a"], sv["lse"], self.row_start, s.heads,
                                  s.kv_heads, s.head_dim ** -0.5, workspace=ws, **outs)
        mux.rope_(dq, self.row_start, s.heads, s.head_dim, s.rope_base, inverse=True)
        mux.rope_(dk, self.row_start, s.kv_heads, s.head_dim, s.rope_base, inverse=True)
        if self.fused:
            dh1 = self._lin_bwd("qkv", dqkv, sv["h1"], self._b("dh1", s.hidden))
            dh1k = dh1v = None
        else:
            dh1 = self._lin_bwd("q", dq, sv["h1"], self._b("dh1", s.hidden))
            dh1k = self._lin_bwd("k", dk, sv["h1"], self._b("dh1k", s.hidden))
            dh1v = self._lin_bwd("v", dv, sv["h1"], self._b("dh1v", s.hidden))
        # dx = RMSNorm'(x)^T (dh1 + dh1k + dh1v) + dx2 (residual), one fused pass
        dx = mux.rmsnorm_bwd(dh1, self.x, self.w["norm1"], s.eps, dx=self._b("dx", s.hidden), dy2=dh1k, dy3=dh1v,
                             resid=dx2)
        if self.overlap_grads:
            torch.cuda.current_stream().wait_stream(self._side)   # dA/dB complete with the returned dx
        return dx

    # kernel launches: forward = 2 norms (the second fused with the residual add) + 7 linears +
    # 2 RoPE + attention + swiglu + 1 residual add = 14; backward = 7 linears x (dX GEMM +
    # adapter-gradient kernel) + swiglu + 2 norms (gradient sums and residuals fused) +
    # attention (D, dV, dK, dQ) + 2 RoPE = 23
    LAUNCHES_FWD = 14
    LAUNCHES_BWD = 23
    # fused projections: forward 4 linears (11); backward 4 dX GEMMs + 7 gradient kernels (one per
    # slice) + swiglu + 2 norms + attention (4) + 2 RoPE (20)
    LAUNCHES_FWD_FUSED = 11
    LAUNCHES_BWD_FUSED = 20

    def launches(self):
        return ((self.LAUNCHES_FWD_FUSED, self.LAUNCHES_BWD_FUSED) if self.fused
                else (self.LAUNCHES_FWD, self.LAUNCHES_BWD))
