"""A tensor-parallel LLaMA decoder block with all seven linears multiplexed
(Megatron TP P:870 with sequence
parallelism P:205): the block of block.py split over the p ranks of a process
group, one process per GPU.

Per rank (R packed rows, hidden H, FFN F, p ranks; x_rows = this rank's
contiguous row block [R/p, H], the same segment table on every rank):

  forward                                            collectives
    h1_rows = RMSNorm(x_rows)                        (rows are local)
    h1 = AG(h1_rows)                       [R, H]    AG  (one, shared by q/k/v)
    q_p, k_p, v_p = column-parallel q/k/v  [R, Hq/p·d], [R, Hkv/p·d]
    RoPE(q_p, k_p); a_p = attention over this rank's heads (head-sharded,
      GQA groups stay on one rank: Hkv % p == 0)
    o_rows = RS(row-parallel o(a_p))       [R/p, H]  RS
    x2_rows = x_rows + o_rows; h2_rows = RMSNorm(x2_rows)   (one fused pass)
    h2 = AG(h2_rows)                       [R, H]    AG  (one, shared by gate/up)
    m_p = SwiGLU(gate_p(h2), up_p(h2))     [R, F/p]
    y_rows = x2_rows + RS(row-parallel down(m_p))    RS
  backward mirrors it: AG(dy) -> down dX -> SwiGLU' -> gate/up dX partials,
    summed, RS -> RMSNorm' (+ residual dy) -> AG -> o dX -> attention' ->
    RoPE^T -> q/k/v dX partials, summed, RS -> RMSNorm' (+ residual).
  Adapter gradients: column layers all-reduce dA_t (Gs_p is a partial sum over
  ranks), row layers all-reduce dB_t (Hs_p is) — tp.py.

Eight big collectives per block step ((p-1)/p · R · H · 2 bytes each), as
SURVEY §8(e) counts.  Every arithmetic step runs in the backend: `tp.MuxBackend`
(libmux kernels) on the product path, an fp64 oracle backend in the CPU tests.
"""
from __future__ import annotations

from dataclasses import dataclass
from typing import Dict, List, Sequence

import torch

from . import tp
from .block import LINEARS, BlockShape

COLUMN = ("q", "k", "v", "gate", "up")
ROW = ("o", "down")
# fused projections (include/mux.h "Fused projections"): q|k|v and gate|up as one column-sliced
# GEMM each, every task keeping its own adapter on every slice
FUSED = {"qkv": ("q", "k", "v"), "gate_up": ("gate", "up")}
FUSED_LINEARS = ("qkv", "o", "gate_up", "down")


@dataclass
class TPBlockShape(BlockShape):
    """BlockShape split over p ranks (heads and FFN columns)."""
    p: int = 1

    def __post_init__(self):
        if self.heads % self.p or self.kv_heads % self.p or self.ffn % self.p or self.hidden % self.p:
            raise ValueError(f"heads {self.heads}, kv_heads {self.kv_heads}, ffn {self.ffn} and hidden "
                             f"{self.hidden} must divide by p = {self.p}")


def shard_block(weights: Dict[str, torch.Tensor], adapters: Dict[str, Sequence], p: int, r: int, make_adapter):
    """This rank's shards: column-parallel q/k/v/gate/up (rows of W, rows of B_t), row-parallel o/down
    (columns of W, columns of A_t); the norm weights are replicated."""
    W, ads = {}, {}
    for name in LINEARS:
        fn = tp.shard_column if name in COLUMN else tp.shard_row
        W[name], ads[name] = fn(weights[name], adapters[name], p, r, make_adapter)
    W["norm1"], W["norm2"] = weights["norm1"], weights["norm2"]
    return W, ads


def shard_block_fused(weights: Dict[str, torch.Tensor], adapters: Dict[str, Sequence], p: int, r: int,
                      make_adapter):
    """shard_block with q|k|v and gate|up fused: W["qkv"] = this rank's q, k, v shards back to back
    (column slices col_off["qkv"]), adapters["qkv"][t] = [q, k, v shard of task t]; likewise gate_up.
    Returns (W, adapters, col_off)."""
    W, ads, col_off = {}, {}, {}
    for name, parts in FUSED.items():
        W[name], ads[name], col_off[name] = tp.shard_column_fused([weights[n] for n in parts],
                                                                  [adapters[n] for n in parts], p, r, make_adapter)
    for name in ROW:
        W[name], ads[name] = tp.shard_row(weights[name], adapters[name], p, r, make_adapter)
    W["norm1"], W["norm2"] = weights["norm1"], weights["norm2"]
    return W, ads, col_off


class TPDecoderBlock:
    """weights / adapters: this rank's shards (shard_block); backend: tp.MuxBackend or a test backend
    with the same op methods (fwd/bwd linears + rmsnorm/rope/attention/swiglu/add)."""

    def __init__(self, backend, shape: TPBlockShape, weights: Dict[str, torch.Tensor],
                 adapters: Dict[str, List], r_cap: int, group=None, nvls=None, col_off=None,
                 shared_shrink=False, shared_gs=False):
        """nvls: a tp.NvlsCollectives — every all-gather / reduce-scatter of the block inside the
        NVSwitch (NVLink SHARP) instead of NCCL.  col_off: the weights/adapters of shard_block_fused
        (q|k|v and gate|up as one column-sliced GEMM each).  shared_shrink: column layers shrink only
        this rank's rows and all-gather Hs (tp.py).  shared_gs: row layers do the same for Gs in the
        backward (built and parity-tested; no gain measured, profiles/r02_shared_gs_ab.jsonl)."""
        self.be, self.s, self.w, self.r_cap, self.group, self.nvls = backend, shape, weights, r_cap, group, nvls
        self.fused = col_off is not None
        self.lin = {}
        for name in (FUSED_LINEARS if self.fused else LINEARS):
            if name in ROW:
                self.lin[name] = tp.RowParallelMuxLinear(backend, weights[name], adapters[name], r_cap, group=group,
                                                         nvls=nvls, shared_shrink=shared_gs)
            else:
                self.lin[name] = tp.ColumnParallelMuxLinear(backend, weights[name], adapters[name], r_cap,
                                                            group=group, shared_shrink=shared_shrink,
                                                            col_off=col_off[name] if self.fused else None)

    def _ag(self, name, rows):
        return self.nvls.ag(name, rows) if self.nvls is not None else tp.all_gather_rows(rows, self.group)

    def _rs_sum(self, name, parts):
        """reduce-scatter over rows of the sum of this rank's partials (one collective for the layers
        that shared an input); with NVLS the last add writes straight into the multicast buffer."""
        out = None
        if self.nvls is not None:
            out = self.nvls.rs_buffer(name, parts[0].shape[0], parts[0].shape[1], parts[0].device)
        acc = parts[0]
        for i, x in enumerate(parts[1:]):
            acc = self.be.add(acc, x, out=out if i == len(parts) - 2 else None)
        return self.nvls.rs(name) if self.nvls is not None else tp.reduce_scatter_rows(acc, self.group)

    def _rs_single(self, name, layer, so, st, dY):
        """reduce-scatter of one fused projection's partial dX (no partials to sum): with NVLS the
        dX GEMM writes straight into the multicast-bound buffer."""
        out = None
        if self.nvls is not None:
            out = self.nvls.rs_buffer(name, dY.shape[0], layer.X.shape[1], dY.device)
        dXp = layer.backward_partial(so, st, dY, dX=out)[0]
        return self.nvls.rs(name) if self.nvls is not None else tp.reduce_scatter_rows(dXp, self.group)

    # ------------------------------------------------------------------ forward
    def forward(self, x_rows, seg_off, seg_task, row_start):
        s, be, lin = self.s, self.be, self.lin
        hq, hkv = s.heads // s.p, s.kv_heads // s.p
        self.seg_off, self.seg_task, self.row_start = seg_off, list(seg_task), row_start
        st = self.seg_task
        self.x_rows = x_rows
        h1 = self._ag("h1", be.rmsnorm_fwd(x_rows, self.w["norm1"], s.eps))
        if self.fused:     # one GEMM; q, k, v are column views of its output
            nq, nk = hq * s.head_dim, hkv * s.head_dim
            qkv = lin["qkv"].forward_full(seg_off, st, h1)
            q, k, v = qkv[:, :nq], qkv[:, nq:nq + nk], qkv[:, nq + nk:]
        else:
            q = lin["q"].forward_full(seg_off, st, h1)
            k = lin["k"].forward_full(seg_off, st, h1)
            v = lin["v"].forward_full(seg_off, st, h1)
        q = be.rope(q, row_start, hq, s.head_dim, s.rope_base)
        k = be.rope(k, row_start, hkv, s.head_dim, s.rope_base)
        a, lse = be.attn_fwd(q, k, v, row_start, hq, hkv, s.head_dim ** -0.5)
        o_rows = lin["o"].forward(seg_off, st, a)                       # RS inside
        h2_rows, x2_rows = be.rmsnorm_fwd(o_rows, self.w["norm2"], s.eps, res=x_rows)
        h2 = self._ag("h2", h2_rows)
        if self.fused:
            nf = s.ffn // s.p
            gu = lin["gate_up"].forward_full(seg_off, st, h2)
            g, u = gu[:, :nf], gu[:, nf:]
        else:
            g = lin["gate"].forward_full(seg_off, st, h2)
            u = lin["up"].forward_full(seg_off, st, h2)
        m = be.swiglu_fwd(g, u)
        d_rows = lin["down"].forward(seg_off, st, m)                    # RS inside
        self.saved = dict(q=q, k=k, v=v, a=a, lse=lse, x2_rows=x2_rows, g=g, u=u)
        return be.add(x2_rows, d_rows)

    # ------------------------------------------------------------------ backward
    def backward(self, dy_rows):
        s, be, lin, sv = self.s, self.be, self.lin, self.saved
        hq, hkv = s.heads // s.p, s.kv_heads // s.p
        so, st = self.seg_off, self.seg_task
        dm, _, _ = lin["down"].backward(so, st, dy_rows)                 # AG(dy) inside; AR(dB)
        if self.fused:     # dgate|dup written side by side: one dX GEMM, no partial sum
            nf = s.ffn // s.p
            dgu = be.empty(dm.shape[0], 2 * nf, dm)
            be.swiglu_bwd(dm, sv["g"], sv["u"], out=(dgu[:, :nf], dgu[:, nf:]))
            dh2_rows = self._rs_single("dh2", lin["gate_up"], so, st, dgu)
        else:
            dg, du = be.swiglu_bwd(dm, sv["g"], sv["u"])
            dh2_rows = self._rs_sum("dh2", [lin["gate"].backward_partial(so, st, dg)[0],
                                            lin["up"].backward_partial(so, st, du)[0]])
        if self.nvls is not None:
            self.nvls.release("h2")          # gate/up backward were the last readers of the gathered h2
        dx2_rows = be.rmsnorm_bwd(dh2_rows, sv["x2_rows"], self.w["norm2"], s.eps, resid=dy_rows)
        da, _, _ = lin["o"].backward(so, st, dx2_rows)                   # AG(dx2) inside; AR(dB)
        out = None
        if self.fused:     # dq|dk|dv written side by side into the fused projection's dY
            nq, nk = hq * s.head_dim, hkv * s.head_dim
            dqkv = be.empty(da.shape[0], nq + 2 * nk, da)
            out = (dqkv[:, :nq], dqkv[:, nq:nq + nk], dqkv[:, nq + nk:])
        dq, dk, dv = be.attn_bwd(da, sv["q"], sv["k"], sv["v"], sv["a"], sv["lse"], self.row_start, hq, hkv,
                                 s.head_dim ** -0.5, out=out)
        dq = be.rope(dq, self.row_start, hq, s.head_dim, s.rope_base, inverse=True)   # in place
        dk = be.rope(dk, self.row_start, hkv, s.head_dim, s.rope_base, inverse=True)
        if self.fused:
            dh1_rows = self._rs_single("dh1", lin["qkv"], so, st, dqkv)
        else:
            dh1_rows = self._rs_sum("dh1", [lin["q"].backward_partial(so, st, dq)[0],
                                            lin["k"].backward_partial(so, st, dk)[0],
                                            lin["v"].backward_partial(so, st, dv)[0]])
        if self.nvls is not None:
            self.nvls.release("h1")
        return be.rmsnorm_bwd(dh1_rows, self.x_rows, self.w["norm1"], s.eps, resid=dx2_rows)

    def adapter_grads(self):
        """{linear: ([dA_t], [dB_t])} of this rank (after backward), per original linear (a fused
        projection's per-slice gradients are split back to q, k, v / gate, up)."""
        if not self.fused:
            return {n: (self.lin[n].dA, self.lin[n].dB) for n in LINEARS}
        out = {n: (self.lin[n].dA, self.lin[n].dB) for n in ROW}
        for f, parts in FUSED.items():
            dA, dB = self.lin[f].dA, self.lin[f].dB
            for i, n in enumerate(parts):
                out[n] = ([row[i] for row in dA], [row[i] for row in dB])
        return out

    # libmux launches per step at world p > 1 (for the bench's gpu_launches): forward = 2 norms +
    # 7 fused linears + 2 RoPE + attention + SwiGLU + add = 14 (+ 2 owner-side sums with fused RS);
    # backward = 7 dX GEMMs + 7 gradient kernels + SwiGLU + 2 norms + attention (4) + 2 RoPE + 3 adds.
    # Fused projections: forward 4 linears (12); backward 4 dX GEMMs + 7 gradient kernels (one per
    # slice) + SwiGLU + 2 norms + attention (4) + 2 RoPE, no adds (20).
    LAUNCHES_FWD = 14
    LAUNCHES_BWD = 26
    LAUNCHES_FWD_FUSED = 12
    LAUNCHES_BWD_FUSED = 20

    def launches(self):
        return ((self.LAUNCHES_FWD_FUSED, self.LAUNCHES_BWD_FUSED) if self.fused
                else (self.LAUNCHES_FWD, self.LAUNCHES_BWD))
