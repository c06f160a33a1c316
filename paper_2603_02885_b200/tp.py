"""Tensor parallelism of the frozen backbone for the multiplexed LoRA linear
(Megatron column/row split, with sequence
parallelism).  One process per GPU; torch.distributed process groups
(NCCL on B200s) carry the collectives; every rank's compute is one
mux_linear_fwd / mux_linear_bwd call on its shard.

Shard placement (reading Q15 in DESIGN.md):
  column-parallel (q, k, v, gate, up): W_p = W[N/p rows], A_t replicated,
      B_{t,p} = B_t[N/p rows].  fwd: AG(X) -> local fwd -> Y_p [R, N/p].
      bwd: local bwd -> RS(dX_partial) -> dX [R/p, K];  AR(dA_t).
      (Gs_p = s dY_p B_{t,p} is a partial sum over ranks; dA_t = Gs^T X is
      linear in Gs, so the per-rank dA_t are summed.)
  row-parallel (o, down): W_p = W[:, K/p cols], A_{t,p} = A_t[:, K/p cols],
      B_t replicated.  fwd: local fwd -> RS(Y_partial) -> Y [R/p, N]
      (H = sum_p X_p A_{t,p}^T enters linearly, so the LoRA term folds into
      the same reduce-scatter).  bwd: AG(dY) -> local bwd -> dX_p [R, K/p];
      AR(dB_t) (dB_t = dY^T Hs is linear in Hs = sum_p Hs_p).
Rows are split into p equal contiguous blocks (sequence parallel); R must be
a multiple of p.  Segment offsets are global (the same on every rank).

The per-rank compute is injected as a `backend` with
  fwd(seg_off, seg_task, adapters, X, W, r_cap) -> (Y, Hs)
  bwd(seg_off, seg_task, adapters, dY, X, W, Hs, r_cap) -> (dX, [dA_t], [dB_t])
`MuxBackend` is the product (libmux through the binding); tests inject the
fp64 oracle to check the collective orchestration on CPU with gloo.

Fused reduce-scatter (`fused_rs=True` on the layer classes, NCCL groups with
torch symmetric memory): the row-parallel forward and the column-parallel dX
GEMM store their output tiles straight into the owner rank's receive slot
over NVLink (mux_linear_fwd_rs / mux_linear_bwd_dx_rs) and the owner sums the
slots (mux_rs_reduce) — no separate collective launch, and the transfer of a
tile overlaps the GEMM of the next ones.  `FusedRs` allocates the peer
buffers once per (layer, direction).
"""
from __future__ import annotations

from dataclasses import dataclass
from typing import List, Optional, Sequence

import torch
import torch.distributed as dist


# ------------------------------------------------------------------ collectives
def _flat(grads):
    """[g_t] or [[g_{t,s}]] (a fused projection's per-slice gradients) -> flat list."""
    out = []
    for g in grads:
        if isinstance(g, (list, tuple)):
            out.extend(g)
        else:
            out.append(g)
    return out


def _world(group=None):
    return dist.get_world_size(group), dist.get_rank(group)


def all_gather_rows(x: torch.Tensor, group=None) -> torch.Tensor:
    p, _ = _world(group)
    out = torch.empty((x.shape[0] * p,) + tuple(x.shape[1:]), dtype=x.dtype, device=x.device)
    if dist.get_backend(group) == "nccl":
        dist.all_gather_into_tensor(out, x.contiguous(), group=group)
    else:
        parts = list(out.chunk(p, 0))
        dist.all_gather(parts, x.contiguous(), group=group)
        out = torch.cat(parts, 0)
    return out


def reduce_scatter_rows(x: torch.Tensor, group=None) -> torch.Tensor:
    p, r = _world(group)
    rows = x.shape[0] // p
    if dist.get_backend(group) == "nccl":
        out = torch.empty((rows,) + tuple(x.shape[1:]), dtype=x.dtype, device=x.device)
        dist.reduce_scatter_tensor(out, x.contiguous(), group=group)
        return out
    y = x.clone()
    dist.all_reduce(y, group=group)
    return y[r * rows:(r + 1) * rows].contiguous()


def all_reduce_(x: torch.Tensor, group=None) -> torch.Tensor:
    dist.all_reduce(x, group=group)
    return x


class NvlsCollectives:
    """All-gather / reduce-scatter over rows reduced or broadcast inside the NVSwitch (NVLink SHARP,
    NEXT-1; libmux mux_nvls_*), one multicast-bound buffer per (name, shape).  `ag(name, x_rows)`
    returns the gathered [R, cols] rows (valid until `release(name)`); `rs_buffer(name, R, cols)` is
    the [R, cols] buffer a GEMM writes its partial into, `rs(name, out)` reduces it into this rank's
    rows.  `ctas` caps the CTAs of each collective (P:791-796 uses 8 with NVLink SHARP)."""

    def __init__(self, group=None, ctas: int = 8):
        self.group, self.ctas = group, ctas
        self.bufs = {}

    def _get(self, name, rows, cols, device):
        b = self.bufs.get(name)
        if b is None or b.rows != rows or b.cols != cols:
            from .nvls import NvlsBuffer
            b = self.bufs[name] = NvlsBuffer(self.group, rows, cols, device)
        return b

    def ag(self, name, x_rows):
        b = self._get(name, x_rows.shape[0], x_rows.shape[1], x_rows.device)
        return b.all_gather(x_rows, self.ctas)

    def release(self, name):
        self.bufs[name].release()

    def rs_buffer(self, name, R, cols, device):
        p = dist.get_world_size(self.group) if dist.is_initialized() else 1
        return self._get(name, R // p, cols, device).uc

    def rs(self, name, out=None):
        b = self.bufs[name]
        if out is None:
            out = torch.empty(b.rows, b.cols, dtype=torch.bfloat16, device=b.uc.device)
        return b.reduce_scatter(out, self.ctas)


class FusedRs:
    """Receive buffers and flags of mux's fused GEMM -> reduce-scatter, allocated with torch
    symmetric memory (every rank maps every rank's buffers over NVLink)."""

    def __init__(self, group, rows_per_rank: int, cols: int, device, exchange=None):
        """`exchange(recv, flags) -> (recv_ptrs, flag_ptrs)` maps every rank's buffers by other
        means (e.g. CUDA IPC handles); default: torch symmetric memory rendezvous."""
        from . import mux
        self.mux = mux
        self.world, self.rank = _world(group)
        self.rows = rows_per_rank
        self.cols = cols
        n_recv, n_flags = self.world * rows_per_rank * cols, mux.rs_flags_elems(self.world)
        if exchange is None:
            import torch.distributed._symmetric_memory as symm
            gname = group.group_name if group is not None else dist.group.WORLD.group_name
            self.recv = symm.empty(n_recv, dtype=torch.bfloat16, device=device)
            self.flags = symm.empty(n_flags, dtype=torch.int64, device=device)
            self.flags.zero_()
            h1 = symm.rendezvous(self.recv, gname)
            h2 = symm.rendezvous(self.flags, gname)
            self.recv_ptrs = list(h1.buffer_ptrs)
            self.flag_ptrs = list(h2.buffer_ptrs)
        else:
            self.recv = torch.zeros(n_recv, dtype=torch.bfloat16, device=device)
            self.flags = torch.zeros(n_flags, dtype=torch.int64, device=device)
            self.recv_ptrs, self.flag_ptrs = exchange(self.recv, self.flags)
        torch.cuda.synchronize()
        dist.barrier(group)
        self.seq = 0

    def next(self):
        self.seq += 1
        return self.mux.make_rs(self.world, self.rank, self.rows, self.seq, self.recv_ptrs, self.flag_ptrs)


# ------------------------------------------------------------------ backends
class MuxBackend:
    """libmux kernels (the product path).  Output buffers and the (zeroed once,
    reused) linear workspace are cached per layer key, so a step allocates
    nothing."""

    def __init__(self):
        from . import mux
        self.mux = mux
        self.cache = {}

    def _buf(self, key, shape, dtype, device, zero=False):
        t = self.cache.get(key)
        if t is None or tuple(t.shape) != tuple(shape):
            t = (torch.zeros if zero else torch.empty)(shape, dtype=dtype, device=device)
            self.cache[key] = t
        return t

    def _ws(self, W, X, seg_task, r_cap, col_off=None):
        R, K = X.shape
        S = 1 if col_off is None else len(col_off) - 1
        n = self.mux.linear_workspace_size(len(seg_task), R, K, W.shape[0], r_cap * S)
        return self._buf(("ws", W.data_ptr()), (n,), torch.uint8, X.device, zero=True)

    @staticmethod
    def _hs_cols(r_cap, col_off):
        return r_cap * (1 if col_off is None else len(col_off) - 1)

    # col_off (fused projections, include/mux.h): column slices of W / Y, adapters[t][s] per task
    def fwd(self, seg_off, seg_task, adapters, X, W, r_cap, Y=None, col_off=None):
        R = X.shape[0]
        if Y is None:
            Y = self._buf(("Y", W.data_ptr()), (R, W.shape[0]), torch.bfloat16, X.device)
        Hs = self._buf(("Hs", W.data_ptr()), (R, self._hs_cols(r_cap, col_off)), torch.bfloat16, X.device)
        ws = self._ws(W, X, seg_task, r_cap, col_off)
        if col_off is not None:
            return self.mux.linear_fwd_sliced(seg_off, seg_task, adapters, X, W, col_off, r_cap, Y=Y, Hs=Hs,
                                              workspace=ws)
        return self.mux.linear_fwd(seg_off, seg_task, adapters, X, W, r_cap, Y=Y, Hs=Hs, workspace=ws)

    def shrink(self, seg_off, seg_task, adapters, X, W, r_cap, row_begin, row_end, col_off=None):
        """Hs rows [row_begin, row_end) of the full (gathered) X only (mux_linear_shrink)."""
        Hs = self._buf(("Hs", W.data_ptr()), (X.shape[0], self._hs_cols(r_cap, col_off)), torch.bfloat16, X.device)
        ws = self._ws(W, X, seg_task, r_cap, col_off)
        if col_off is not None:
            self.mux.linear(self.mux.OP_SHRINK, seg_off, seg_task, adapters, col_off, X.shape[1], W.shape[0], r_cap,
                            X.shape[0], X=X, Hs=Hs, row_begin=row_begin, row_end=row_end, workspace=ws)
            return Hs
        return self.mux.linear_shrink(seg_off, seg_task, adapters, X, W.shape[0], r_cap, row_begin, row_end, Hs=Hs,
                                      workspace=ws)

    def fwd_hs(self, seg_off, seg_task, adapters, X, W, Hs, r_cap, col_off=None):
        """Forward with the shrink given (mux_linear_fwd_hs): no shrink tiles in the GEMM."""
        Y = self._buf(("Y", W.data_ptr()), (X.shape[0], W.shape[0]), torch.bfloat16, X.device)
        ws = self._ws(W, X, seg_task, r_cap, col_off)
        if col_off is not None:
            self.mux.linear(self.mux.OP_FWD_HS, seg_off, seg_task, adapters, col_off, X.shape[1], W.shape[0], r_cap,
                            X.shape[0], X=X, W=W, Y=Y, Hs=Hs, workspace=ws)
            return Y
        return self.mux.linear_fwd_hs(seg_off, seg_task, adapters, X, W, Hs, r_cap, Y=Y, workspace=ws)

    def shrink_bwd(self, seg_off, seg_task, adapters, dY, W, r_cap, row_begin, row_end, col_off=None):
        """Gs rows [row_begin, row_end) of the full (gathered) dY only (mux_linear MUX_OP_SHRINK_BWD)."""
        R = dY.shape[0]
        Gs = self._buf(("Gs", W.data_ptr()), (R, self._hs_cols(r_cap, col_off)), torch.bfloat16, dY.device)
        n = self.mux.linear_workspace_size(len(seg_task), R, W.shape[1], W.shape[0], self._hs_cols(r_cap, col_off))
        ws = self._buf(("ws", W.data_ptr()), (n,), torch.uint8, dY.device, zero=True)
        return self.mux.linear_shrink_bwd(seg_off, seg_task, adapters, dY, W.shape[1], r_cap, row_begin, row_end,
                                          Gs=Gs, col_off=col_off, workspace=ws)

    def bwd(self, seg_off, seg_task, adapters, dY, X, W, Hs, r_cap, dX=None, col_off=None, Gs=None):
        """Gs: the shrink of dY given (all-gathered rows; no shrink tiles in the dX GEMM)."""
        if dX is None:
            dX = self._buf(("dX", W.data_ptr()), tuple(X.shape), torch.bfloat16, X.device)
        ws = self._ws(W, X, seg_task, r_cap, col_off)
        if Gs is not None:
            dX = self.mux.linear_bwd_gs(seg_off, seg_task, adapters, dY, X, W, Hs, Gs, r_cap, dX=dX, col_off=col_off,
                                        workspace=ws)
            if col_off is not None:
                return dX, [[a.dA for a in row] for row in adapters], [[a.dB for a in row] for row in adapters]
            return dX, [a.dA for a in adapters], [a.dB for a in adapters]
        if col_off is not None:
            dX = self.mux.linear_bwd_sliced(seg_off, seg_task, adapters, dY, X, W, Hs, col_off, r_cap, dX=dX,
                                            workspace=ws)
            return dX, [[a.dA for a in row] for row in adapters], [[a.dB for a in row] for row in adapters]
        dX = self.mux.linear_bwd(seg_off, seg_task, adapters, dY, X, W, Hs, r_cap, dX=dX, workspace=ws)
        return dX, [a.dA for a in adapters], [a.dB for a in adapters]

    # ---- decoder-block ops (tp_block.py): libmux kernels, fresh outputs (caching allocator)
    def rmsnorm_fwd(self, x, w, eps, res=None):
        return self.mux.rmsnorm_fwd(x, w, eps, res=res)

    def rmsnorm_bwd(self, dy, x, w, eps, resid=None):
        return self.mux.rmsnorm_bwd(dy, x, w, eps, resid=resid)

    def rope(self, x, row_start, heads, head_dim, base, inverse=False):
        return self.mux.rope_(x, row_start, heads, head_dim, base, inverse=inverse)

    def attn_fwd(self, q, k, v, row_start, heads, kv_heads, scale):
        return self.mux.attn_fwd(q, k, v, row_start, heads, kv_heads, scale)

    def attn_bwd(self, dO, q, k, v, o, lse, row_start, heads, kv_heads, scale, out=None):
        """out: (dq, dk, dv) views to write (e.g. column slices of a fused projection's dY)."""
        ws = self._buf(("attn_ws", q.shape[0], heads), (self.mux.attn_workspace_size(q.shape[0], heads),),
                       torch.uint8, q.device)
        dq, dk, dv = out if out is not None else (None, None, None)
        return self.mux.attn_bwd(dO, q, k, v, o, lse, row_start, heads, kv_heads, scale, dq=dq, dk=dk, dv=dv,
                                 workspace=ws)

    def swiglu_fwd(self, g, u):
        return self.mux.swiglu_fwd(g, u)

    def swiglu_bwd(self, dh, g, u, out=None):
        """out: (dg, du) views to write."""
        dg, du = out if out is not None else (None, None)
        return self.mux.swiglu_bwd(dh, g, u, dg=dg, du=du)

    def empty(self, rows, cols, like):
        return torch.empty(rows, cols, dtype=torch.bfloat16, device=like.device)

    def add(self, a, b, out=None):
        return self.mux.add(a, b, y=out)

    # fused GEMM -> reduce-scatter (peer stores + owner-side sum; see FusedRs)
    rs_exchange = None  # optional buffer-mapping hook for FusedRs (default: symmetric memory)

    def _rs_for(self, lay, rows, cols, device):
        if lay._rs is None or lay._rs.rows != rows or lay._rs.cols != cols:
            lay._rs = FusedRs(lay.group, rows, cols, device, exchange=self.rs_exchange)
        return lay._rs

    # fused all-gather (copy-engine push + per-row-block waits in the GEMM producer)
    def _ag_for(self, lay, attr, rows, cols, device):
        cur = getattr(lay, attr, None)
        if cur is None or cur.rows != rows or cur.cols != cols:
            cur = FusedRs(lay.group, rows, cols, device, exchange=self.rs_exchange)
            setattr(lay, attr, cur)
        return cur

    def _push(self, ag, rows_t):
        """Push this rank's rows to every rank on the copy stream.  Returns the event that marks
        the end of all pushes: the source must not be rewritten (or freed) before it, so the
        caller makes its compute stream wait on it when it releases the gather (by then every
        push has long finished, so the wait costs nothing and keeps the overlap)."""
        if getattr(self, "copy_stream", None) is None:
            self.copy_stream = torch.cuda.Stream()
        ev = torch.cuda.Event()
        ev.record()
        self.copy_stream.wait_event(ev)           # this rank's rows are ready
        self.mux.ag_push(ag, rows_t, stream=self.copy_stream)
        rows_t.record_stream(self.copy_stream)    # the allocator keeps the block until the pushes end
        done = torch.cuda.Event()
        done.record(self.copy_stream)
        return done

    def fwd_ag(self, lay, seg_off, seg_task, x_rows):
        p, _ = _world(lay.group)
        rows, K = x_rows.shape
        if lay._ag_held is not None:
            # the previous forward's gather is still held for its backward: pushing again would
            # wait forever for this rank's own release (and the GEMM would trap on the flags)
            raise RuntimeError("fused_ag: forward called again before the backward of the previous call; "
                               "call release_ag() first for forward-only use")
        fb = self._ag_for(lay, "_ag", rows, K, x_rows.device)
        ag = fb.next()
        lay._ag_pushed = self._push(ag, x_rows)
        R, N = rows * p, lay.W.shape[0]
        co = getattr(lay, "col_off", None)
        Y = self._buf(("Y", lay.W.data_ptr()), (R, N), torch.bfloat16, x_rows.device)
        Hs = self._buf(("Hs", lay.W.data_ptr()), (R, self._hs_cols(lay.r_cap, co)), torch.bfloat16, x_rows.device)
        ws = self._ws(lay.W, fb.recv.view(R, K), seg_task, lay.r_cap, co)
        if co is not None:
            self.mux.linear(self.mux.OP_FWD, seg_off, seg_task, lay.ads, co, K, N, lay.r_cap, R, W=lay.W, Y=Y, Hs=Hs,
                            ag=ag, workspace=ws)
        else:
            self.mux.linear_fwd_ag(ag, seg_off, seg_task, lay.ads, K, lay.W, lay.r_cap, Y=Y, Hs=Hs, workspace=ws)
        lay._ag_held = ag                         # released after the backward re-read X
        return Y, Hs, fb.recv.view(R, K)

    def bwd_ag(self, lay, seg_off, seg_task, dy_rows):
        p, _ = _world(lay.group)
        rows, N = dy_rows.shape
        fb = self._ag_for(lay, "_ag", rows, N, dy_rows.device)
        ag = fb.next()
        pushed = self._push(ag, dy_rows)
        X = lay.X
        dX = self._buf(("dX", lay.W.data_ptr()), tuple(X.shape), torch.bfloat16, X.device)
        self.mux.linear_bwd_ag(ag, seg_off, seg_task, lay.ads, X, lay.W, lay.Hs, lay.r_cap, dX=dX,
                               workspace=self._ws(lay.W, X, seg_task, lay.r_cap))
        torch.cuda.current_stream().wait_event(pushed)   # dy_rows may be rewritten after this point
        self.mux.ag_release(ag)                   # dY fully consumed (dX GEMM + gradients)
        return dX, [a.dA for a in lay.ads], [a.dB for a in lay.ads]

    def fwd_rs(self, lay, seg_off, seg_task, X):
        p, _ = _world(lay.group)
        R, N = X.shape[0], lay.W.shape[0]
        rs = self._rs_for(lay, R // p, N, X.device).next()
        Hs = self._buf(("Hs", lay.W.data_ptr()), (R, lay.r_cap), torch.bfloat16, X.device)
        self.mux.linear_fwd_rs(rs, seg_off, seg_task, lay.ads, X, lay.W, lay.r_cap, Hs=Hs,
                               workspace=self._ws(lay.W, X, seg_task, lay.r_cap))
        Y = self._buf(("Yrs", lay.W.data_ptr()), (R // p, N), torch.bfloat16, X.device)
        return self.mux.rs_reduce(rs, Y), Hs

    def bwd_rs(self, lay, seg_off, seg_task, dY):
        p, _ = _world(lay.group)
        X = lay.X
        R, K = X.shape
        rs = self._rs_for(lay, R // p, K, X.device).next()
        co = getattr(lay, "col_off", None)
        ws = self._ws(lay.W, X, seg_task, lay.r_cap, co)
        dX = self._buf(("dXrs", lay.W.data_ptr()), (R // p, K), torch.bfloat16, X.device)
        if co is not None:
            N = lay.W.shape[0]
            self.mux.linear(self.mux.OP_BWD_DX, seg_off, seg_task, lay.ads, co, K, N, lay.r_cap, R, X=X, W=lay.W,
                            dY=dY, Hs=lay.Hs, rs=rs, workspace=ws)
            self.mux.linear_bwd_sliced(seg_off, seg_task, lay.ads, dY, X, lay.W, lay.Hs, co, lay.r_cap, want_dx=False,
                                       workspace=ws, part=self.mux.BWD_GRADS)
            return (self.mux.rs_reduce(rs, dX), [[a.dA for a in row] for row in lay.ads],
                    [[a.dB for a in row] for row in lay.ads])
        self.mux.linear_bwd_dx_rs(rs, seg_off, seg_task, lay.ads, dY, X, lay.W, lay.Hs, lay.r_cap, ws)
        self.mux.linear_bwd(seg_off, seg_task, lay.ads, dY, X, lay.W, lay.Hs, lay.r_cap, workspace=ws,
                            part=self.mux.BWD_GRADS)
        return self.mux.rs_reduce(rs, dX), [a.dA for a in lay.ads], [a.dB for a in lay.ads]


@dataclass
class ShardAdapter:
    """One task's adapter shard on this rank (same fields as mux.Adapter)."""
    A: Optional[torch.Tensor]
    B: Optional[torch.Tensor]
    rank: int
    scale: float
    dA: Optional[torch.Tensor] = None
    dB: Optional[torch.Tensor] = None


def shard_column(W: torch.Tensor, adapters: Sequence, p: int, r: int, make_adapter):
    """Column-parallel shard of (W [N,K], adapters) for rank r of p."""
    N = W.shape[0]
    n = N // p
    Wp = W[r * n:(r + 1) * n].contiguous()
    ads = [make_adapter(a.A, None if a.B is None else a.B[r * n:(r + 1) * n], a.rank, a.scale) for a in adapters]
    return Wp, ads


def shard_column_fused(Ws: Sequence[torch.Tensor], adapter_lists: Sequence[Sequence], p: int, r: int, make_adapter):
    """Column-parallel shard of a fused projection (e.g. q|k|v): rank r's rows of every W_s back to
    back, col_off = the slice offsets inside that shard, and per task the list of its slice shards
    (adapters[t][s]).  Returns (W_p, adapters, col_off)."""
    parts, per_slice, col_off = [], [], [0]
    for W, ads in zip(Ws, adapter_lists):
        Wp, ap = shard_column(W, ads, p, r, make_adapter)
        parts.append(Wp)
        per_slice.append(ap)
        col_off.append(col_off[-1] + Wp.shape[0])
    T = len(adapter_lists[0])
    return torch.cat(parts, 0).contiguous(), [[per_slice[s][t] for s in range(len(Ws))] for t in range(T)], col_off


def shard_row(W: torch.Tensor, adapters: Sequence, p: int, r: int, make_adapter):
    """Row-parallel shard of (W [N,K], adapters) for rank r of p."""
    K = W.shape[1]
    k = K // p
    Wp = W[:, r * k:(r + 1) * k].contiguous()
    ads = [make_adapter(None if a.A is None else a.A[:, r * k:(r + 1) * k].contiguous(), a.B, a.rank, a.scale)
           for a in adapters]
    return Wp, ads


class ColumnParallelMuxLinear:
    """shared_shrink: A_t is replicated, so Hs = s_t X A_t^T is the same on every rank.  Instead of
    each rank recomputing all T rows of it inside its fused GEMM (shrink tiles over the gathered X),
    each rank shrinks only its own R/p rows (mux_linear_shrink), the Hs rows are all-gathered
    (T x r_cap, ~1/(K/r_cap) of X's gather) and the GEMM runs without shrink tiles
    (mux_linear_fwd_hs).  R/p must be a multiple of 256 (pair row blocks).  It applies to the
    NCCL all-gather path; with fused_ag the gathered rows arrive inside the GEMM, which then
    computes the shrink itself."""

    def __init__(self, backend, W_shard, adapters_shard, r_cap, group=None, fused_rs=False, fused_ag=False,
                 shared_shrink=False, nvls=None, col_off=None):
        """col_off: a fused projection (q|k|v, gate|up; include/mux.h "Fused projections"): this rank's
        W_shard rows are the slices' shards back to back, col_off their column offsets, and
        adapters_shard[t][s] task t's adapter shard on slice s."""
        self.be, self.W, self.ads, self.r_cap, self.group = backend, W_shard, adapters_shard, r_cap, group
        self.fused_rs, self.fused_ag, self.shared_shrink = fused_rs, fused_ag, shared_shrink
        self.col_off = None if col_off is None else list(col_off)
        self.kw = {} if col_off is None else {"col_off": self.col_off}
        self.nvls = nvls    # NvlsCollectives: AG(X) and RS(dX) inside the NVSwitch
        self._rs = self._ag = self._ag_held = self._ag_pushed = None
        self._nvls_held = False

    def forward(self, seg_off, seg_task, x_rows):
        """x_rows [R/p, K] (this rank's row block) -> Y_p [R, N/p]."""
        if self.fused_ag:
            Y, self.Hs, self.X = self.be.fwd_ag(self, seg_off, seg_task, x_rows)
            return Y
        if self.nvls is not None:
            if self._nvls_held:
                raise RuntimeError("nvls: forward called again before the backward of the previous call; "
                                   "call release_ag() first for forward-only use")
            self.X = self.nvls.ag(("ag", id(self)), x_rows)
            self._nvls_held = True
            Y, self.Hs = self.be.fwd(seg_off, seg_task, self.ads, self.X, self.W, self.r_cap, **self.kw)
            return Y
        self.X = all_gather_rows(x_rows, self.group)
        if self.shared_shrink:
            return self._fwd_shared_shrink(seg_off, seg_task, x_rows.shape[0])
        Y, self.Hs = self.be.fwd(seg_off, seg_task, self.ads, self.X, self.W, self.r_cap, **self.kw)
        return Y

    def _fwd_shared_shrink(self, seg_off, seg_task, rows_p):
        r0 = rows_p * _world(self.group)[1]
        Hs = self.be.shrink(seg_off, seg_task, self.ads, self.X, self.W, self.r_cap, r0, r0 + rows_p, **self.kw)
        self.Hs = all_gather_rows(Hs[r0:r0 + rows_p].contiguous(), self.group)
        return self.be.fwd_hs(seg_off, seg_task, self.ads, self.X, self.W, self.Hs, self.r_cap, **self.kw)

    def forward_full(self, seg_off, seg_task, X):
        """X [R, K] already gathered (one all-gather shared by several column layers reading the
        same input, e.g. q/k/v or gate/up) -> Y_p [R, N/p].  With shared_shrink, the shrink of this
        rank's rows is all-gathered instead of recomputed (as in forward)."""
        self.X = X
        if self.shared_shrink:
            return self._fwd_shared_shrink(seg_off, seg_task, X.shape[0] // _world(self.group)[0])
        Y, self.Hs = self.be.fwd(seg_off, seg_task, self.ads, X, self.W, self.r_cap, **self.kw)
        return Y

    def _reduce_dA(self, dA):
        for g in _flat(dA):
            if g is not None:
                all_reduce_(g, self.group)

    def backward_partial(self, seg_off, seg_task, dY_cols, dX=None):
        """dY_p [R, N/p] -> this rank's partial dX [R, K] (the caller sums the partials of the layers
        that shared the input, then reduce-scatters once; dX = an output buffer or None); dA_t
        all-reduced, dB_{t,p} local."""
        dXp, dA, dB = self.be.bwd(seg_off, seg_task, self.ads, dY_cols, self.X, self.W, self.Hs, self.r_cap,
                                  dX=dX, **self.kw)
        self._reduce_dA(dA)
        self.dA, self.dB = dA, dB
        return dXp, dA, dB

    def backward(self, seg_off, seg_task, dY_cols):
        """dY_p [R, N/p] -> dX rows [R/p, K]; dA_t all-reduced, dB_{t,p} local."""
        if self.fused_rs:
            dX_rows, dA, dB = self.be.bwd_rs(self, seg_off, seg_task, dY_cols)
        elif self.nvls is not None:   # the partial dX goes straight into the multicast-bound buffer
            R, K = self.X.shape
            buf = self.nvls.rs_buffer(("rs", id(self)), R, K, self.X.device)
            _, dA, dB = self.be.bwd(seg_off, seg_task, self.ads, dY_cols, self.X, self.W, self.Hs, self.r_cap,
                                    dX=buf, **self.kw)
            self.release_ag()
            dX_rows = self.nvls.rs(("rs", id(self)))
        else:
            dXp, dA, dB = self.be.bwd(seg_off, seg_task, self.ads, dY_cols, self.X, self.W, self.Hs, self.r_cap,
                                      **self.kw)
            dX_rows = None
        self._reduce_dA(dA)
        self.dA, self.dB = dA, dB
        self.release_ag()
        return (reduce_scatter_rows(dXp, self.group) if dX_rows is None else dX_rows), dA, dB

    def release_ag(self):
        """The gathered X is no longer needed (after the backward): its owners may push again."""
        if self._nvls_held:
            self.nvls.release(("ag", id(self)))
            self._nvls_held = False
        if self._ag_held is not None:
            if self._ag_pushed is not None:   # the pushed source rows may be rewritten after this point
                torch.cuda.current_stream().wait_event(self._ag_pushed)
                self._ag_pushed = None
            self.be.mux.ag_release(self._ag_held)
            self._ag_held = None


class RowParallelMuxLinear:
    """shared_shrink: B_t is replicated and every rank holds the full gathered dY, so Gs = s_t dY B_t is the
    same on every rank: each rank shrinks only its own R/p rows (MUX_OP_SHRINK_BWD), the Gs rows are
    all-gathered (T x r_cap) and the dX GEMM runs without shrink tiles (the backward mirror of
    ColumnParallelMuxLinear's shared_shrink; R/p a multiple of 256)."""

    def __init__(self, backend, W_shard, adapters_shard, r_cap, group=None, fused_rs=False, fused_ag=False,
                 nvls=None, shared_shrink=False):
        self.be, self.W, self.ads, self.r_cap, self.group = backend, W_shard, adapters_shard, r_cap, group
        self.fused_rs, self.fused_ag, self.shared_shrink = fused_rs, fused_ag, shared_shrink
        self.nvls = nvls    # NvlsCollectives: RS(Y) and AG(dY) inside the NVSwitch
        self._rs = self._ag = None

    def forward(self, seg_off, seg_task, x_cols):
        """x_cols [R, K/p] (this rank's column shard) -> Y rows [R/p, N]."""
        self.X = x_cols
        if self.fused_rs:
            Y_rows, self.Hs = self.be.fwd_rs(self, seg_off, seg_task, x_cols)
            return Y_rows
        if self.nvls is not None:     # the partial Y goes straight into the multicast-bound buffer
            buf = self.nvls.rs_buffer(("rs", id(self)), x_cols.shape[0], self.W.shape[0], x_cols.device)
            _, self.Hs = self.be.fwd(seg_off, seg_task, self.ads, x_cols, self.W, self.r_cap, Y=buf)
            return self.nvls.rs(("rs", id(self)))
        Yp, self.Hs = self.be.fwd(seg_off, seg_task, self.ads, x_cols, self.W, self.r_cap)
        return reduce_scatter_rows(Yp, self.group)

    def backward(self, seg_off, seg_task, dy_rows):
        """dY rows [R/p, N] -> dX_p [R, K/p]; dB_t all-reduced, dA_{t,p} local."""
        if self.fused_ag:
            dXp, dA, dB = self.be.bwd_ag(self, seg_off, seg_task, dy_rows)
        elif self.nvls is not None:
            dY = self.nvls.ag(("ag", id(self)), dy_rows)
            dXp, dA, dB = self.be.bwd(seg_off, seg_task, self.ads, dY, self.X, self.W, self.Hs, self.r_cap)
            self.nvls.release(("ag", id(self)))
        else:
            dY = all_gather_rows(dy_rows, self.group)
            Gs = None
            if self.shared_shrink:
                rows_p = dy_rows.shape[0]
                r0 = rows_p * _world(self.group)[1]
                Gs_own = self.be.shrink_bwd(seg_off, seg_task, self.ads, dY, self.W, self.r_cap, r0, r0 + rows_p)
                Gs = all_gather_rows(Gs_own[r0:r0 + rows_p].contiguous(), self.group)
            dXp, dA, dB = self.be.bwd(seg_off, seg_task, self.ads, dY, self.X, self.W, self.Hs, self.r_cap, Gs=Gs)
        for g in dB:
            if g is not None:
                all_reduce_(g, self.group)
        self.dA, self.dB = dA, dB
        return dXp, dA, dB
