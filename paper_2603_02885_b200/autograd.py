"""PyTorch autograd integration of the multiplexed LoRA linear.

`MuxLoRALinear` holds one frozen backbone weight W [N, K] and one LoRA adapter
(A_t [r_t, K], B_t [N, r_t], scale s_t) per task as trainable parameters; its
forward takes the packed activations X [rows, K] plus the segment table from
mux_pack_chunks and runs mux_linear_fwd; backward runs mux_linear_bwd and
hands dX and every adapter's (dA_t, dB_t) to autograd (no gradient for W: the
backbone is frozen).  Thin glue only: all arithmetic is in libmux.

    lin = MuxLoRALinear(W, ranks=[16, 8], scales=[2.0, 2.0])
    Y = lin(X, seg_off, seg_task=[0, 1])      # X: packed rows (bf16, requires_grad ok)
    loss(Y).backward()                         # fills lin.A[t].grad, lin.B[t].grad
"""
from __future__ import annotations

from typing import List, Sequence

import torch

from . import mux


class _MuxLinearFn(torch.autograd.Function):
    @staticmethod
    def forward(ctx, X, seg_off, W, mod, *params):
        ads = mod._adapters()
        seg_task = list(mod._seg_task)
        Xc = X.contiguous()       # the tensor the kernel reads is the one backward re-reads
        Y, Hs = mux.linear_fwd(seg_off, seg_task, ads, Xc, W, mod.r_cap,
                               workspace=mod._workspace(Xc.shape[0], len(seg_task)))
        ctx.save_for_backward(Xc, seg_off, Hs)
        ctx.mod = mod
        ctx.seg_task = seg_task   # this call's segment -> adapter map (the module may be re-called)
        return Y

    @staticmethod
    def backward(ctx, dY):
        X, seg_off, Hs = ctx.saved_tensors
        mod = ctx.mod
        ads = mod._adapters()
        want_dx = ctx.needs_input_grad[0]
        dX = mux.linear_bwd(seg_off, ctx.seg_task, ads, dY.contiguous(), X, mod.W, Hs, mod.r_cap,
                            want_dx=want_dx, workspace=mod._workspace(X.shape[0], len(ctx.seg_task)))
        grads: List = []
        for t, a in enumerate(ads):
            if a.rank == 0:
                continue
            grads.append(a.dA.to(mod.A[t].dtype))
            grads.append(a.dB.to(mod.B[t].dtype))
        return (dX if want_dx else None, None, None, None, *grads)


class MuxLoRALinear(torch.nn.Module):
    """Frozen backbone linear shared by several tasks, each with its own LoRA
    adapter; one fused call serves all tasks' rows (spatial multiplexing)."""

    def __init__(self, W: torch.Tensor, ranks: Sequence[int], scales: Sequence[float], init_B_zero: bool = True):
        super().__init__()
        assert W.dtype == torch.bfloat16 and W.dim() == 2
        self.register_buffer("W", W.contiguous(), persistent=True)
        N, K = W.shape
        self.ranks = [int(r) for r in ranks]
        self.scales = [float(s) for s in scales]
        self.r_cap = max(16, 16 * -(-max(self.ranks + [1]) // 16))
        self.A = torch.nn.ParameterList()
        self.B = torch.nn.ParameterList()
        self._B_storage = []
        for r in self.ranks:
            A = torch.randn(r, K, device=W.device) / K ** 0.5
            self.A.append(torch.nn.Parameter(A.bfloat16()))
            Bst = mux.make_B_storage(N, r, device=W.device)   # [N, r] view of 16-byte-aligned rows
            if not init_B_zero:
                Bst.copy_((torch.randn(N, r, device=W.device) / max(r, 1) ** 0.5).bfloat16())
            self.B.append(torch.nn.Parameter(Bst))
            self._B_storage.append(Bst)
        self._seg_task: List[int] = []
        self._ws = None

    def _adapters(self):
        return [mux.Adapter(self.A[t].data if r else None, self.B[t].data if r else None, r, self.scales[t])
                for t, r in enumerate(self.ranks)]

    def _workspace(self, rows: int, num_segs: int):
        need = mux.linear_workspace_size(max(1, num_segs), rows, self.W.shape[1], self.W.shape[0], self.r_cap)
        if self._ws is None or self._ws.numel() < need:
            self._ws = torch.zeros(need, dtype=torch.uint8, device=self.W.device)
        return self._ws

    def forward(self, X: torch.Tensor, seg_off: torch.Tensor, seg_task: Sequence[int]):
        self._seg_task = [int(s) for s in seg_task]
        params = [p for t, r in enumerate(self.ranks) if r for p in (self.A[t], self.B[t])]
        return _MuxLinearFn.apply(X, seg_off, self.W, self, *params)
