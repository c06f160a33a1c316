#!/usr/bin/env python
"""Fine-tune three LoRA tasks at once on one frozen backbone (spatial
multiplexing, the MuxTune hot path), end to end through the public API:

  1. each task brings its own variable-length sequences (token-major rows);
  2. mux.pack_chunks aligns them into chunks and gives the packed
     row map; mux.pack_apply dispatches the token rows into packed order;
  3. two MuxLoRALinear layers (frozen W, one adapter per task) run every
     task's rows in one fused tcgen05 GEMM each, forward and backward;
  4. a per-task loss (plain torch, user code) drives one optimizer over all
     adapters; the backbone never changes.

usage: python examples/multitask_lora_train.py [--steps 30]
Prints each task's loss; they fall independently (each task's targets come
from a teacher with the same backbone and its own hidden adapters).
"""
import argparse
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2603_02885_b200 import mux  # noqa: E402
from paper_2603_02885_b200.autograd import MuxLoRALinear  # noqa: E402


def main(steps=30, seed=0, verbose=True):
    torch.manual_seed(seed)
    dev = "cuda"
    H, F = 1024, 2816
    seq_lens = [[200, 120, 64], [512], [96, 96, 96, 40]]        # per task: its sequences this step
    ranks, scales = [16, 8, 32], [2.0, 2.0, 2.0]
    off = [0]
    for x in seq_lens:
        off.append(off[-1] + len(x))
    lens = [v for x in seq_lens for v in x]
    T = sum(lens)
    max_rows = mux.pack_bound_rows(T, len(lens), 64)
    pk = mux.pack_chunks(off, lens, None, 0, 64, max_rows=max_rows, max_chunks=max_rows // 64)
    seg_off, seg_task = pk["seg_off"], list(range(len(seq_lens)))

    W1 = (torch.randn(F, H, device=dev) / H ** 0.5).bfloat16()
    W2 = (torch.randn(H, F, device=dev) / F ** 0.5).bfloat16()
    up = MuxLoRALinear(W1, ranks, scales)
    down = MuxLoRALinear(W2, ranks, scales)
    opt = torch.optim.Adam(list(up.parameters()) + list(down.parameters()), lr=2e-3)

    x_tok = torch.randn(T, H, device=dev).bfloat16()              # token-major inputs of all tasks
    X = mux.pack_apply(pk["row_src"], x_tok, max_rows)             # packed rows (pads = 0)
    row_src = pk["row_src"].long()
    valid = row_src >= 0
    tok_task = torch.repeat_interleave(torch.arange(len(seq_lens), device=dev),
                                       torch.tensor([sum(x) for x in seq_lens], device=dev))
    row_task = torch.full((max_rows,), -1, device=dev, dtype=torch.long)
    row_task[valid] = tok_task[row_src[valid]]
    # each task's "dataset": the outputs of a teacher with the same frozen backbone and its own
    # (hidden) adapters; the students start from B = 0 and must recover them
    t_up = MuxLoRALinear(W1, ranks, scales, init_B_zero=False)
    t_down = MuxLoRALinear(W2, ranks, scales, init_B_zero=False)
    with torch.no_grad():
        target = t_down(torch.nn.functional.silu(t_up(X, seg_off, seg_task).float()).bfloat16(),
                        seg_off, seg_task).float()

    history = []
    for step in range(steps):
        h = up(X, seg_off, seg_task)                               # [max_rows, F] bf16
        h = torch.nn.functional.silu(h.float()).bfloat16()
        y = down(h, seg_off, seg_task).float()                     # [max_rows, H]
        err = (y - target) ** 2
        losses = [err[row_task == t].mean() for t in range(len(seq_lens))]
        opt.zero_grad()
        sum(losses).backward()
        opt.step()
        history.append([l.item() for l in losses])
        if verbose and (step % 5 == 0 or step == steps - 1):
            print(f"step {step:3d}  " + "  ".join(f"task{t} {v:.4f}" for t, v in enumerate(history[-1])))
    return history


if __name__ == "__main__":
    ap = argparse.ArgumentParser()
    ap.add_argument("--steps", type=int, default=30)
    a = ap.parse_args()
    main(a.steps)
