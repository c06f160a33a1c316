#!/usr/bin/env python
"""SURVEY §8(d) config-2 sweeps of the whole fused fwd+bwd (mux_linear_fwd +
mux_linear_bwd through the three LLaMA-7B linears 4096->4096, 4096->11008,
11008->4096), device time from a CUDA graph of the three layers' calls:

  tasks  1, 2, 4, 8, 16 at 2560 tokens per task, rank 16 (the analogue of P:528)
  T      512, 2048, 10240 tokens over 4 tasks, rank 16
  rank   4, 8, 16, 32, 64 at 4 tasks, 10240 tokens (analogue of E-2)

Segments are equal, multiples of 64 rows, all rows valid (no chunk padding, so
tokens = rows).  Reports tokens/s, algorithmic TFLOP/s (4KN + 6r(K+N) per token
per linear) and the fraction of the measured bf16 peaks.
usage: python tools/sweep.py [--out profiles/r01_sweep.jsonl]
"""
import argparse
import json
import os
import statistics
import sys

import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "tools"))

BURST, SUSTAINED = 1666.9, 1420.8  # TFLOP/s, MEASURED_PEAKS


def point(mux, LayerSet, tasks, tokens, rank, reps=5):
    seg = tokens // tasks // 64 * 64
    rows = seg * tasks
    ls = LayerSet(mux, rows, tasks, rank)
    seg_off = torch.tensor([i * seg for i in range(tasks + 1)], dtype=torch.int32, device="cuda")
    st = list(range(tasks))

    def step():
        for li in range(3):
            ls.run(li, seg_off, st, ls.L[li]["ads"], rows)

    s = torch.cuda.Stream()
    s.wait_stream(torch.cuda.current_stream())
    with torch.cuda.stream(s):
        step()
    torch.cuda.synchronize()
    g = torch.cuda.CUDAGraph()
    with torch.cuda.graph(g, stream=s):
        for _ in range(reps):
            step()
    for _ in range(2):
        g.replay()
    torch.cuda.synchronize()
    vals = []
    for _ in range(7):
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record()
        g.replay()
        b.record()
        torch.cuda.synchronize()
        vals.append(a.elapsed_time(b) / reps)
    ms = statistics.median(vals)
    flops = sum(rows * (4 * K * N + 6 * rank * (K + N)) for K, N in ((4096, 4096), (4096, 11008), (11008, 4096)))
    tf = flops / ms / 1e9
    del g, ls
    torch.cuda.empty_cache()
    return {"tasks": tasks, "tokens": rows, "rank": rank, "ms_fwd_bwd": round(ms, 4),
            "tokens_per_s": round(rows / ms * 1e3), "tflops": round(tf, 1),
            "frac_burst": round(tf / BURST, 3), "frac_sustained": round(tf / SUSTAINED, 3)}


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--out", default=None)
    a = ap.parse_args()
    from paper_2603_02885_b200 import mux
    from op_profile import LayerSet
    out = open(a.out, "w") if a.out else None
    pts = [("tasks", t, 2560 * t, 16) for t in (1, 2, 4, 8, 16)]
    pts += [("T", 4, T, 16) for T in (512, 2048, 10240)]
    pts += [("rank", 4, 10240, r) for r in (4, 8, 16, 32, 64)]
    for sweep, tasks, tokens, rank in pts:
        r = {"sweep": sweep, **point(mux, LayerSet, tasks, tokens, rank)}
        line = json.dumps(r)
        print(line, flush=True)
        if out:
            out.write(line + "\n")


if __name__ == "__main__":
    main()
