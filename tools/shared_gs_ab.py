#!/usr/bin/env python
"""Interleaved A/B of a row-parallel layer's backward at TP shard shapes: (plain) mux_linear_bwd, every
rank computing Gs for all rows inside the dX GEMM, vs (shared) MUX_OP_SHRINK_BWD of this rank's 1/p rows
followed by the backward with Gs given (tp.py RowParallelMuxLinear shared_shrink; the Gs all-gather,
T x r_cap bf16, is not run).  CUDA-graph device time, median of --rounds.
usage: python tools/shared_gs_ab.py [--out profiles/r02_shared_gs_ab.jsonl]"""
import argparse
import json
import os
import statistics
import sys

import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "tools"))

SHAPES = {"o_7b_tp8": (512, 4096, 8), "down_7b_tp8": (1376, 4096, 8), "o_7b_tp4": (1024, 4096, 4),
          "o_70b_tp8": (1024, 8192, 8), "down_70b_tp8": (3584, 8192, 8)}


def graph_ms(fn, reps=3, rounds=7):
    s = torch.cuda.Stream()
    s.wait_stream(torch.cuda.current_stream())
    with torch.cuda.stream(s):
        fn()
    torch.cuda.synchronize()
    g = torch.cuda.CUDAGraph()
    with torch.cuda.graph(g, stream=s):
        for _ in range(reps):
            fn()
    g.replay()
    torch.cuda.synchronize()
    out = []
    for _ in range(rounds):
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record()
        g.replay()
        b.record()
        torch.cuda.synchronize()
        out.append(a.elapsed_time(b) / reps)
    return out


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--rows", type=int, default=21504)
    ap.add_argument("--tasks", type=int, default=16)
    ap.add_argument("--out", default=None)
    a = ap.parse_args()
    from paper_2603_02885_b200 import mux
    R, M = a.rows, a.tasks
    ranks = [(8, 16, 32, 64)[t % 4] for t in range(M)]
    r_cap = 64
    seg = R // M // 64 * 64
    seg_off = torch.tensor([i * seg if i < M else R for i in range(M + 1)], dtype=torch.int32, device="cuda")
    st = list(range(M))
    g = torch.Generator(device="cuda").manual_seed(0)
    out = open(a.out, "a") if a.out else None
    for name, (K, N, p) in SHAPES.items():
        W = (torch.randn(N, K, device="cuda", generator=g) / K ** 0.5).bfloat16()
        ads = []
        for r in ranks:
            B = mux.make_B_storage(N, r)
            B.copy_(torch.randn(N, r, device="cuda", generator=g).bfloat16())
            ads.append(mux.Adapter((torch.randn(r, K, device="cuda", generator=g) / K ** 0.5).bfloat16(), B, r, 2.0,
                                   torch.empty(r, K, device="cuda"), torch.empty(N, r, device="cuda")))
        X = torch.randn(R, K, device="cuda", generator=g).bfloat16()
        dY = torch.randn(R, N, device="cuda", generator=g).bfloat16()
        Hs = torch.empty(R, r_cap, dtype=torch.bfloat16, device="cuda")
        Gs = torch.empty(R, r_cap, dtype=torch.bfloat16, device="cuda")
        dX = torch.empty(R, K, dtype=torch.bfloat16, device="cuda")
        ws = torch.zeros(mux.linear_workspace_size(M, R, K, N, r_cap), dtype=torch.uint8, device="cuda")
        mux.linear_fwd(seg_off, st, ads, X, W, r_cap, Hs=Hs, workspace=ws)
        hi = -(-R // p // 256) * 256
        impl = {
            "plain": lambda: mux.linear_bwd(seg_off, st, ads, dY, X, W, Hs, r_cap, dX=dX, workspace=ws),
            "shared": lambda: (mux.linear_shrink_bwd(seg_off, st, ads, dY, K, r_cap, 0, hi, Gs=Gs, workspace=ws),
                               mux.linear_bwd_gs(seg_off, st, ads, dY, X, W, Hs, Gs, r_cap, dX=dX, workspace=ws)),
        }
        times = {k: [] for k in impl}
        for _ in range(5):
            for k, f in impl.items():
                times[k] += graph_ms(f, rounds=3)
        for k in impl:
            line = {"shape": name, "K": K, "N": N, "tp": p, "impl": k, "rows": R, "tasks": M,
                    "ms": round(statistics.median(times[k]), 4)}
            print(json.dumps(line), flush=True)
            if out:
                out.write(json.dumps(line) + "\n")
        del W, ads, X, dY, Hs, Gs, dX, ws
        torch.cuda.empty_cache()


if __name__ == "__main__":
    main()
