#!/usr/bin/env python
"""Interleaved A/B: a fused projection (one column-sliced mux_linear call, include/mux.h "Fused
projections") vs the same slices as separate mux_linear_fwd / _bwd calls, same process, same
tensors, round-robin (--rounds x --iters, median round) so clock drift under the power cap hits both
alike.  Passes: fwd, dX (the backward GEMM), grads (adapter gradients).  Config-4 style: 16 tasks,
ranks cycling 8/16/32/64, ~21.5k rows.
usage: python tools/fused_ab.py [--sets qkv1,gu1,qkv8,gu8] [--out profiles/r02_fused_ab.jsonl]
"""
import argparse
import json
import os
import statistics
import sys

import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

SETS = {  # name: (K, slice widths)
    "qkv1": (4096, [4096, 4096, 4096]), "gu1": (4096, [11008, 11008]),
    "qkv2": (4096, [2048, 2048, 2048]), "gu2": (4096, [5504, 5504]),
    "qkv4": (4096, [1024, 1024, 1024]), "gu4": (4096, [2752, 2752]),
    "qkv8": (4096, [512, 512, 512]), "gu8": (4096, [1376, 1376]),
    "qkv70b8": (8192, [1024, 128, 128]), "gu70b8": (8192, [3584, 3584]),
    "o8": (512, [4096]), "down8": (1376, [4096]),   # one slice: per-pass times of the row-parallel shards
}


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--sets", default="qkv1,gu1,qkv8,gu8")
    ap.add_argument("--rows", type=int, default=21504)
    ap.add_argument("--tasks", type=int, default=16)
    ap.add_argument("--iters", type=int, default=5)
    ap.add_argument("--rounds", type=int, default=9)
    ap.add_argument("--out", default=None)
    a = ap.parse_args()
    from paper_2603_02885_b200 import mux
    M, R = a.tasks, a.rows
    ranks = [(8, 16, 32, 64)[t % 4] for t in range(M)]
    r_cap = 64
    seg = R // M // 64 * 64
    seg_off = torch.tensor([min(i * seg, R) if i < M else R for i in range(M + 1)], dtype=torch.int32, device="cuda")
    st = list(range(M))
    g = torch.Generator(device="cuda").manual_seed(0)
    out = open(a.out, "a") if a.out else None
    for name in a.sets.split(","):
        K, widths = SETS[name]
        S, N = len(widths), sum(widths)
        col_off = [0]
        for w in widths:
            col_off.append(col_off[-1] + w)
        W = (torch.randn(N, K, device="cuda", generator=g) / K ** 0.5).bfloat16()
        Ws = [W[col_off[s]:col_off[s + 1]] for s in range(S)]   # row slices: contiguous views
        ads = []
        for r in ranks:
            row = []
            for w in widths:
                B = mux.make_B_storage(w, r)
                B.copy_(torch.randn(w, r, device="cuda", generator=g).bfloat16())
                row.append(mux.Adapter((torch.randn(r, K, device="cuda", generator=g) / K ** 0.5).bfloat16(), B, r,
                                       2.0, torch.empty(r, K, device="cuda"), torch.empty(w, r, device="cuda")))
            ads.append(row)
        per_slice = [[ads[t][s] for t in range(M)] for s in range(S)]
        X = torch.randn(R, K, device="cuda", generator=g).bfloat16()
        dY = torch.randn(R, N, device="cuda", generator=g).bfloat16()
        dYs = [dY[:, col_off[s]:col_off[s + 1]].contiguous() for s in range(S)]
        Y = torch.empty(R, N, dtype=torch.bfloat16, device="cuda")
        Ys = [torch.empty(R, w, dtype=torch.bfloat16, device="cuda") for w in widths]
        Hs = torch.empty(R, S * r_cap, dtype=torch.bfloat16, device="cuda")
        Hss = [torch.empty(R, r_cap, dtype=torch.bfloat16, device="cuda") for _ in widths]
        dX = torch.empty(R, K, dtype=torch.bfloat16, device="cuda")
        dXs = [torch.empty(R, K, dtype=torch.bfloat16, device="cuda") for _ in widths]
        wsf = torch.zeros(mux.linear_workspace_size(M, R, K, N, S * r_cap), dtype=torch.uint8, device="cuda")
        wss = [torch.zeros(mux.linear_workspace_size(M, R, K, w, r_cap), dtype=torch.uint8, device="cuda")
               for w in widths]
        impl = {
            "fused": {
                "fwd": lambda: mux.linear_fwd_sliced(seg_off, st, ads, X, W, col_off, r_cap, Y=Y, Hs=Hs, workspace=wsf),
                "dx": lambda: mux.linear_bwd_sliced(seg_off, st, ads, dY, X, W, Hs, col_off, r_cap, dX=dX,
                                                    workspace=wsf, part=mux.BWD_DX),
                "grads": lambda: mux.linear_bwd_sliced(seg_off, st, ads, dY, X, W, Hs, col_off, r_cap, want_dx=False,
                                                       workspace=wsf, part=mux.BWD_GRADS)},
            "separate": {
                "fwd": lambda: [mux.linear_fwd(seg_off, st, per_slice[s], X, Ws[s], r_cap, Y=Ys[s], Hs=Hss[s],
                                               workspace=wss[s]) for s in range(S)],
                "dx": lambda: [mux.linear_bwd(seg_off, st, per_slice[s], dYs[s], X, Ws[s], Hss[s], r_cap, dX=dXs[s],
                                              workspace=wss[s], part=mux.BWD_DX) for s in range(S)],
                "grads": lambda: [mux.linear_bwd(seg_off, st, per_slice[s], dYs[s], X, Ws[s], Hss[s], r_cap,
                                                 want_dx=False, workspace=wss[s], part=mux.BWD_GRADS)
                                  for s in range(S)]},
        }
        for pas in ("fwd", "dx", "grads"):
            for k in impl:
                impl[k]["fwd"]()
                impl[k][pas]()
            torch.cuda.synchronize()
            times = {k: [] for k in impl}
            for _ in range(a.rounds):
                for k in impl:
                    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                    e0.record()
                    for _ in range(a.iters):
                        impl[k][pas]()
                    e1.record()
                    torch.cuda.synchronize()
                    times[k].append(e0.elapsed_time(e1) / a.iters)
            for k in impl:
                med = statistics.median(times[k])
                line = {"set": name, "K": K, "widths": widths, "pass": pas, "impl": k, "rows": R, "tasks": M,
                        "ms": round(med, 4), "spread": round((max(times[k]) - min(times[k])) / med, 3)}
                print(json.dumps(line), flush=True)
                if out:
                    out.write(json.dumps(line) + "\n")
        del W, Ws, ads, per_slice, X, dY, dYs, Y, Ys, Hs, Hss, dX, dXs, wsf, wss
        torch.cuda.empty_cache()


if __name__ == "__main__":
    main()
