#!/usr/bin/env python
"""Interleaved A/B of the fused GEMM's two schedules (data-parallel tiles vs stream-K, MUX_SK=0/1,
read by the host at launch time) on tensor-parallel shard shapes, each timed as a CUDA graph of
--reps launches (device time only; no host launch overhead), median over --rounds rounds.
Passes: fwd (shrink side tiles + main tiles), fwd_hs (Hs given: main tiles only), dX (bwd part 1).
usage: python tools/sk_ab.py [--rows 21504 --tasks 16 --shapes 4096x512,512x4096]"""
import argparse
import json
import os
import statistics
import sys

import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def graph_of(fn, reps):
    s = torch.cuda.Stream()
    s.wait_stream(torch.cuda.current_stream())
    with torch.cuda.stream(s):
        fn()
    torch.cuda.synchronize()
    g = torch.cuda.CUDAGraph()
    with torch.cuda.graph(g, stream=s):
        for _ in range(reps):
            fn()
    torch.cuda.synchronize()
    return g


def time_graph(g, reps):
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record()
    g.replay()
    b.record()
    torch.cuda.synchronize()
    return a.elapsed_time(b) / reps


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--rows", type=int, default=21504)
    ap.add_argument("--tasks", type=int, default=16)
    ap.add_argument("--shapes", default="4096x512,512x4096,4096x1376,1376x4096")
    ap.add_argument("--reps", type=int, default=10)
    ap.add_argument("--rounds", type=int, default=7)
    ap.add_argument("--modes", default="0,1")
    a = ap.parse_args()
    from paper_2603_02885_b200 import mux
    R, M = a.rows, a.tasks
    seg = R // M // 64 * 64
    seg_off = torch.tensor([min(i * seg, R) if i < M else R for i in range(M + 1)], dtype=torch.int32, device="cuda")
    st = list(range(M))
    ranks = [(8, 16, 32, 64)[t % 4] for t in range(M)]
    r_cap = 64
    torch.manual_seed(0)
    for shp in a.shapes.split(","):
        K, N = (int(v) for v in shp.split("x"))
        X = torch.randn(R, K, device="cuda").bfloat16()
        W = (torch.randn(N, K, device="cuda") / K ** 0.5).bfloat16()
        dY = torch.randn(R, N, device="cuda").bfloat16()
        ads = []
        for r in ranks:
            B = mux.make_B_storage(N, r)
            B.copy_(torch.randn(N, r, device="cuda").bfloat16())
            ads.append(mux.Adapter((torch.randn(r, K, device="cuda") / K ** 0.5).bfloat16(), B, r, 2.0,
                                   torch.empty(r, K, device="cuda"), torch.empty(N, r, device="cuda")))
        Y = torch.empty(R, N, dtype=torch.bfloat16, device="cuda")
        Hs = torch.empty(R, r_cap, dtype=torch.bfloat16, device="cuda")
        dX = torch.empty(R, K, dtype=torch.bfloat16, device="cuda")
        ws = torch.zeros(mux.linear_workspace_size(M, R, K, N, r_cap), dtype=torch.uint8, device="cuda")
        mux.linear_fwd(seg_off, st, ads, X, W, r_cap, Y=Y, Hs=Hs, workspace=ws)
        passes = {
            "fwd": lambda: mux.linear_fwd(seg_off, st, ads, X, W, r_cap, Y=Y, Hs=Hs, workspace=ws),
            "fwd_hs": lambda: mux.linear_fwd_hs(seg_off, st, ads, X, W, Hs, r_cap, Y=Y, workspace=ws),
            "dX": lambda: mux.linear_bwd(seg_off, st, ads, dY, X, W, Hs, r_cap, dX=dX, workspace=ws,
                                         part=mux.BWD_DX),
        }
        flops = {"fwd": sum(seg * (2 * K * N + 2 * r * (K + N)) for r in ranks),
                 "fwd_hs": sum(seg * (2 * K * N + 2 * r * N) for r in ranks),
                 "dX": sum(seg * (2 * K * N + 2 * r * (K + N)) for r in ranks)}
        for name, fn in passes.items():
            graphs = {}
            for m in a.modes.split(","):
                os.environ["MUX_SK"] = m
                graphs[m] = graph_of(fn, a.reps)
            times = {m: [] for m in graphs}
            for _ in range(a.rounds):
                for m, g in graphs.items():
                    times[m].append(time_graph(g, a.reps))
            for m in graphs:
                ms = statistics.median(times[m])
                print(json.dumps({"K": K, "N": N, "rows": R, "tasks": M, "pass": name, "MUX_SK": m,
                                  "ms": round(ms, 5), "tflops": round(flops[name] / ms / 1e9, 1),
                                  "spread": round((max(times[m]) - min(times[m])) / ms, 3)}), flush=True)
            del graphs
        os.environ.pop("MUX_SK", None)


if __name__ == "__main__":
    main()
