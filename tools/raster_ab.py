#!/usr/bin/env python
"""Interleaved A/B of the fused GEMM's raster direction (MUX_RASTER, read by libmux per call):
row bands (m: a band of A rows L2-resident, W streamed once per band) vs column bands (n: a band
of W tiles L2-resident, A streamed once per band) on the config-2 shapes, forward and dX, 11648
rows, 4 tasks r = 16.  Modes are timed round-robin (--rounds x --iters launches, median round) so
clock drift under the power cap hits both alike.  --once runs every (shape, pass, mode) a single
time for an ncu DRAM-traffic capture (ncu -k regex:mux_gemm ... --once: launches in the order
shape x pass x mode).
usage: python tools/raster_ab.py [--modes m,n] [--out profiles/r02_raster_ab.jsonl] [--once]
       python tools/raster_ab.py --var MUX_TILE_N --modes 256,512   (any per-call env switch of libmux)
"""
import argparse
import json
import os
import statistics
import sys

import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--rows", type=int, default=11648)
    ap.add_argument("--iters", type=int, default=10)
    ap.add_argument("--rounds", type=int, default=9)
    ap.add_argument("--modes", default="m,n")
    ap.add_argument("--var", default="MUX_RASTER")
    ap.add_argument("--tasks", type=int, default=4)
    ap.add_argument("--rank", type=int, default=16)
    ap.add_argument("--shapes", default="4096x4096,4096x11008,11008x4096")
    ap.add_argument("--once", action="store_true")
    ap.add_argument("--out", default=None)
    a = ap.parse_args()
    from paper_2603_02885_b200 import mux
    R, T = a.rows, a.tasks
    V = a.var
    modes = a.modes.split(",")
    torch.manual_seed(0)
    out = open(a.out, "a") if a.out else None
    for shp in a.shapes.split(","):
        K, N = (int(v) for v in shp.split("x"))
        X = torch.randn(R, K, device="cuda").bfloat16()
        W = (torch.randn(N, K, device="cuda") / K ** 0.5).bfloat16()
        dY = torch.randn(R, N, device="cuda").bfloat16()
        seg = R // T // 64 * 64
        seg_off = torch.tensor([i * seg if i < T else R for i in range(T + 1)], dtype=torch.int32, device="cuda")
        ads = []
        rk = a.rank
        rc = max(16, -(-rk // 16) * 16)
        for _ in range(T):
            B = mux.make_B_storage(N, rk)
            B.copy_(torch.randn(N, rk, device="cuda").bfloat16())
            ads.append(mux.Adapter((torch.randn(rk, K, device="cuda") / K ** 0.5).bfloat16(), B, rk, 2.0))
        Y = torch.empty(R, N, dtype=torch.bfloat16, device="cuda")
        Hs = torch.empty(R, rc, dtype=torch.bfloat16, device="cuda")
        dX = torch.empty(R, K, dtype=torch.bfloat16, device="cuda")
        ws = torch.zeros(mux.linear_workspace_size(T, R, K, N, rc), dtype=torch.uint8, device="cuda")
        st = list(range(T))
        mux.linear_fwd(seg_off, st, ads, X, W, rc, Y=Y, Hs=Hs, workspace=ws)
        passes = {
            "fwd": lambda: mux.linear_fwd(seg_off, st, ads, X, W, rc, Y=Y, Hs=Hs, workspace=ws),
            "dx": lambda: mux.linear_bwd(seg_off, st, ads, dY, X, W, Hs, rc, dX=dX, workspace=ws, part=mux.BWD_DX),
        }
        flops = R * (2 * K * N + 2 * rk * (K + N))
        for pname, fn in passes.items():
            if a.once:
                for m in modes:
                    os.environ[V] = m
                    fn()
                torch.cuda.synchronize()
                continue
            times = {m: [] for m in modes}
            for m in modes:       # warm-up
                os.environ[V] = m
                fn()
            for _ in range(a.rounds):
                for m in modes:
                    os.environ[V] = m
                    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                    e0.record()
                    for _ in range(a.iters):
                        fn()
                    e1.record()
                    torch.cuda.synchronize()
                    times[m].append(e0.elapsed_time(e1) / a.iters)
            for m in modes:
                med = statistics.median(times[m])
                line = {"shape": f"{K}x{N}", "pass": pname, V: m, "rows": R, "ms": round(med, 4),
                        "tflops": round(flops / med / 1e9, 1),
                        "spread": round((max(times[m]) - min(times[m])) / med, 3)}
                print(json.dumps(line), flush=True)
                if out:
                    out.write(json.dumps(line) + "\n")
        del X, W, dY, Y, Hs, dX, ws, ads
        torch.cuda.empty_cache()
    os.environ.pop(V, None)


if __name__ == "__main__":
    main()
