#!/usr/bin/env python
"""Interleaved A/B of the adapter-gradient kernels: tcgen05 (grad.cu, default
build) vs CUDA cores (grad_simt.cu, libmux_gsimt.so) on the config-2 linears
at ranks 4..64 (north_star: "warp-level reductions where rank is too small for
tensor cores").  Times mux_linear_bwd_part(BWD_GRADS) only (Gs comes from a
preceding dX pass on the same workspace).  Algorithmic bytes per launch:
2·R·(K+N) (X, dY) + 4·R·r_cap (Hs, Gs read once) + 4·Σ_t r_t·(K+N) (dA, dB).

usage: python tools/grad_ab.py [--rows 10816] [--tasks 4] [--ranks 4,8,16,32,64]
Prints one JSON line per (impl, shape, rank).
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
    ap.add_argument("--rows", type=int, default=10816)
    ap.add_argument("--tasks", type=int, default=4)
    ap.add_argument("--ranks", default="4,8,16,32,64")
    ap.add_argument("--shapes", default="4096x4096,4096x11008,11008x4096")
    ap.add_argument("--iters", type=int, default=20)
    ap.add_argument("--rounds", type=int, default=9)
    a = ap.parse_args()
    from paper_2603_02885_b200 import build as mbuild, mux
    libs = {"tcgen05": mux.LIB_PATH,
            "simt": mbuild.build(defines=("MUX_GRAD_SIMT_MAX_RANK=64",), out="libmux_gsimt.so")}
    handles = {}
    for name, path in libs.items():
        mux.LIB_PATH, mux._lib = path, None
        handles[name] = mux.lib()
    R = a.rows
    torch.manual_seed(0)
    for shape in a.shapes.split(","):
        K, N = (int(v) for v in shape.split("x"))
        X = torch.randn(R, K, device="cuda").bfloat16()
        W = (torch.randn(N, K, device="cuda") / K ** 0.5).bfloat16()
        dY = torch.randn(R, N, device="cuda").bfloat16()
        seg = R // a.tasks // 64 * 64
        seg_off = torch.tensor([i * seg for i in range(a.tasks)] + [R], dtype=torch.int32, device="cuda")
        for r in (int(v) for v in a.ranks.split(",")):
            r_cap = max(16, -(-r // 16) * 16)
            ads = []
            for t in range(a.tasks):
                A = (torch.randn(r, K, device="cuda") / K ** 0.5).bfloat16()
                B = mux.make_B_storage(N, r)
                B.copy_(torch.randn(N, r, device="cuda").bfloat16())
                ads.append(mux.Adapter(A, B, r, 2.0))
            st = list(range(a.tasks))
            ws = torch.zeros(mux.linear_workspace_size(a.tasks, R, K, N, r_cap), dtype=torch.uint8, device="cuda")
            mux._lib = handles["tcgen05"]
            Y, Hs = mux.linear_fwd(seg_off, st, ads, X, W, r_cap, workspace=ws)
            dX = mux.linear_bwd(seg_off, st, ads, dY, X, W, Hs, r_cap, workspace=ws, part=mux.BWD_DX)

            def run(name):
                mux._lib = handles[name]
                mux.linear_bwd(seg_off, st, ads, dY, X, W, Hs, r_cap, dX=dX, workspace=ws, part=mux.BWD_GRADS)

            times = {n: [] for n in libs}
            for n in libs:
                for _ in range(3):
                    run(n)
            torch.cuda.synchronize()
            for _ in range(a.rounds):
                for n in libs:
                    s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                    s.record()
                    for _ in range(a.iters):
                        run(n)
                    e.record()
                    torch.cuda.synchronize()
                    times[n].append(s.elapsed_time(e) / a.iters)
            byts = 2 * R * (K + N) + 4 * R * r_cap + 4 * a.tasks * r * (K + N)
            flops = 4 * R * r * (K + N)
            for n in libs:
                ms = statistics.median(times[n])
                print(json.dumps({"impl": n, "K": K, "N": N, "rank": r, "rows": R, "tasks": a.tasks,
                                  "ms": round(ms, 4), "GB/s": round(byts / ms / 1e6, 1),
                                  "TFLOP/s": round(flops / ms / 1e9, 2),
                                  "spread": round((max(times[n]) - min(times[n])) / ms, 3)}), flush=True)
    mux._lib = None


if __name__ == "__main__":
    main()
