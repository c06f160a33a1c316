#!/usr/bin/env python
"""A/B timing of the fused GEMM (one or more libmux builds) against cuBLAS
(torch.matmul) on the same shapes, same process, same clocks.

usage: python tools/gemm_ab.py [--libs path1.so path2.so] [--rows 11648] [--iters 50]
Prints one JSON line per (lib, shape, pass) with TFLOP/s (executed rows).
"""
import argparse
import json
import os
import sys

import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def timeit(fn, iters, warm=5):
    for _ in range(warm):
        fn()
    torch.cuda.synchronize()
    s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    s.record()
    for _ in range(iters):
        fn()
    e.record()
    torch.cuda.synchronize()
    return s.elapsed_time(e) / iters


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--libs", nargs="*", default=[os.path.join(ROOT, "paper_2603_02885_b200", "libmux.so")])
    ap.add_argument("--rows", type=int, default=11648)
    ap.add_argument("--iters", type=int, default=30)
    ap.add_argument("--tasks", type=int, default=4)
    ap.add_argument("--rank", type=int, default=16)
    ap.add_argument("--shapes", default="4096x4096,4096x11008,11008x4096")
    a = ap.parse_args()
    from paper_2603_02885_b200 import mux
    R = a.rows
    shapes = [tuple(int(v) for v in s.split("x")) for s in a.shapes.split(",")]
    torch.manual_seed(0)
    for K, N in shapes:
        X = torch.randn(R, K, device="cuda").bfloat16()
        W = (torch.randn(N, K, device="cuda") / K ** 0.5).bfloat16()
        dY = torch.randn(R, N, device="cuda").bfloat16()
        ms = timeit(lambda: torch.matmul(X, W.t()), a.iters)
        print(json.dumps({"impl": "cublas", "pass": "fwd", "K": K, "N": N, "rows": R, "ms": ms,
                          "tflops": 2 * R * K * N / ms / 1e9}), flush=True)
        ms = timeit(lambda: torch.matmul(dY, W), a.iters)
        print(json.dumps({"impl": "cublas", "pass": "dX", "K": K, "N": N, "rows": R, "ms": ms,
                          "tflops": 2 * R * K * N / ms / 1e9}), flush=True)
        seg = R // a.tasks // 64 * 64
        seg_off = torch.tensor([min(i * seg, R) if i < a.tasks else R for i in range(a.tasks + 1)],
                               dtype=torch.int32, device="cuda")
        for lib in a.libs:
            mux.LIB_PATH = lib
            mux._lib = None
            ads = []
            for t in range(a.tasks):
                B = mux.make_B_storage(N, a.rank)
                B.copy_(torch.randn(N, a.rank, device="cuda").bfloat16())
                ads.append(mux.Adapter((torch.randn(a.rank, K, device="cuda") / K ** 0.5).bfloat16(), B,
                                       a.rank, 2.0))
            r_cap = max(16, 16 * -(-a.rank // 16))
            Y = torch.empty(R, N, dtype=torch.bfloat16, device="cuda")
            Hs = torch.empty(R, r_cap, dtype=torch.bfloat16, device="cuda")
            dX = torch.empty(R, K, dtype=torch.bfloat16, device="cuda")
            ws = torch.zeros(mux.linear_workspace_size(a.tasks, R, K, N, r_cap), dtype=torch.uint8, device="cuda")
            st = list(range(a.tasks))
            f = lambda: mux.linear_fwd(seg_off, st, ads, X, W, r_cap, Y=Y, Hs=Hs, workspace=ws)  # noqa: E731
            ms = timeit(f, a.iters)
            fl = 2 * R * K * N + 2 * R * a.rank * (K + N)
            print(json.dumps({"impl": os.path.basename(lib), "pass": "fwd", "K": K, "N": N, "rows": R, "ms": ms,
                              "tflops": fl / ms / 1e9}), flush=True)
            b = lambda: mux.linear_bwd(seg_off, st, ads, dY, X, W, Hs, r_cap, dX=dX, workspace=ws)  # noqa: E731
            ms = timeit(b, a.iters)
            fl = 2 * R * K * N + 4 * R * a.rank * (K + N)
            print(json.dumps({"impl": os.path.basename(lib), "pass": "bwd(dX+grads)", "K": K, "N": N, "rows": R,
                              "ms": ms, "tflops": fl / ms / 1e9}), flush=True)


if __name__ == "__main__":
    main()
