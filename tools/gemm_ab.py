#!/usr/bin/env python
"""Interleaved A/B timing of the fused GEMM (one or more libmux builds) and
cuBLAS (torch.matmul) on the same shapes, same process.  Implementations are
timed round-robin for --rounds rounds of --iters launches each and the median
round is reported, so clock drift under the power cap hits all of them alike.

usage: python tools/gemm_ab.py [--libs a.so b.so] [--rows 11648] [--rank 16]
Prints one JSON line per (impl, shape, pass): median ms, TFLOP/s, spread.
"""
import argparse
import json
import os
import statistics
import sys

import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def time_once(fn, iters):
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
    ap.add_argument("--iters", type=int, default=10)
    ap.add_argument("--rounds", type=int, default=9)
    ap.add_argument("--tasks", type=int, default=4)
    ap.add_argument("--rank", type=int, default=16)
    ap.add_argument("--shapes", default="4096x4096,4096x11008,11008x4096")
    ap.add_argument("--no-cublas", action="store_true")
    ap.add_argument("--fwd-only", action="store_true")
    ap.add_argument("--env-ab", default="",
                    help="VAR=a,b: time every lib once per value of the environment variable VAR (read per "
                         "call by libmux, e.g. MUX_CARRY=1,0)")
    a = ap.parse_args()
    from paper_2603_02885_b200 import mux
    handles = {}
    for lib in a.libs:
        mux.LIB_PATH = lib
        mux._lib = None
        handles[lib] = mux.lib()
    R = a.rows
    shapes = [tuple(int(v) for v in s.split("x")) for s in a.shapes.split(",")]
    torch.manual_seed(0)
    for K, N in shapes:
        X = torch.randn(R, K, device="cuda").bfloat16()
        W = (torch.randn(N, K, device="cuda") / K ** 0.5).bfloat16()
        dY = torch.randn(R, N, device="cuda").bfloat16()
        seg = R // a.tasks // 64 * 64
        seg_off = torch.tensor([min(i * seg, R) if i < a.tasks else R for i in range(a.tasks + 1)],
                               dtype=torch.int32, device="cuda")
        ads = []
        for t in range(a.tasks):
            B = mux.make_B_storage(N, a.rank)
            B.copy_(torch.randn(N, a.rank, device="cuda").bfloat16())
            ads.append(mux.Adapter((torch.randn(a.rank, K, device="cuda") / K ** 0.5).bfloat16(), B, a.rank, 2.0))
        r_cap = max(16, 16 * -(-a.rank // 16))
        Y = torch.empty(R, N, dtype=torch.bfloat16, device="cuda")
        Hs = torch.empty(R, r_cap, dtype=torch.bfloat16, device="cuda")
        dX = torch.empty(R, K, dtype=torch.bfloat16, device="cuda")
        st = list(range(a.tasks))
        cands = {}
        if not a.no_cublas:
            cands[("cublas", "fwd")] = (lambda: torch.matmul(X, W.t()), 2 * R * K * N)
            cands[("cublas", "dX")] = (lambda: torch.matmul(dY, W), 2 * R * K * N)
        var, vals = (a.env_ab.split("=", 1) + [""])[:2] if a.env_ab else ("", "")
        for lib, h in handles.items():
          for val in (vals.split(",") if var else [None]):
            ws = torch.zeros(mux.linear_workspace_size(a.tasks, R, K, N, r_cap), dtype=torch.uint8, device="cuda")

            def setenv(val=val):
                if val is not None:
                    os.environ[var] = val

            def fwd(h=h, ws=ws, setenv=setenv):
                mux._lib = h
                setenv()
                mux.linear_fwd(seg_off, st, ads, X, W, r_cap, Y=Y, Hs=Hs, workspace=ws)

            def bwd(h=h, ws=ws, setenv=setenv):
                mux._lib = h
                setenv()
                mux.linear_bwd(seg_off, st, ads, dY, X, W, Hs, r_cap, dX=dX, workspace=ws)
            name = os.path.basename(lib) + (f"[{var}={val}]" if val is not None else "")
            cands[(name, "fwd")] = (fwd, 2 * R * K * N + 2 * R * a.rank * (K + N))
            if not a.fwd_only:
                cands[(name, "bwd(dX+grads)")] = (bwd, 2 * R * K * N + 4 * R * a.rank * (K + N))
        for fn, _ in cands.values():
            for _ in range(3):
                fn()
        torch.cuda.synchronize()
        times = {k: [] for k in cands}
        for _ in range(a.rounds):
            for k, (fn, _) in cands.items():
                times[k].append(time_once(fn, a.iters))
        for (impl, ps), ts in times.items():
            med = statistics.median(ts)
            print(json.dumps({"impl": impl, "pass": ps, "K": K, "N": N, "rows": R, "rank": a.rank, "ms": med,
                              "tflops": cands[(impl, ps)][1] / med / 1e9,
                              "spread": (max(ts) - min(ts)) / med}), flush=True)


if __name__ == "__main__":
    main()
