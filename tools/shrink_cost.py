#!/usr/bin/env python
"""What the side-tile shrink costs inside the fused GEMM, i.e. the most any other
placement of the shrink (SURVEY §7 hard part 3, D2: on the n-tile-0 stages, no
extra pass over A) could save.

Per shape, interleaved round-robin (median round), on the same inputs:
  fused   mux_linear_fwd / dX part of mux_linear_bwd: side tiles + main tiles
  given   the same main tiles with Hs / Gs given (mux_linear_fwd_hs /
          mux_linear(OP_BWD_DX) with Gs): no side tiles, extension blocks kept
  shrink  the side tiles alone (mux_linear_shrink / OP_SHRINK_BWD)
  cublas  torch.matmul of the backbone alone (no adapters), for scale
fused - given is the upper bound of the saving; given - cublas is the rest
(extension blocks + the kernel's own gap to cuBLAS).

usage: python tools/shrink_cost.py [--rows 11648 --tasks 4 --rank 16 --shapes 4096x4096,...]
One JSON line per (shape, pass).
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
    ap.add_argument("--rows", type=int, default=11648)
    ap.add_argument("--tasks", type=int, default=4)
    ap.add_argument("--rank", type=int, default=16)
    ap.add_argument("--iters", type=int, default=10)
    ap.add_argument("--rounds", type=int, default=9)
    ap.add_argument("--shapes", default="4096x4096,4096x11008,11008x4096")
    ap.add_argument("--label", default="")
    a = ap.parse_args()
    from paper_2603_02885_b200 import mux
    R, T, r = a.rows, a.tasks, a.rank
    r_cap = max(16, 16 * -(-r // 16))
    torch.manual_seed(0)
    for shp in a.shapes.split(","):
        K, N = (int(v) for v in shp.split("x"))
        X = torch.randn(R, K, device="cuda").bfloat16()
        W = (torch.randn(N, K, device="cuda") / K ** 0.5).bfloat16()
        dY = torch.randn(R, N, device="cuda").bfloat16()
        seg = R // T // 64 * 64
        seg_off = torch.tensor([i * seg for i in range(T)] + [R], dtype=torch.int32, device="cuda")
        ads = []
        for _ in range(T):
            B = mux.make_B_storage(N, r)
            B.copy_(torch.randn(N, r, device="cuda").bfloat16())
            ads.append(mux.Adapter((torch.randn(r, K, device="cuda") / K ** 0.5).bfloat16(), B, r, 2.0))
        st = list(range(T))
        ws = torch.zeros(mux.linear_workspace_size(T, R, K, N, r_cap), dtype=torch.uint8, device="cuda")
        Y = torch.empty(R, N, dtype=torch.bfloat16, device="cuda")
        Hs = torch.empty(R, r_cap, dtype=torch.bfloat16, device="cuda")
        Gs = torch.empty(R, r_cap, dtype=torch.bfloat16, device="cuda")
        dX = torch.empty(R, K, dtype=torch.bfloat16, device="cuda")
        mux.linear_fwd(seg_off, st, ads, X, W, r_cap, Y=Y, Hs=Hs, workspace=ws)
        mux.linear_shrink_bwd(seg_off, st, ads, dY, K, r_cap, Gs=Gs, workspace=ws)
        cands = {
            ("fwd", "fused"): lambda: mux.linear_fwd(seg_off, st, ads, X, W, r_cap, Y=Y, Hs=Hs, workspace=ws),
            ("fwd", "given"): lambda: mux.linear_fwd_hs(seg_off, st, ads, X, W, Hs, r_cap, Y=Y, workspace=ws),
            ("fwd", "shrink"): lambda: mux.linear_shrink(seg_off, st, ads, X, N, r_cap, Hs=Hs, workspace=ws),
            ("fwd", "cublas"): lambda: torch.matmul(X, W.t()),
            ("dX", "fused"): lambda: mux.linear_bwd(seg_off, st, ads, dY, X, W, Hs, r_cap, dX=dX, workspace=ws,
                                                    part=mux.BWD_DX),
            ("dX", "given"): lambda: mux.linear_bwd_gs(seg_off, st, ads, dY, X, W, Hs, Gs, r_cap, dX=dX,
                                                       workspace=ws, part=mux.BWD_DX),
            ("dX", "shrink"): lambda: mux.linear_shrink_bwd(seg_off, st, ads, dY, K, r_cap, Gs=Gs, workspace=ws),
            ("dX", "cublas"): lambda: torch.matmul(dY, W),
        }
        for f in cands.values():
            for _ in range(3):
                f()
        torch.cuda.synchronize()
        res = {k: [] for k in cands}
        for _ in range(a.rounds):
            for k, f in cands.items():
                res[k].append(time_once(f, a.iters))
        fl = 2 * R * K * N
        for ps in ("fwd", "dX"):
            med = {v: statistics.median(res[(ps, v)]) for v in ("fused", "given", "shrink", "cublas")}
            print(json.dumps({"label": a.label, "rows": R, "tasks": T, "rank": r, "K": K, "N": N, "pass": ps,
                              **{f"{v}_ms": round(m, 4) for v, m in med.items()},
                              "shrink_share": round((med["fused"] - med["given"]) / med["fused"], 4),
                              "fused_vs_cublas": round(med["cublas"] / med["fused"], 4),
                              "given_vs_cublas": round(med["cublas"] / med["given"], 4),
                              "backbone_tflops_fused": round(fl / med["fused"] / 1e9, 1)}), flush=True)


if __name__ == "__main__":
    main()
