#!/usr/bin/env python
"""Is the dX GEMM slower than the forward because W is read MN-major?  Interleaved A/B of
dX = dY W + s (dY B_t) A_t two ways on the same tensors: (mn) mux_linear_bwd's dX part, W [N, K]
read MN-major; (kmajor) the forward kernel on a transposed copy, Y' = dY (W^T)^T + Hs' B'^T with
A' = B_t^T and B' = A_t^T (the same product, every operand K-major).  Config-2 shapes, 11648 rows,
4 tasks r = 16 (--tasks/--rank to change).
usage: python tools/dx_layout_ab.py [--out profiles/r02_dx_layout_ab.jsonl]"""
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
    ap.add_argument("--tasks", type=int, default=4)
    ap.add_argument("--rank", type=int, default=16)
    ap.add_argument("--iters", type=int, default=10)
    ap.add_argument("--rounds", type=int, default=11)
    ap.add_argument("--shapes", default="4096x4096,4096x11008,11008x4096")
    ap.add_argument("--out", default=None)
    a = ap.parse_args()
    from paper_2603_02885_b200 import mux
    R, T, r = a.rows, a.tasks, a.rank
    rc = max(16, -(-r // 16) * 16)
    out = open(a.out, "a") if a.out else None
    torch.manual_seed(0)
    for shp in a.shapes.split(","):
        K, N = (int(v) for v in shp.split("x"))
        X = torch.randn(R, K, device="cuda").bfloat16()
        W = (torch.randn(N, K, device="cuda") / K ** 0.5).bfloat16()
        Wt = W.t().contiguous()
        dY = torch.randn(R, N, device="cuda").bfloat16()
        seg = R // T // 64 * 64
        seg_off = torch.tensor([i * seg if i < T else R for i in range(T + 1)], dtype=torch.int32, device="cuda")
        st = list(range(T))
        ads, ads_t = [], []
        for _ in range(T):
            A = (torch.randn(r, K, device="cuda") / K ** 0.5).bfloat16()
            B = mux.make_B_storage(N, r)
            B.copy_(torch.randn(N, r, device="cuda").bfloat16())
            ads.append(mux.Adapter(A, B, r, 2.0))
            Bt = mux.make_B_storage(K, r)          # B' = A^T [K, r]
            Bt.copy_(A.t())
            ads_t.append(mux.Adapter(B.t().contiguous(), Bt, r, 2.0))   # A' = B^T [r, N]
        Hs = torch.empty(R, rc, dtype=torch.bfloat16, device="cuda")
        Hs2 = torch.empty(R, rc, dtype=torch.bfloat16, device="cuda")
        dX = torch.empty(R, K, dtype=torch.bfloat16, device="cuda")
        dX2 = torch.empty(R, K, dtype=torch.bfloat16, device="cuda")
        ws = torch.zeros(mux.linear_workspace_size(T, R, K, N, rc), dtype=torch.uint8, device="cuda")
        ws2 = torch.zeros(mux.linear_workspace_size(T, R, N, K, rc), dtype=torch.uint8, device="cuda")
        mux.linear_fwd(seg_off, st, ads, X, W, rc, Hs=Hs, workspace=ws)
        impl = {
            "mn": lambda: mux.linear_bwd(seg_off, st, ads, dY, X, W, Hs, rc, dX=dX, workspace=ws, part=mux.BWD_DX),
            "kmajor": lambda: mux.linear_fwd(seg_off, st, ads_t, dY, Wt, rc, Y=dX2, Hs=Hs2, workspace=ws2),
        }
        for f in impl.values():
            f()
        torch.cuda.synchronize()
        err = float((dX.float() - dX2.float()).abs().max() / dX.float().abs().max())
        times = {k: [] for k in impl}
        for _ in range(a.rounds):
            for k, f in impl.items():
                e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                e0.record()
                for _ in range(a.iters):
                    f()
                e1.record()
                torch.cuda.synchronize()
                times[k].append(e0.elapsed_time(e1) / a.iters)
        flops = R * (2 * K * N + 2 * r * (K + N))
        for k in impl:
            med = statistics.median(times[k])
            line = {"shape": f"{K}x{N}", "dx_layout": k, "rows": R, "ms": round(med, 4),
                    "tflops": round(flops / med / 1e9, 1), "rel_diff_vs_mn": err}
            print(json.dumps(line), flush=True)
            if out:
                out.write(json.dumps(line) + "\n")


if __name__ == "__main__":
    main()
