#!/usr/bin/env python
"""Run the fused GEMM from a -DMUX_PROFILE build (libmux_prof.so) on the
config-2 shapes and print where each role's cycles go (fraction of the role's
lifetime spent waiting on each barrier)."""
import ctypes
import json
import os
import sys

import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def main():
    from paper_2603_02885_b200 import mux
    mux.LIB_PATH = os.path.join(ROOT, "paper_2603_02885_b200", os.environ.get("MUX_PROF_LIB", "libmux_prof.so"))
    mux._lib = None
    L = mux.lib()
    L.mux_debug_counters.argtypes = [ctypes.c_void_p, ctypes.c_int]
    R = int(os.environ.get("MUX_ROWS", "11648"))
    rank = int(sys.argv[1]) if len(sys.argv) > 1 else 16
    shapes = [(4096, 4096), (4096, 11008), (11008, 4096)]
    if len(sys.argv) > 2:  # e.g. 512x4096,4096x512 (tensor-parallel shard shapes)
        shapes = [tuple(int(v) for v in x.split("x")) for x in sys.argv[2].split(",")]
    for K, N in shapes:
        X = torch.randn(R, K, device="cuda").bfloat16()
        W = (torch.randn(N, K, device="cuda") / K ** 0.5).bfloat16()
        dY = torch.randn(R, N, device="cuda").bfloat16()
        T = int(os.environ.get("MUX_TASKS", "4"))   # MUX_TASKS=16 MUX_MIXED=1: config-4 style ranks 8/16/32/64
        seg = R // T // 64 * 64
        seg_off = torch.tensor([i * seg if i < T else R for i in range(T + 1)], dtype=torch.int32, device="cuda")
        ranks = [(8, 16, 32, 64)[t % 4] for t in range(T)] if os.environ.get("MUX_MIXED") else [rank] * T
        ads = []
        for r in ranks:
            B = mux.make_B_storage(N, r)
            B.copy_(torch.randn(N, r, device="cuda").bfloat16())
            ads.append(mux.Adapter((torch.randn(r, K, device="cuda") / K ** 0.5).bfloat16(), B, r, 2.0))
        r_cap = max(16, 16 * -(-max(ranks) // 16))
        ws = torch.zeros(mux.linear_workspace_size(T, R, K, N, r_cap), dtype=torch.uint8, device="cuda")
        Y = torch.empty(R, N, dtype=torch.bfloat16, device="cuda")
        Hs = torch.empty(R, r_cap, dtype=torch.bfloat16, device="cuda")
        dX = torch.empty(R, K, dtype=torch.bfloat16, device="cuda")
        st = list(range(T))
        for name, fn in [("fwd", lambda: mux.linear_fwd(seg_off, st, ads, X, W, r_cap, Y=Y, Hs=Hs, workspace=ws)),
                         ("bwd", lambda: mux.linear_bwd(seg_off, st, ads, dY, X, W, Hs, r_cap, dX=dX,
                                                         workspace=ws, part=mux.BWD_DX))]:
            fn()
            buf = (ctypes.c_ulonglong * 64)()
            L.mux_debug_counters(buf, 64)
            for _ in range(5):
                fn()
            L.mux_debug_counters(buf, 64)
            c = list(buf)[:12]
            out = {"shape": f"{K}x{N}", "pass": name, "rank": rank, "tasks": T, "rows": R,
                   "mma_wait_full": c[1] / max(c[0], 1), "mma_wait_tmem_empty": c[2] / max(c[0], 1),
                   "producer_wait_empty": c[4] / max(c[3], 1), "producer_setup": c[7] / max(c[3], 1),
                   "producer_issue": c[8] / max(c[3], 1), "producer_flag_wait": c[9] / max(c[3], 1),
                   "epilogue_wait_tmem_full": c[6] / max(c[5], 1), "epilogue_wait_store_buf": c[10] / max(c[5], 1),
                   "producer_cycles_per_main_tile": c[3] / max(c[11], 1)}
            print(json.dumps(out), flush=True)


if __name__ == "__main__":
    main()
