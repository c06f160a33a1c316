#!/usr/bin/env python
"""Run the three config-2 forward GEMMs once (for an ncu DRAM-traffic capture of a
given libmux build: MUX_LIB=<file> under paper_2603_02885_b200/)."""
import os
import sys

import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def main():
    from paper_2603_02885_b200 import mux
    mux.LIB_PATH = os.path.join(ROOT, "paper_2603_02885_b200", os.environ.get("MUX_LIB", "libmux.so"))
    mux._lib = None
    R = 11648
    torch.manual_seed(0)
    for K, N in [(4096, 4096), (4096, 11008), (11008, 4096)]:
        X = torch.randn(R, K, device="cuda").bfloat16()
        W = (torch.randn(N, K, device="cuda") / K ** 0.5).bfloat16()
        seg_off = torch.tensor([0, 2944, 5888, 8768, R], dtype=torch.int32, device="cuda")
        ads = []
        for _ in range(4):
            B = mux.make_B_storage(N, 16)
            B.copy_(torch.randn(N, 16, device="cuda").bfloat16())
            ads.append(mux.Adapter((torch.randn(16, K, device="cuda") / K ** 0.5).bfloat16(), B, 16, 2.0))
        mux.linear_fwd(seg_off, [0, 1, 2, 3], ads, X, W, 16)
        torch.cuda.synchronize()


if __name__ == "__main__":
    main()
