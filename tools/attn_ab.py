#!/usr/bin/env python
"""Interleaved A/B timing of the packed causal attention (mux_attn_fwd /
mux_attn_bwd) across libmux builds on the config-4 layout (16 tasks x 4
sequences, lengths U{128..512}, 32 heads of 128).  Prints one JSON line per
(lib, pass): median ms over --rounds, algorithmic TFLOP/s (fwd 4 d H per
causal pair, bwd 8 d H)."""
import argparse
import json
import os
import statistics
import sys

import numpy as np
import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--libs", nargs="+", default=[os.path.join(ROOT, "paper_2603_02885_b200", "libmux.so")])
    ap.add_argument("--config", default="4")
    ap.add_argument("--heads", type=int, default=32)
    ap.add_argument("--kv-heads", type=int, default=32)
    ap.add_argument("--iters", type=int, default=10)
    ap.add_argument("--rounds", type=int, default=7)
    a = ap.parse_args()
    import synth
    from paper_2603_02885_b200 import mux
    wl = synth.workload(a.config)
    off, lens = wl.csr()
    T = int(lens.sum())
    max_rows = int(T + len(lens) * 64)
    pk = mux.pack_chunks(off, lens, wl.pack_capacity, 0, 64, max_rows=max_rows, max_chunks=max_rows // 64)
    rs = mux.row_start(torch.tensor(lens, dtype=torch.int32, device="cuda"), pk["seq_row"], max_rows)
    R, H, Hkv = max_rows, a.heads, a.kv_heads
    g = torch.Generator(device="cuda").manual_seed(0)
    q = torch.randn(R, H * 128, device="cuda", generator=g).bfloat16()
    k = torch.randn(R, Hkv * 128, device="cuda", generator=g).bfloat16()
    v = torch.randn(R, Hkv * 128, device="cuda", generator=g).bfloat16()
    dO = torch.randn(R, H * 128, device="cuda", generator=g).bfloat16()
    pairs = sum(int(L) * (int(L) + 1) // 2 for L in lens)
    fl = {"fwd": 4 * 128 * H * pairs, "bwd": 8 * 128 * H * pairs}
    handles = {}
    for lib in a.libs:
        mux.LIB_PATH = lib
        mux._lib = None
        handles[lib] = mux.lib()
    res = {(lib, ps): [] for lib in a.libs for ps in ("fwd", "bwd")}
    outs = {}
    for _ in range(a.rounds):
        for lib, hdl in handles.items():
            mux._lib = hdl
            o, lse = mux.attn_fwd(q, k, v, rs, H, Hkv, 128 ** -0.5)
            for ps in ("fwd", "bwd"):
                s0, s1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                s0.record()
                for _ in range(a.iters):
                    if ps == "fwd":
                        mux.attn_fwd(q, k, v, rs, H, Hkv, 128 ** -0.5, o=o, lse=lse)
                    else:
                        mux.attn_bwd(dO, q, k, v, o, lse, rs, H, Hkv, 128 ** -0.5)
                s1.record()
                torch.cuda.synchronize()
                res[(lib, ps)].append(s0.elapsed_time(s1) / a.iters)
            outs[lib] = o.clone()
    base = outs[a.libs[0]]
    for (lib, ps), v_ in res.items():
        ms = statistics.median(v_)
        diff = float((outs[lib].float() - base.float()).abs().max())
        print(json.dumps({"lib": os.path.basename(lib), "pass": ps, "ms": ms, "tflops": fl[ps] / ms / 1e9,
                          "rows": R, "heads": H, "kv_heads": Hkv, "pairs": pairs,
                          "max_abs_diff_o_vs_first_lib": diff}), flush=True)


if __name__ == "__main__":
    main()
