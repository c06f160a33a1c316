#!/usr/bin/env python
"""NEXT-2: chunk-based alignment vs zero-padding to the global max length
(the SL-PEFT strategy) on the paper's task mixes, on B200.

Workloads: `tab:workloads` WL-A / WL-B task order and batch sizes
 with the per-dataset padded lengths SST2 64 / QA 128 / RTE 256
(P:944), plus a raw-length variant (lengths uniform below each dataset's
pad length).  Shapes: LLaMA-7B decoder linears 4096->4096, 4096->11008,
11008->4096 (rank 16 LoRA, s = 2).  Strategies:
  zero-pad : every sequence padded to the global max length, one segment per
             task of b_t * L_max rows;
  chunk c  : mux_pack_chunks with chunk_size c in {64, 128, 256}.
Reports per strategy: executed rows, effective fraction (valid/rows),
fwd+bwd ms through the 3 linears, overall rows/s and effective tokens/s,
and the effective-throughput ratio vs zero-pad (the paper's P:1126-1129
reports 3.59x/2.57x effective for chunk 64/128 on a 4-GPU pipeline with
attention; this sweep is the linear-layer-only B200 analogue).
Prints one JSON line per (workload, strategy).
"""
import json
import os
import sys

import numpy as np
import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import synth  # noqa: E402
from synth import gen  # noqa: E402

PAD = {"SST2": 64, "QA": 128, "RTE": 256}
WL = {"WL-A": ["SST2", "QA", "QA", "SST2", "SST2", "SST2", "QA", "QA"],
      "WL-B": ["RTE", "SST2", "RTE", "SST2", "SST2", "RTE", "RTE", "RTE"]}
BSZ = [4, 2, 4, 4, 8, 2, 4, 4]
SHAPES = [(4096, 4096), (4096, 11008), (11008, 4096)]


def task_lens(wl, raw, mult, seed):
    out = []
    st = gen.Stream(seed, first=500)
    for d, b in zip(WL[wl], BSZ):
        n = b * mult
        if raw:
            out.append(gen.seq_lengths(seed, st.take(), n, max(8, PAD[d] // 4), PAD[d]))
        else:
            out.append(np.full(n, PAD[d], np.int32))
    return out


def run(mux, seg_off, R, layers, r_cap, iters=20):
    X = torch.randn(R, SHAPES[0][0], device="cuda").bfloat16()
    tasks = len(layers[0]["ads"])
    st = list(range(tasks))

    def step():
        x = X
        for ly in layers:
            ly["Y"], ly["Hs"] = mux.linear_fwd(seg_off, st, ly["ads"], x, ly["W"], r_cap, Y=ly.get("Y"),
                                               Hs=ly.get("Hs"), workspace=ly["ws"])
            x = ly["Y"]
        dy = torch.ones_like(x) if "dy" not in layers[-1] else layers[-1]["dy"]
        layers[-1]["dy"] = dy
        for i in reversed(range(len(layers))):
            ly = layers[i]
            xin = X if i == 0 else layers[i - 1]["Y"]
            dy = mux.linear_bwd(seg_off, st, ly["ads"], dy, xin, ly["W"], ly["Hs"], r_cap, dX=ly.get("dX"),
                                workspace=ly["ws"])
            ly["dX"] = dy

    for _ in range(3):
        step()
    torch.cuda.synchronize()
    s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    s.record()
    for _ in range(iters):
        step()
    e.record()
    torch.cuda.synchronize()
    return s.elapsed_time(e) / iters


def main():
    from paper_2603_02885_b200 import mux
    torch.manual_seed(0)
    rank, r_cap, M = 16, 16, 8
    for wl in ("WL-A", "WL-B"):
        for raw in (False, True):
            for mult in (4,):
                lens_t = task_lens(wl, raw, mult, 2603028850)
                off = np.concatenate([[0], np.cumsum([len(x) for x in lens_t])]).astype(np.int32)
                lens = np.concatenate(lens_t).astype(np.int32)
                T = int(lens.sum())
                lmax = int(lens.max())
                strategies = [("zero-pad", None)] + [(f"chunk{c}", c) for c in (64, 128, 256)]
                base_eff = None
                for name, c in strategies:
                    if c is None:
                        # one segment per task of b_t * round_up(L_max, 64) rows (segments must be 64-aligned)
                        L = -(-lmax // 64) * 64
                        seg = np.concatenate([[0], np.cumsum([len(x) * L for x in lens_t])]).astype(np.int32)
                        R = int(seg[-1])
                        seg_off = torch.from_numpy(seg).cuda()
                    else:
                        bound = int(mux.pack_bound_rows(T, len(lens), c))
                        o = mux.pack_chunks(off, lens, None, c, 64, max_rows=bound, max_chunks=bound // 64)
                        info = mux.read_info(o["info"])
                        R = info["total_rows"]
                        seg_off = o["seg_off"]
                    layers = []
                    for K, N in SHAPES:
                        ads = []
                        for t in range(M):
                            B = mux.make_B_storage(N, rank)
                            B.copy_((torch.randn(N, rank, device="cuda") / 4).bfloat16())
                            ads.append(mux.Adapter((torch.randn(rank, K, device="cuda") / K ** 0.5).bfloat16(), B,
                                                   rank, 2.0))
                        layers.append({"W": (torch.randn(N, K, device="cuda") / K ** 0.5).bfloat16(), "ads": ads,
                                       "ws": torch.zeros(mux.linear_workspace_size(M, R, K, N, r_cap),
                                                         dtype=torch.uint8, device="cuda")})
                    ms = run(mux, seg_off, R, layers, r_cap)
                    eff = T / (ms * 1e-3)
                    if base_eff is None:
                        base_eff = eff
                    print(json.dumps({"workload": wl + (" raw" if raw else " padded(P:944)") + f" x{mult}",
                                      "strategy": name, "rows": R, "valid_tokens": T,
                                      "effective_fraction": T / R, "ms_fwd_bwd_3_linears": ms,
                                      "rows_per_s": R / (ms * 1e-3), "effective_tokens_per_s": eff,
                                      "effective_vs_zero_pad": eff / base_eff}), flush=True)
                    del layers
                    torch.cuda.empty_cache()


if __name__ == "__main__":
    main()
