#!/usr/bin/env python
"""Per-rank compute of tensor parallelism measured on one B200:
every linear of a config-4 / config-5 block at its p-way Megatron shard shape
(column-parallel q, k, v, gate, up: N/p; row-parallel o, down: K/p; sequence
parallelism gives every rank all T rows at the GEMM), fused fwd+bwd of the
packed multi-task call (16 / 32 tasks, ranks as the config), device time of a
CUDA graph.  Beside it, the per-rank collective bytes of one block step
(AG before q/k/v and gate/up, RS after o and down, and the mirrored pair in
backward: 8 collectives of (p-1)/p * T * H * 2 bytes) and the time they take at
the NVLink 5 per-direction peak of 900 GB/s — what must hide under the compute
for TP to scale.  One GPU only: the collectives themselves are not run here.
usage: python tools/tp_shard_profile.py [--out profiles/r01_tp_shard_profile.jsonl]
"""
import argparse
import json
import os
import statistics
import sys

import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

NVLINK_GBS = 900.0
COLUMN = {"q", "k", "v", "gate", "up"}


def time_graph(fn, reps=3):
    s = torch.cuda.Stream()
    s.wait_stream(torch.cuda.current_stream())
    with torch.cuda.stream(s):
        fn()
    torch.cuda.synchronize()
    g = torch.cuda.CUDAGraph()
    with torch.cuda.graph(g, stream=s):
        for _ in range(reps):
            fn()
    g.replay()
    torch.cuda.synchronize()
    vals = []
    for _ in range(5):
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record()
        g.replay()
        b.record()
        torch.cuda.synchronize()
        vals.append(a.elapsed_time(b) / reps)
    del g
    return statistics.median(vals)


FUSED = {"q": "qkv", "k": "qkv", "v": "qkv", "gate": "gate_up", "up": "gate_up"}


def groups_of(wl, fused):
    """The linears as calls: one per linear, or (fused) q|k|v and gate|up as one column-sliced call
    each (include/mux.h "Fused projections")."""
    out = []
    for L in wl.linears:
        key = FUSED.get(L.name, L.name) if fused else L.name
        if out and out[-1][0] == key:
            out[-1][1].append(L)
        else:
            out.append((key, [L]))
    return out


def block_at(mux, wl, p, shared_shrink=False, fused=False, parts=False):
    M = wl.num_tasks
    seg = -(-wl.valid_tokens // M // 64) * 64
    R = seg * M
    seg_off = torch.tensor([i * seg for i in range(M + 1)], dtype=torch.int32, device="cuda")
    st = list(range(M))
    gen = torch.Generator(device="cuda").manual_seed(0)
    r_cap = max(16, -(-max(wl.ranks) // 16) * 16)
    total_ms, flops, per = 0.0, 0.0, []
    for name, Ls in groups_of(wl, fused):
        L = Ls[0]
        col = L.name in COLUMN
        K = L.K if col else L.K // p
        widths = [(x.N // p if col else x.N) for x in Ls]
        N = sum(widths)
        col_off = [0]
        for w in widths:
            col_off.append(col_off[-1] + w)
        S = len(Ls)
        W = (torch.randn(N, K, device="cuda", generator=gen) / K ** 0.5).bfloat16()
        ads = []
        for r in wl.ranks:
            row = []
            for w in widths:
                B = mux.make_B_storage(w, r)
                B.copy_(torch.randn(w, r, device="cuda", generator=gen).bfloat16())
                row.append(mux.Adapter((torch.randn(r, K, device="cuda", generator=gen) / K ** 0.5).bfloat16(), B,
                                       r, 2.0, torch.empty(r, K, device="cuda"), torch.empty(w, r, device="cuda")))
            ads.append(row)
        X = torch.randn(R, K, device="cuda", generator=gen).bfloat16()
        dY = torch.randn(R, N, device="cuda", generator=gen).bfloat16()
        Y = torch.empty(R, N, dtype=torch.bfloat16, device="cuda")
        Hs = torch.empty(R, S * r_cap, dtype=torch.bfloat16, device="cuda")
        Gs = torch.empty(R, S * r_cap, dtype=torch.bfloat16, device="cuda")
        dX = torch.empty(R, K, dtype=torch.bfloat16, device="cuda")
        ws = torch.zeros(mux.linear_workspace_size(M, R, K, N, S * r_cap), dtype=torch.uint8, device="cuda")
        flat = [row[0] for row in ads]

        hi = -(-R // p // 256) * 256  # this rank's rows (rounded to pair blocks)

        def step():
            if S > 1:
                if shared_shrink and col:
                    mux.linear(mux.OP_SHRINK, seg_off, st, ads, col_off, K, N, r_cap, R, X=X, Hs=Hs, row_begin=0,
                               row_end=hi, workspace=ws)
                    mux.linear(mux.OP_FWD_HS, seg_off, st, ads, col_off, K, N, r_cap, R, X=X, W=W, Y=Y, Hs=Hs,
                               workspace=ws)
                else:
                    mux.linear(mux.OP_FWD, seg_off, st, ads, col_off, K, N, r_cap, R, X=X, W=W, Y=Y, Hs=Hs,
                               workspace=ws)
                mux.linear(mux.OP_BWD, seg_off, st, ads, col_off, K, N, r_cap, R, X=X, W=W, dY=dY, Hs=Hs, dX=dX,
                           workspace=ws, want_grads=True)
                return
            if shared_shrink and col:
                # tp.py shared_shrink: own rows' shrink, (Hs all-gather: T x r_cap, not run), then
                # the fused GEMM without shrink tiles
                mux.linear_shrink(seg_off, st, flat, X, N, r_cap, 0, hi, Hs=Hs, workspace=ws)
                mux.linear_fwd_hs(seg_off, st, flat, X, W, Hs, r_cap, Y=Y, workspace=ws)
            else:
                mux.linear_fwd(seg_off, st, flat, X, W, r_cap, Y=Y, Hs=Hs, workspace=ws)
            if shared_shrink and not col:
                # row-parallel backward: own rows' Gs (MUX_OP_SHRINK_BWD), (Gs all-gather, not run), then
                # the dX GEMM and gradients with Gs given
                mux.linear_shrink_bwd(seg_off, st, flat, dY, K, r_cap, 0, hi, Gs=Gs, workspace=ws)
                mux.linear_bwd_gs(seg_off, st, flat, dY, X, W, Hs, Gs, r_cap, dX=dX, workspace=ws)
            else:
                mux.linear_bwd(seg_off, st, flat, dY, X, W, Hs, r_cap, dX=dX, workspace=ws)

        ms = time_graph(step)
        split = None
        if parts:
            # the same call split into its launches: forward (with its shrink), dX GEMM, adapter gradients
            def fwd():
                if shared_shrink and col:
                    mux.linear(mux.OP_SHRINK, seg_off, st, ads, col_off, K, N, r_cap, R, X=X, Hs=Hs, row_begin=0,
                               row_end=hi, workspace=ws)
                    mux.linear(mux.OP_FWD_HS, seg_off, st, ads, col_off, K, N, r_cap, R, X=X, W=W, Y=Y, Hs=Hs,
                               workspace=ws)
                else:
                    mux.linear(mux.OP_FWD, seg_off, st, ads, col_off, K, N, r_cap, R, X=X, W=W, Y=Y, Hs=Hs,
                               workspace=ws)

            def dx():
                mux.linear(mux.OP_BWD_DX, seg_off, st, ads, col_off, K, N, r_cap, R, X=X, W=W, dY=dY, Hs=Hs, dX=dX,
                           Gs=Gs, workspace=ws)

            def grads():
                mux.linear(mux.OP_BWD_GRADS, seg_off, st, ads, col_off, K, N, r_cap, R, X=X, W=W, dY=dY, Hs=Hs,
                           Gs=Gs, workspace=ws, want_grads=True)
            dx()
            split = {k: round(time_graph(fn), 4) for k, fn in (("fwd", fwd), ("dx", dx), ("grads", grads))}
        f = sum(seg * (4 * K * w + 6 * r * (K + w)) for r in wl.ranks for w in widths)  # SURVEY §8(d) per token
        per.append({"linear": name, "K": K, "N": N, "slices": widths if S > 1 else None, "ms": round(ms, 4),
                    "tflops": round(f / ms / 1e9, 1), **({"parts_ms": split} if split else {})})
        total_ms += ms
        flops += f
        del W, ads, flat, X, dY, Y, Hs, Gs, dX, ws
        torch.cuda.empty_cache()
    H = wl.linears[0].K
    comm_bytes = 8 * (p - 1) / p * R * H * 2
    comm_ms = comm_bytes / (NVLINK_GBS * 1e9) * 1e3
    return {"config": wl.config_id, "tp": p, "shared_shrink": shared_shrink, "fused": fused, "rows": R, "tasks": M, "compute_ms_per_rank": round(total_ms, 3),
            "tflops_per_rank": round(flops / total_ms / 1e9, 1), "comm_bytes_per_rank": int(comm_bytes),
            "comm_ms_at_900GBs": round(comm_ms, 3), "comm_over_compute": round(comm_ms / total_ms, 3),
            "linears": per}


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--out", default=None)
    ap.add_argument("--points", default="4:1,4:2,4:4,4:8,5:1,5:8")
    ap.add_argument("--shared-shrink", action="store_true",
                    help="column layers: own-rows shrink + fwd_hs; row layers: own-rows Gs + bwd with Gs given")
    ap.add_argument("--fused", action="store_true", help="q|k|v and gate|up as one column-sliced call each")
    ap.add_argument("--parts", action="store_true", help="also time fwd / dX / gradients apart (through mux_linear; a row layer's dX part computes Gs "
                         "in the GEMM)")
    a = ap.parse_args()
    from paper_2603_02885_b200 import mux
    import synth
    out = open(a.out, "w") if a.out else None
    for pt in a.points.split(","):
        cid, p = pt.split(":")
        r = block_at(mux, synth.configs.workload(cid), int(p), a.shared_shrink, a.fused, a.parts)
        line = json.dumps(r)
        print(line, flush=True)
        if out:
            out.write(line + "\n")


if __name__ == "__main__":
    main()
