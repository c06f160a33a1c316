#!/usr/bin/env python
"""Measured operator profiles for the hTask planner (planner.py, NEXT-4) and
the task-count sweep of SURVEY §8(d) config 2 (the B200 analogue of P:528,
"batching 8 tasks ... only improves throughput by 1.12x").

1. For each config-2 linear (4096->4096, 4096->11008, 11008->4096): fused
   fwd+bwd latency (mux_linear_fwd + mux_linear_bwd, one segment) at packed
   token counts x in --tokens, with rank 0 (BaseOp only, t_o(x)) and with one
   rank-r adapter (t_o(x) + t_a(x)).  -> profiles/r02_op_profile.json
2. Task-count sweep: m tasks x --per-task tokens each, rank r, multiplexed in
   one call per linear vs the same m tasks run one after another (temporal
   interleaving on one GPU), tokens/s of each; and the planner's choice for
   that task set from the measured profile (single stage, S = 1, C = 1).
   -> appended to the same JSON as "sweep".

Timing: CUDA events around --iters back-to-back launches, median of --rounds.
"""
import argparse
import json
import os
import statistics
import sys

import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

SHAPES = [(4096, 4096), (4096, 11008), (11008, 4096)]


def timed(fn, iters, rounds):
    vals = []
    for _ in range(rounds):
        s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        s.record()
        for _ in range(iters):
            fn()
        e.record()
        torch.cuda.synchronize()
        vals.append(s.elapsed_time(e) / iters)
    return statistics.median(vals)


class LayerSet:
    """Device buffers for the three linears at up to `rows` packed rows and
    up to `tasks` adapters of rank `rank`."""

    def __init__(self, mux, rows, tasks, rank):
        self.mux, self.rows = mux, rows
        g = torch.Generator(device="cuda").manual_seed(0)
        self.r_cap = max(16, 16 * -(-rank // 16))
        self.L = []
        for K, N in SHAPES:
            W = (torch.randn(N, K, device="cuda", generator=g) / K ** 0.5).bfloat16()
            ads = []
            for _ in range(tasks):
                B = mux.make_B_storage(N, rank)
                B.copy_(torch.randn(N, rank, device="cuda", generator=g).bfloat16())
                ads.append(mux.Adapter((torch.randn(rank, K, device="cuda", generator=g) / K ** 0.5).bfloat16(),
                                       B, rank, 2.0,
                                       torch.empty(rank, K, dtype=torch.float32, device="cuda"),
                                       torch.empty(N, rank, dtype=torch.float32, device="cuda")))
            self.L.append({"K": K, "N": N, "W": W, "ads": ads,
                           "X": torch.randn(rows, K, device="cuda", generator=g).bfloat16(),
                           "dY": torch.randn(rows, N, device="cuda", generator=g).bfloat16(),
                           "Y": torch.empty(rows, N, dtype=torch.bfloat16, device="cuda"),
                           "Hs": torch.empty(rows, self.r_cap, dtype=torch.bfloat16, device="cuda"),
                           "dX": torch.empty(rows, K, dtype=torch.bfloat16, device="cuda"),
                           "ws": torch.zeros(mux.linear_workspace_size(tasks, rows, K, N, self.r_cap),
                                             dtype=torch.uint8, device="cuda")})

    def run(self, li, seg_off, seg_task, ads, rows):
        """fused fwd + bwd of linear li over the first `rows` packed rows."""
        m, d = self.mux, self.L[li]
        X, dY = d["X"][:rows], d["dY"][:rows]
        Y, Hs, dX = d["Y"][:rows], d["Hs"][:rows], d["dX"][:rows]
        m.linear_fwd(seg_off, seg_task, ads, X, d["W"], self.r_cap, Y=Y, Hs=Hs, workspace=d["ws"])
        m.linear_bwd(seg_off, seg_task, ads, dY, X, d["W"], Hs, self.r_cap, dX=dX, workspace=d["ws"])


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--tokens", default="256,512,1024,2048,4096,8192,16384")
    ap.add_argument("--rank", type=int, default=16)
    ap.add_argument("--per-task", type=int, default=1024)
    ap.add_argument("--sweep", default="1,2,4,8,16")
    ap.add_argument("--iters", type=int, default=10)
    ap.add_argument("--rounds", type=int, default=5)
    ap.add_argument("--out", default=os.path.join(ROOT, "profiles", "r02_op_profile.json"))
    a = ap.parse_args()
    from paper_2603_02885_b200 import mux, planner
    toks = [int(v) for v in a.tokens.split(",")]
    sweep = [int(v) for v in a.sweep.split(",")]
    max_rows = max(max(toks), max(sweep) * a.per_task)
    ls = LayerSet(mux, max_rows, max(sweep), a.rank)
    i32 = dict(dtype=torch.int32, device="cuda")
    prof = {"device": torch.cuda.get_device_name(), "rank": a.rank, "linears": [],
            "note": "fused fwd+bwd ms per linear at x packed tokens (one segment); ms_rank0 = BaseOp only"}
    for li, (K, N) in enumerate(SHAPES):
        r0, rr = [], []
        for x in toks:
            so = torch.tensor([0, x], **i32)
            none = [mux.Adapter(None, None, 0, 0.0)]
            one = [ls.L[li]["ads"][0]]
            r0.append(timed(lambda: ls.run(li, so, [0], none, x), a.iters, a.rounds))
            rr.append(timed(lambda: ls.run(li, so, [0], one, x), a.iters, a.rounds))
        prof["linears"].append({"shape": [K, N], "tokens": toks, "ms_rank0": r0, "ms_rank": rr})
        print(json.dumps(prof["linears"][-1]), flush=True)
    stage = planner.stage_from_profile(prof)
    L = planner.htask_latency([stage], C=1)
    prof["sweep"] = []
    for m in sweep:
        rows = m * a.per_task
        so = torch.tensor([i * a.per_task for i in range(m + 1)], **i32)
        fused = timed(lambda: [ls.run(li, so, list(range(m)), ls.L[li]["ads"][:m], rows) for li in range(3)],
                      max(1, a.iters // 2), a.rounds)
        so1 = torch.tensor([0, a.per_task], **i32)

        def interleaved():
            for t in range(m):
                for li in range(3):
                    ls.run(li, so1, [0], [ls.L[li]["ads"][t]], a.per_task)
        inter = timed(interleaved, max(1, a.iters // 2), a.rounds)
        tasks = [planner.Task(f"t{t}", a.per_task, a.rank) for t in range(m)]
        plan = planner.fuse_tasks(tasks, L, S=1)
        rec = {"tasks": m, "tokens_per_task": a.per_task, "fused_ms": fused, "interleaved_ms": inter,
               "fused_tok_s": rows / fused * 1e3, "interleaved_tok_s": rows / inter * 1e3,
               "fused_over_interleaved": inter / fused,
               "model_fused_ms": L([a.per_task] * m), "model_interleaved_ms": m * L([a.per_task]),
               "planner_htasks": [len(h) for h in plan.htasks]}
        prof["sweep"].append(rec)
        print(json.dumps(rec), flush=True)
    os.makedirs(os.path.dirname(a.out), exist_ok=True)
    with open(a.out, "w") as f:
        json.dump(prof, f, indent=1)


if __name__ == "__main__":
    main()
