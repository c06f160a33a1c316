#!/usr/bin/env python
"""Time mux_pack_chunks on its own ("the pack kernel is timed on
its own"; bar <= 10 us at config 5) at the workloads of configs 2, 3b, 4, 5.

Three numbers per config: (1) back-to-back stream launches, events around 200
calls (includes launch gaps); (2) one CUDA graph of 50 pack calls, replayed
(device time per call without host launch cost); (3) with --profile, a
-DMUX_PACK_PROFILE build prints thread 0's clock64() phase deltas.
usage: python tools/pack_time.py [--configs 2,3b,4,5] [--profile]
"""
import argparse
import json
import os
import subprocess
import sys

import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--configs", default="2,3b,4,5")
    ap.add_argument("--profile", action="store_true")
    ap.add_argument("--lib", default=None)
    a = ap.parse_args()
    from paper_2603_02885_b200 import mux
    from paper_2603_02885_b200 import build as mbuild
    import synth
    if a.lib:
        mux.LIB_PATH, mux._lib = a.lib, None
    for cid in a.configs.split(","):
        wl = synth.configs.workload(cid)
        tso_h, sl_h = wl.csr()
        M, S = wl.num_tasks, wl.num_seqs
        max_rows = int(mux.pack_bound_rows(wl.valid_tokens, S, 64))
        max_chunks = max_rows // 64
        out = mux.alloc_pack_outputs(M, S, max_rows, max_chunks)
        tso = torch.from_numpy(tso_h).cuda()
        sl = torch.from_numpy(sl_h).cuda()
        cap = None if wl.pack_capacity is None else torch.tensor(wl.pack_capacity, dtype=torch.int32).cuda()

        def call():
            mux.pack_chunks(tso, sl, cap, wl.chunk_size, wl.chunk_min, max_rows=max_rows, max_chunks=max_chunks,
                            out=out)

        for _ in range(10):
            call()
        torch.cuda.synchronize()
        s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        n = 200
        s.record()
        for _ in range(n):
            call()
        e.record()
        torch.cuda.synchronize()
        stream_us = s.elapsed_time(e) / n * 1e3
        g = torch.cuda.CUDAGraph()
        st = torch.cuda.Stream()
        st.wait_stream(torch.cuda.current_stream())
        with torch.cuda.stream(st):
            call()
            torch.cuda.synchronize()
            with torch.cuda.graph(g, stream=st):
                for _ in range(50):
                    call()
        torch.cuda.synchronize()
        g.replay()
        torch.cuda.synchronize()
        s.record()
        for _ in range(4):
            g.replay()
        e.record()
        torch.cuda.synchronize()
        graph_us = s.elapsed_time(e) / 200 * 1e3
        print(json.dumps({"config": cid, "tasks": M, "seqs": S, "valid_tokens": wl.valid_tokens,
                          "max_rows": max_rows, "stream_us_per_call": round(stream_us, 2),
                          "graph_us_per_call": round(graph_us, 2)}), flush=True)
    if a.profile and not a.lib:
        lib = mbuild.build(defines=("MUX_PACK_PROFILE",), out="libmux_packprof.so")
        code = ("import sys; sys.argv=['x','--configs',%r,'--lib',%r]; sys.path.insert(0,%r); "
                "import runpy; runpy.run_path(%r, run_name='__main__')") % (a.configs, lib, ROOT, __file__)
        r = subprocess.run([sys.executable, "-c", code], capture_output=True, text=True)
        lines = [l for l in (r.stdout + r.stderr).splitlines() if l.startswith("pack_profile")]
        last = {}
        for l in lines:  # warm (last) calls per config
            key = l.split(" cycles")[0]
            last.setdefault(key, []).append(l)
        for key, ls in last.items():
            for l in ls[-2:]:
                print(l)


if __name__ == "__main__":
    main()
