#!/usr/bin/env python
"""bench.py — multiplexed valid tokens/s, fwd+bwd, of MuxTune's hot path on B200.

Workload (BASELINE.json configs[1], "config 2"): LLaMA-7B-shaped decoder
linears chained as one layer stack 4096->4096 -> 4096->11008 -> 11008->4096,
4 LoRA tasks rank 16 (s = 2), 8 sequences per task, lengths U{128..512},
pack capacity 512.  One step = the whole hot path over one batch:
  mux_pack_chunks (chunk alignment)
  -> mux_pack_apply (Dispatch of the token-major layer input into packed rows)
  -> mux_linear_fwd x3 (fused backbone + LoRA, Eq. 1)
  -> mux_pack_apply (Dispatch of the loss gradient dY)
  -> mux_linear_bwd x3 (dX with LoRA + dA_t/dB_t, Eq. 2; dX of layer i is
     dY of layer i-1).
Metric: valid (non-pad) tokens / s (effective throughput).
Algorithmic FLOPs per valid token per linear K->N, rank r: 4KN + 6r(K+N).

N > 1 (torchrun): task-sharded replicas ("replicas only" for this path, see
DESIGN.md §Multi-GPU): every rank runs its own hTask of the same shape with a
rank-specific seed; no collective in the data path; scaling = weak; value =
tokens of all ranks / max-over-ranks time.
"""
from __future__ import annotations

import argparse
import json
import os
import statistics
import sys
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

import synth  # noqa: E402

# fused projections (q|k|v, gate|up as one column-sliced GEMM): the interleaved GEMM A/B in
# profiles/r02_fused_ab_v2.jsonl has the fused call at 0.68-0.99x the time of the separate calls (the
# gain grows as the shards narrow: 0.69 for TP-8 q|k|v dX); whole steps at full width are a wash
# (profiles/r02_bench_{tp4,block4}_ab.jsonl: TP arm at world 1 +0.5 %, the one-GPU block -1.8 %: its
# fused gate|up dX reduces over 22016 columns, and a row band of that A re-streams W twice as often as
# two 11008-deep dX GEMMs do, profiles/r02_block_launches_{fused,unfused}.md).  So auto fuses where a
# shard is narrower than the full 4096-wide 7B projections (every TP > 1 shard, config 5's k/v)
FUSE_BELOW_COLS = 4096
METRIC = "multiplexed tokens/s fwd+bwd at 1/2/4/8 B200; % of BF16 tensor-core peak"
UNIT = "tokens/s"


def peaks():
    p = os.path.join(ROOT, "MEASURED_PEAKS.json")
    try:
        d = json.load(open(p))
        return {"hbm_gbs": float(d["hbm_gbs"]), "bf16_tflops": float(d["bf16_tflops"]),
                "bf16_tflops_sustained": float(d.get("bf16_tflops_sustained", d["bf16_tflops"])),
                "source": "measured"}
    except Exception:
        return {"hbm_gbs": 6650.0, "bf16_tflops": 1590.0, "bf16_tflops_sustained": 1400.0,
                "source": "fallback (B200_PROFILING.md)"}


def flops_per_token(K, N, r):
    return 4 * K * N + 6 * r * (K + N)


# ------------------------------------------------------------------ workload
class Workload:
    def __init__(self, cid="2", rank_seed=0):
        self.wl = synth.workload(cid)
        if rank_seed:
            self.wl.seed = self.wl.seed + 1000 * rank_seed
            st = synth.Stream(self.wl.seed, first=1000)
            self.wl.task_lens = [synth.seq_lengths(self.wl.seed, st.take(), len(x), 128, 512)
                                 for x in self.wl.task_lens]
        wl = self.wl
        self.off, self.lens = wl.csr()
        self.T = wl.valid_tokens
        self.M = wl.num_tasks
        self.S = wl.num_seqs
        self.cap = wl.pack_capacity
        self.max_cap = max(self.cap) if self.cap else 512
        self.linears = wl.linears
        # algorithmic FLOPs at each task's own rank: sum_t T_t * sum_L (4KN + 6 r_t (K+N))
        self.task_tokens = [int(x.sum()) for x in wl.task_lens]
        self.flops = sum(Tt * flops_per_token(L.K, L.N, r) for Tt, r in zip(self.task_tokens, wl.ranks)
                         for L in wl.linears)

    def fwd_flops(self, L, K=None, N=None):
        """forward GEMM FLOPs of one call on linear L (or a K x N shard of it): sum_t T_t (2KN + 2 r_t (K+N))."""
        K = L.K if K is None else K
        N = L.N if N is None else N
        return sum(Tt * (2 * K * N + 2 * r * (K + N)) for Tt, r in zip(self.task_tokens, self.wl.ranks))

    def host_tensors(self):
        wl = self.wl
        h = {"X1": synth.token_input(wl, 0, "X", self.linears[0].K),
             "dY3": synth.token_input(wl, len(self.linears) - 1, "dY", self.linears[-1].N)}
        for li in range(len(self.linears)):
            h[f"W{li}"] = synth.weight(wl, li)
            for t in range(self.M):
                h[f"A{li}_{t}"], h[f"B{li}_{t}"] = synth.adapter(wl, li, t)
        return h


def _bits_to_dev(bits, torch):
    return torch.from_numpy(np.ascontiguousarray(bits).view(np.int16)).cuda().view(torch.bfloat16)


class MuxStep:
    """Device-resident buffers + one step of the hot path through the C ABI."""

    def __init__(self, w: Workload, torch, mux):
        self.w, self.torch, self.mux = w, torch, mux
        h = w.host_tensors()
        dev = "cuda"
        i32 = dict(dtype=torch.int32, device=dev)
        self.tso = [torch.tensor(w.off, **i32) for _ in range(2)]
        self.sl = [torch.tensor(w.lens, **i32) for _ in range(2)]
        self.cap = torch.tensor(w.cap, **i32) if w.cap else None
        self.max_rows = int(mux.pack_bound_rows(w.T, w.S, 64))
        self.max_chunks = self.max_rows // 64
        self.pk = mux.alloc_pack_outputs(w.M, w.S, self.max_rows, self.max_chunks, dev)
        # two input slots so the e2e loop can prefetch step i+1 while step i runs
        self.X1tok = [_bits_to_dev(h["X1"], torch) for _ in range(2)]
        self.dY3tok = [_bits_to_dev(h["dY3"], torch) for _ in range(2)]
        self.r_cap = 16 * -(-max(w.wl.ranks) // 16)
        self.seg_task = list(range(w.M))
        self.layers = []
        for li, L in enumerate(w.linears):
            ads = []
            for t in range(w.M):
                r = w.wl.ranks[t]
                B = mux.make_B_storage(L.N, r)
                B.copy_(_bits_to_dev(h[f"B{li}_{t}"], torch))
                ads.append(mux.Adapter(_bits_to_dev(h[f"A{li}_{t}"], torch), B, r, w.wl.scales[t],
                                       torch.empty(r, L.K, dtype=torch.float32, device=dev),
                                       torch.empty(L.N, r, dtype=torch.float32, device=dev)))
            self.layers.append({
                "L": L, "W": _bits_to_dev(h[f"W{li}"], torch), "ads": ads,
                "Y": torch.empty(self.max_rows, L.N, dtype=torch.bfloat16, device=dev),
                "Hs": torch.empty(self.max_rows, self.r_cap, dtype=torch.bfloat16, device=dev),
                "dX": torch.empty(self.max_rows, L.K, dtype=torch.bfloat16, device=dev),
                "ws": torch.zeros(mux.linear_workspace_size(w.M, self.max_rows, L.K, L.N, self.r_cap),
                                  dtype=torch.uint8, device=dev),
            })
        self.X1 = torch.empty(self.max_rows, w.linears[0].K, dtype=torch.bfloat16, device=dev)
        self.dY3 = torch.empty(self.max_rows, w.linears[-1].N, dtype=torch.bfloat16, device=dev)
        self.launches_per_step = 1 + 2 + len(self.layers) + 2 * len(self.layers)
        self.fwd_events = None
        # adapter gradients of layer l (HBM-bound) run on a side stream, in the tail of
        # the dX GEMM of layer l-1 (tensor-bound; its PDL-launched CTAs claim the SMs first)
        self.overlap_grads = True
        self.side = torch.cuda.Stream()
        self.gemm_done = [torch.cuda.Event() for _ in self.layers]

    def step(self, record=None, slot=0, before_bwd=None):
        mux, w = self.mux, self.w
        mux.pack_chunks(self.tso[slot], self.sl[slot], self.cap, 0, 64, max_rows=self.max_rows,
                        max_chunks=self.max_chunks, out=self.pk)
        seg_off = self.pk["seg_off"]
        mux.pack_apply(self.pk["row_src"], self.X1tok[slot], self.max_rows, out=self.X1)
        x = self.X1
        for li, ly in enumerate(self.layers):
            if record is not None:
                record("fwd", li, 0)
            mux.linear_fwd(seg_off, self.seg_task, ly["ads"], x, ly["W"], self.r_cap, Y=ly["Y"], Hs=ly["Hs"],
                           workspace=ly["ws"])
            if record is not None:
                record("fwd", li, 1)
            x = ly["Y"]
        mux.pack_apply(self.pk["row_src"], self.dY3tok[slot], self.max_rows, out=self.dY3)
        if before_bwd is not None:
            before_bwd()
        dy = self.dY3
        for li in reversed(range(len(self.layers))):
            ly = self.layers[li]
            xin = self.X1 if li == 0 else self.layers[li - 1]["Y"]
            if record is not None:
                record("bwd", li, 0)
            if not self.overlap_grads:
                mux.linear_bwd(seg_off, self.seg_task, ly["ads"], dy, xin, ly["W"], ly["Hs"], self.r_cap,
                               dX=ly["dX"], workspace=ly["ws"])
            else:
                main = self.torch.cuda.current_stream()
                mux.linear_bwd(seg_off, self.seg_task, ly["ads"], dy, xin, ly["W"], ly["Hs"], self.r_cap,
                               dX=ly["dX"], workspace=ly["ws"], part=mux.BWD_DX)
                self.gemm_done[li].record(main)
                self.side.wait_event(self.gemm_done[li])
                mux.linear_bwd(seg_off, self.seg_task, ly["ads"], dy, xin, ly["W"], ly["Hs"], self.r_cap,
                               dX=ly["dX"], workspace=ly["ws"], part=mux.BWD_GRADS, stream=self.side)
            if record is not None:
                record("bwd", li, 1)
            dy = ly["dX"]
        if self.overlap_grads:
            self.torch.cuda.current_stream().wait_stream(self.side)


# ------------------------------------------------------------------ clocks
class ClockSampler:
    """Samples SM clock, power and throttle reasons through NVML every 2 ms
    while the timed region runs (nvidia-smi's 100 ms floor would see only a
    handful of samples of a sub-second region).  The sampler is a separate
    process (no GIL contention with the launching thread; an in-process
    thread once got a single sample on a busy host), with an in-process
    thread as the fallback."""

    _CHILD = r"""
import json, select, sys, time
import pynvml as nv
nv.nvmlInit()
h = nv.nvmlDeviceGetHandleByIndex(int(sys.argv[1]))
print("ready", flush=True)
out = []
while not select.select([sys.stdin], [], [], 0)[0]:
    try:
        out.append((nv.nvmlDeviceGetClockInfo(h, nv.NVML_CLOCK_SM), nv.nvmlDeviceGetPowerUsage(h) / 1000.0,
                    nv.nvmlDeviceGetCurrentClocksEventReasons(h)))
    except Exception:
        pass
    time.sleep(0.002)
print(json.dumps(out), flush=True)
"""

    def __init__(self, gpu_index):
        self.idx = gpu_index
        self.samples = []
        self.stop_evt = None
        self.th = None
        self.proc = None
        self.err = None

    def start(self):
        import threading
        try:
            import pynvml as nv
            nv.nvmlInit()
            h = nv.nvmlDeviceGetHandleByIndex(self.idx)
            self.smax = nv.nvmlDeviceGetMaxClockInfo(h, nv.NVML_CLOCK_SM)
        except Exception as e:  # noqa: BLE001
            self.err = f"nvml unavailable: {e}"
            return
        try:
            import subprocess
            self.proc = subprocess.Popen([sys.executable, "-c", self._CHILD, str(self.idx)], stdin=subprocess.PIPE,
                                         stdout=subprocess.PIPE, stderr=subprocess.DEVNULL)
            if self.proc.stdout.readline().strip() != b"ready":
                raise RuntimeError("sampler process did not start")
            time.sleep(0.01)
            return
        except Exception:  # noqa: BLE001
            if self.proc is not None:
                self.proc.kill()
            self.proc = None
        self.stop_evt = threading.Event()

        def loop():
            while not self.stop_evt.is_set():
                try:
                    sm = nv.nvmlDeviceGetClockInfo(h, nv.NVML_CLOCK_SM)
                    pw = nv.nvmlDeviceGetPowerUsage(h) / 1000.0
                    rs = nv.nvmlDeviceGetCurrentClocksEventReasons(h)
                    self.samples.append((sm, pw, rs))
                except Exception:  # noqa: BLE001
                    pass
                time.sleep(0.002)
        self.th = threading.Thread(target=loop, daemon=True)
        self.th.start()
        time.sleep(0.01)

    def stop(self):
        src = "nvml, 2 ms, timed region only"
        if self.proc is not None:
            try:
                out, _ = self.proc.communicate(b"stop\n", timeout=30)
                self.samples = [tuple(x) for x in json.loads(out.decode().strip().splitlines()[-1])]
                src += " (sampler process)"
            except Exception as e:  # noqa: BLE001
                self.proc.kill()
                return {"sm_mhz": None, "sm_max_mhz": self.smax, "reasons": [f"sampler process failed: {e}"]}
        elif self.th is None:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": [self.err or "no sampler"]}
        else:
            self.stop_evt.set()
            self.th.join()
        import pynvml as nv
        names = {"hw_slowdown": nv.nvmlClocksEventReasonHwSlowdown,
                 "hw_thermal_slowdown": nv.nvmlClocksEventReasonHwThermalSlowdown,
                 "sw_thermal_slowdown": nv.nvmlClocksEventReasonSwThermalSlowdown,
                 "sw_power_cap": nv.nvmlClocksEventReasonSwPowerCap,
                 "hw_power_brake": nv.nvmlClocksEventReasonHwPowerBrakeSlowdown}
        if not self.samples:
            return {"sm_mhz": None, "sm_max_mhz": self.smax, "reasons": ["no samples"]}
        sm = [x[0] for x in self.samples]
        reasons = sorted({n for (_, _, r) in self.samples for n, b in names.items() if r & b})
        return {"sm_mhz": statistics.median(sm), "sm_max_mhz": self.smax, "reasons": reasons,
                "samples": len(sm), "power_w_max": max(x[1] for x in self.samples),
                "sm_mhz_min": min(sm), "source": src}


# ------------------------------------------------------------------ cpu / reference arm
def oracle_sample(w: Workload, rows_per_task: int, seed_off=0):
    """The oracle (as it stands) on a bounded sample of the workload: the same
    three linear shapes, tasks and ranks, with `rows_per_task` rows per task;
    full fwd (Y, Hs) + bwd (dX, dA_t, dB_t) on every sampled row."""
    from oracle import linear as olin
    wl = w.wl
    M = w.M
    seg_off = np.arange(M + 1, dtype=np.int32) * rows_per_task
    R = int(seg_off[-1])
    st = synth.Stream(wl.seed + 77 + seed_off)
    ranks, scales = wl.ranks, wl.scales
    r_cap = 16 * -(-max(ranks) // 16)
    data = []
    for li, L in enumerate(w.linears):
        X = synth.normal_bf16(wl.seed, st.take(), (R, L.K))
        dY = synth.normal_bf16(wl.seed, st.take(), (R, L.N))
        W = synth.weight(wl, li)
        A, B = zip(*[synth.adapter(wl, li, t) for t in range(M)])
        data.append((X, dY, W, list(A), list(B)))

    def run():
        for (X, dY, W, A, B) in data:
            olin.linear_fwd(seg_off, list(range(M)), A, B, ranks, scales, X, W, r_cap)
            olin.linear_bwd(seg_off, list(range(M)), A, B, ranks, scales, dY, X, W, r_cap)
    return run, R


def cpu_model():
    try:
        for line in open("/proc/cpuinfo"):
            if line.startswith("model name"):
                return line.split(":", 1)[1].strip()
    except OSError:
        pass
    return None


def cpu_baseline(w: Workload, target_s=12.0):
    """The oracle as it stands on the host cores (OpenMP over all of them), plus the same sample on
    one thread (core count, 1-thread figure and CPU model on record)."""
    from oracle import linear as olin
    olin.build()
    run, R = oracle_sample(w, 2)
    t0 = time.perf_counter()
    run()
    t1 = time.perf_counter() - t0
    rows_per_task = max(2, min(512, int(2 * target_s / max(t1, 1e-3))))
    run, R = oracle_sample(w, rows_per_task)
    t0 = time.perf_counter()
    run()
    dt = time.perf_counter() - t0
    cores = olin.num_threads()
    # one thread, a quarter of the rows (the per-token cost does not depend on the row count)
    rows1 = max(1, rows_per_task // 4)
    run1, R1 = oracle_sample(w, rows1)
    olin.set_num_threads(1)
    try:
        t0 = time.perf_counter()
        run1()
        dt1 = time.perf_counter() - t0
    finally:
        olin.set_num_threads(cores)
    return {"value": R / dt, "unit": UNIT, "cores": cores, "kind": "oracle", "cpu_model": cpu_model(),
            "sample": f"{R} tokens ({w.M} tasks x {rows_per_task} rows, ranks {w.wl.ranks}) through the "
                      f"3 config-2 linear shapes, full fp64 fwd+bwd (Y, Hs, dX, dA, dB); {dt:.1f} s",
            "seconds": dt,
            "one_thread": {"value": R1 / dt1, "unit": UNIT, "cores": 1, "seconds": dt1,
                           "sample": f"{R1} tokens ({w.M} tasks x {rows1} rows), same shapes"}}


def reference_arm(args):
    rank = int(os.environ.get("RANK", "0"))
    if rank != 0:
        return
    from oracle import linear as olin
    olin.build()
    w = Workload(args.config)
    rows_per_task = args.ref_rows
    run, R = oracle_sample(w, rows_per_task)
    for _ in range(args.warmup):
        run()
    t0 = time.perf_counter()
    for _ in range(args.steps):
        run()
    dt = (time.perf_counter() - t0) / args.steps
    v = R / dt
    cores = olin.num_threads()
    line = {"impl": "reference", "metric": METRIC, "value": v, "unit": UNIT, "n_gpus": args.gpus,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": dt * 1e3, "higher_is_better": True,
            "scaling": "weak", "vs_baseline": None, "dtype": "f64", "data": "synthetic",
            "config": {"workload": f"config {args.config}: " + w.wl.description,
                       "sample_tokens_per_step": R},
            "cpu_baseline": {"value": v, "unit": UNIT, "cores": cores, "kind": "oracle",
                             "sample": f"{R} tokens per step ({w.M} tasks x {rows_per_task} rows) through "
                                       "the 3 linear shapes, fp64 fwd+bwd"},
            "e2e": {"value": v, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
    print(json.dumps(line), flush=True)


# ------------------------------------------------------------------ main arm
def main_arm(args):
    import torch
    import torch.distributed as dist
    from paper_2603_02885_b200 import mux

    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    # MUX_BENCH_DIST_BACKEND=gloo (test only): exercise the N > 1 path with several ranks sharing
    # the visible GPUs (device = LOCAL_RANK mod count); the driver's runs use NCCL, one GPU per rank
    backend = os.environ.get("MUX_BENCH_DIST_BACKEND", "nccl")
    if backend != "nccl":
        local = local % torch.cuda.device_count()
    torch.cuda.set_device(local)
    if world > 1:
        if backend == "nccl":
            dist.init_process_group("nccl", device_id=torch.device("cuda", local))
        else:
            dist.init_process_group(backend)
    mux.lib()

    w = Workload(args.config, rank_seed=rank)
    bad = [i for i in range(1, len(w.linears)) if w.linears[i].K != w.linears[i - 1].N]
    if bad:  # e.g. config 4's seven block linears (gate's N = 11008 is not up's K = 4096)
        raise SystemExit(f"bench.py: config {args.config}'s linears do not chain as one layer stack (linear {bad[0]} "
                         f"has K = {w.linears[bad[0]].K}, the previous N = {w.linears[bad[0] - 1].N}); "
                         f"use --mode block (or --mode tp) for it")
    ms = MuxStep(w, torch, mux)
    ms.overlap_grads = not args.no_overlap_grads
    stream = torch.cuda.current_stream()

    for _ in range(args.warmup):
        ms.step()
    torch.cuda.synchronize()
    info = mux.read_info(ms.pk["info"])
    assert info["overflow"] == 0 and info["valid_rows"] == w.T, info

    # per-launch events for the fused GEMM (fwd calls) inside the timed region
    ev_pairs = {"fwd": [], "bwd": []}
    pending = {}

    def record(kind, li, which):
        e = torch.cuda.Event(enable_timing=True)
        e.record(stream)
        if which == 0:
            pending[(kind, li)] = e
        else:
            ev_pairs[kind].append((li, pending.pop((kind, li)), e))

    clocks = ClockSampler(local)
    if world > 1:
        dist.barrier()
    torch.cuda.synchronize()
    clocks.start()
    t_start = torch.cuda.Event(enable_timing=True)
    t_end = torch.cuda.Event(enable_timing=True)
    t_start.record(stream)
    for _ in range(args.steps):
        ms.step(record=record)
    t_end.record(stream)
    torch.cuda.synchronize()
    if world > 1:
        dist.barrier()
    clk = clocks.stop()
    ms_total = t_start.elapsed_time(t_end)
    t = torch.tensor([ms_total], dtype=torch.float64, device="cuda")
    if world > 1:
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
    ms_total = float(t.item())
    ms_step = ms_total / args.steps
    # every rank packs its own tasks (own seed): value counts the valid tokens of all ranks
    T_all = w.T
    if world > 1:
        tt = torch.tensor([w.T], dtype=torch.int64, device="cuda")
        dist.all_reduce(tt, op=dist.ReduceOp.SUM)
        T_all = int(tt.item())

    # roofline of the dominant kernel (fused tcgen05 GEMM, forward calls)
    fwd_ms = sum(a.elapsed_time(b) for (_, a, b) in ev_pairs["fwd"])
    bwd_ms = sum(a.elapsed_time(b) for (_, a, b) in ev_pairs["bwd"])
    fwd_flops = sum(w.fwd_flops(L) for L in w.linears) * args.steps
    # the events bracket each layer's backward call on the main stream: with the adapter gradients
    # overlapped on the side stream that is the dX GEMM (2KN + 2r(K+N) per token), else dX + gradients
    bwd_flops = sum(Tt * (2 * L.K * L.N + (2 if ms.overlap_grads else 4) * r * (L.K + L.N))
                    for L in w.linears for Tt, r in zip(w.task_tokens, w.wl.ranks)) * args.steps
    pk = peaks()
    achieved = fwd_flops / (fwd_ms * 1e-3) / 1e12
    roof = _roofline(achieved, pk, ms_total, clk, len(w.linears),
                     "mux_gemm_kernel<fwd> (fused backbone + LoRA; events around each mux_linear_fwd call)")
    roof["algorithmic_bytes_per_launch"] = sum(2 * (w.T * (L.K + L.N) + L.K * L.N) for L in w.linears) / len(w.linears)
    roof["traffic"], roof["traffic_source"] = traffic_of_this_build()

    # ---------------- e2e: same step through the public API with host buffers.
    # Every step copies its inputs host->device (pinned) and its result (all
    # adapter gradients) device->host inside the timed region.  Like a data
    # loader, the copy of step i+1's inputs runs on a copy stream while step i
    # computes (two input slots); the gradient read-back is on the compute
    # stream after the step.
    e2e = None
    if not args.no_e2e:
        pin = lambda t: t.cpu().pin_memory()  # noqa: E731
        h_in = [(pin(ms.tso[0]), pin(ms.sl[0]), pin(ms.X1tok[0]), pin(ms.dY3tok[0])) for _ in range(2)]
        grads = [a.dA for ly in ms.layers for a in ly["ads"]] + [a.dB for ly in ms.layers for a in ly["ads"]]
        h_grads = [torch.empty(g.shape, dtype=g.dtype, pin_memory=True) for g in grads]
        h2d = sum(x.numel() * x.element_size() for x in h_in[0])
        d2h = sum(g.numel() * g.element_size() for g in grads)
        # two H2D streams (the layer input and the loss gradient, 90 MB each at config 2, on separate
        # copy engines: one stream alone moved ~41 GB/s and bounded the step) and one D2H stream
        h2d_streams = [torch.cuda.Stream(), torch.cuda.Stream()]
        d2h_stream = torch.cuda.Stream()
        copied = [[torch.cuda.Event() for _ in range(2)] for _ in range(2)]   # [slot][h2d stream]
        consumed = [torch.cuda.Event() for _ in range(2)]
        step_done = torch.cuda.Event()
        d2h_done = torch.cuda.Event()

        def h2d_copy(i):
            slot = i % 2
            dsts = (ms.tso[slot], ms.sl[slot], ms.X1tok[slot], ms.dY3tok[slot])
            for j, cs in enumerate(h2d_streams):
                with torch.cuda.stream(cs):
                    cs.wait_event(consumed[slot])
                    for k, (dst, src) in enumerate(zip(dsts, h_in[slot])):
                        if (k == 3) == (j == 1):   # stream 1: dY; stream 0: metadata and X
                            dst.copy_(src, non_blocking=True)
                    copied[slot][j].record(cs)

        def e2e_run(n):
            for ev in consumed:
                ev.record(stream)
            d2h_done.record(stream)
            h2d_copy(0)
            for i in range(n):
                slot = i % 2
                if i + 1 < n:
                    h2d_copy(i + 1)
                for ev in copied[slot]:
                    stream.wait_event(ev)
                # the gradient read-back of step i-1 must finish before this step's backward
                # overwrites dA/dB
                ms.step(slot=slot, before_bwd=lambda: stream.wait_event(d2h_done))
                consumed[slot].record(stream)
                step_done.record(stream)
                with torch.cuda.stream(d2h_stream):
                    d2h_stream.wait_event(step_done)
                    for g, hg in zip(grads, h_grads):
                        hg.copy_(g, non_blocking=True)
                    d2h_done.record(d2h_stream)

        e2e_run(max(1, args.warmup))
        torch.cuda.synchronize()
        if world > 1:
            dist.barrier()
        e0 = torch.cuda.Event(enable_timing=True)
        e1 = torch.cuda.Event(enable_timing=True)
        e0.record(stream)
        for cs in h2d_streams + [d2h_stream]:
            cs.wait_event(e0)
        e2e_run(args.steps)
        for cs in h2d_streams + [d2h_stream]:
            stream.wait_stream(cs)
        e1.record(stream)
        torch.cuda.synchronize()
        te = torch.tensor([e0.elapsed_time(e1)], dtype=torch.float64, device="cuda")
        if world > 1:
            dist.all_reduce(te, op=dist.ReduceOp.MAX)
        e2e_ms = float(te.item()) / args.steps
        e2e = {"value": T_all / (e2e_ms * 1e-3), "unit": UNIT, "h2d_bytes_per_step": int(h2d),
               "d2h_bytes_per_step": int(d2h), "ms_per_step": e2e_ms,
               "what": "pinned H2D of seq metadata + token-major layer input X and loss gradient dY (prefetched "
                       "one step ahead on two copy streams); D2H of every adapter gradient dA_t/dB_t (fp32) on "
                       "a third stream, overlapped with the next step's forward"}

    value = T_all / (ms_step * 1e-3)
    tflops = w.flops / (ms_step * 1e-3) / 1e12
    line = {
        "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world, "steps": args.steps,
        "warmup": args.warmup, "ms_per_step": ms_step, "higher_is_better": True, "scaling": "weak",
        "vs_baseline": None, "dtype": "bf16", "data": "synthetic",
        "config": {"workload": f"config {args.config}: " + w.wl.description,
                   "layers": [f"{L.K}->{L.N}" for L in w.linears], "tasks": w.M, "ranks": w.wl.ranks,
                   "valid_tokens_per_gpu": w.T, "packed_rows": info["total_rows"],
                   "chunk_size": info["chunk_size"], "parallelism": f"replicas x{world} (task-sharded)",
                   "l2": "inputs larger than L2 (weights 214 MB + activations per step > 126 MB)"},
        "tflops_per_gpu_algorithmic": tflops,
        "frac_of_peak": {"measured_burst": tflops / pk["bf16_tflops"],
                         "measured_sustained": tflops / pk["bf16_tflops_sustained"],
                         "datasheet_2250": tflops / 2250.0},
        "kernels": {"fwd_calls_ms_per_step": fwd_ms / args.steps, "bwd_calls_ms_per_step": bwd_ms / args.steps,
                    "bwd_tflops": bwd_flops / (bwd_ms * 1e-3) / 1e12,
                    "bwd_calls": "dX GEMM only (adapter gradients overlapped on a side stream)"
                    if ms.overlap_grads else "dX GEMM + adapter gradients"},
        "roofline": roof,
        "clocks": clk,
        "gpu_launches": ms.launches_per_step * args.steps,
        "e2e": e2e,
    }
    if rank == 0 and world == 1 and not args.no_cpu_baseline:
        line["cpu_baseline"] = cpu_baseline(w, args.cpu_seconds)
    if rank == 0:
        print(json.dumps(line), flush=True)
    if world > 1:
        dist.destroy_process_group()


# ------------------------------------------------------------------ tensor-parallel arm
def dist_setup(torch):
    """One process per GPU (torchrun env).  NCCL over NVLink on the driver's runs;
    MUX_BENCH_DIST_BACKEND=gloo is test-only (ranks may then share the visible GPUs)."""
    import torch.distributed as dist
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    backend = os.environ.get("MUX_BENCH_DIST_BACKEND", "nccl")
    if backend != "nccl":
        local = local % torch.cuda.device_count()
    torch.cuda.set_device(local)
    if not dist.is_initialized():
        os.environ.setdefault("MASTER_ADDR", "127.0.0.1")
        os.environ.setdefault("MASTER_PORT", "29511")
        if backend == "nccl":
            dist.init_process_group("nccl", rank=rank, world_size=world, device_id=torch.device("cuda", local))
        else:
            dist.init_process_group(backend, rank=rank, world_size=world)
    return dist, world, rank, local, backend


def timed_backend_cls(tp, torch):
    class TimedMuxBackend(tp.MuxBackend):
        """tp.MuxBackend whose forward GEMM calls (the roofline's dominant kernel) are bracketed by
        CUDA events on the launching stream while `record` is a list; FLOPs per call are
        sum_t T_t (2 K N + 2 r_t (K + N)) over the call's tasks (`task_tokens`, host-known)."""
        record = None
        task_tokens = None

        def _flops(self, ads, K, N, col_off=None):
            if col_off is None:
                return sum(Tt * (2 * K * N + 2 * a.rank * (K + N)) for Tt, a in zip(self.task_tokens, ads))
            # fused projection: adapters[t][s] on column slices
            w = [col_off[i + 1] - col_off[i] for i in range(len(col_off) - 1)]
            return sum(Tt * sum(2 * K * n + 2 * a.rank * (K + n) for a, n in zip(row, w))
                       for Tt, row in zip(self.task_tokens, ads))

        def _timed(self, fn, flops, *a, **kw):
            if self.record is None:
                return fn(*a, **kw)
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record()
            out = fn(*a, **kw)
            e1.record()
            self.record.append((e0, e1, flops))
            return out

        def fwd(self, seg_off, seg_task, ads, X, W, r_cap, Y=None, col_off=None):
            return self._timed(super().fwd, self._flops(ads, X.shape[1], W.shape[0], col_off), seg_off, seg_task,
                               ads, X, W, r_cap, Y=Y, col_off=col_off)

        def fwd_hs(self, seg_off, seg_task, ads, X, W, Hs, r_cap, col_off=None):
            return self._timed(super().fwd_hs, self._flops(ads, X.shape[1], W.shape[0], col_off), seg_off, seg_task,
                               ads, X, W, Hs, r_cap, col_off=col_off)

        def fwd_rs(self, lay, seg_off, seg_task, X):
            return self._timed(super().fwd_rs, self._flops(lay.ads, X.shape[1], lay.W.shape[0]), lay, seg_off,
                               seg_task, X)

        def fwd_ag(self, lay, seg_off, seg_task, x_rows):
            return self._timed(super().fwd_ag, self._flops(lay.ads, x_rows.shape[1], lay.W.shape[0],
                                                           getattr(lay, "col_off", None)), lay, seg_off,
                               seg_task, x_rows)
    return TimedMuxBackend


def _gen(torch, seed, shape, std):
    g = torch.Generator(device="cuda").manual_seed(int(seed) & 0x7FFFFFFFFFFFFFFF)
    return (torch.randn(*shape, device="cuda", generator=g) * std).bfloat16()


def _packed_rows_once(torch, mux, task_off, lens, cap):
    """Setup only (outside every timed region): pack the workload once at its worst-case bound and
    read the packed row count, so the tensor-parallel buffers and collectives carry the rows the pack
    produces instead of the bound (+12 % at config 2)."""
    lens = [int(x) for x in lens]
    bound = int(mux.pack_bound_rows(sum(lens), len(lens), 64))
    pk = mux.pack_chunks([int(x) for x in task_off], lens, None if cap is None else [int(c) for c in cap], 0, 64,
                         max_rows=bound, max_chunks=bound // 64)
    info = mux.read_info(pk["info"])
    assert info["overflow"] == 0, info
    return int(info["total_rows"])


def _tp_chain(args, w, torch, mux, tp, orchestrate, Backend, world, rank):
    """Config-2-style layer stack (3 linears) tensor-parallel.  `--chain rcr` (default, Megatron's
    pairing for o / up / down): L0 row-parallel on the column shard of the input, RS of its output,
    AG into L1 column-parallel, L2 row-parallel on L1's column-sharded output (no collective), RS;
    every collective is K wide (4096), none crosses the 11008-wide intermediate.  `--chain crc`: L0
    column (AG of the row-sharded input), L1 row (RS), L2 column.  Backward mirrors either.
    `--htasks g` splits the tasks into g hTasks interleaved by Alg. 1 (orchestrate.py, NEXT-1)."""
    plan_note = None
    if args.htasks < 0:
        args.htasks = 2 if world > 1 else 1
    if args.htasks == 0:
        from paper_2603_02885_b200 import planner
        prof = planner.load_profile(os.path.join(ROOT, "profiles", "r02_op_profile.json"))
        L = planner.htask_latency([planner.stage_from_profile(prof, n_gpus=world)], C=1)
        tasks_ = [planner.Task(str(t), w.task_tokens[t], w.wl.ranks[t]) for t in range(w.M)]
        plan = planner.fuse_tasks(tasks_, L, S=1)
        groups = [[int(t.name) for t in h] for h in plan.htasks]
        plan_note = {"planner_cost_ms": plan.cost, "groups": groups}
    else:
        g = max(1, min(args.htasks, w.M))
        groups = [list(range(w.M))[i * w.M // g:(i + 1) * w.M // g] for i in range(g)]
    r_cap = 16 * -(-max(w.wl.ranks) // 16)
    kinds = (["row", "col", "row"] if args.chain == "rcr" else ["col", "row", "col"])[:len(w.linears)]
    first_row, last_row = kinds[0] == "row", kinds[-1] == "row"
    mk = lambda A, B, r, sc: mux.Adapter(A, B, r, sc)  # noqa: E731
    seed = w.wl.seed
    Wsh = []
    for li, L in enumerate(w.linears):
        W = _gen(torch, seed * 97 + li, (L.N, L.K), L.K ** -0.5)
        Wsh.append((tp.shard_column if kinds[li] == "col" else tp.shard_row)(W, [], world, rank, mk)[0])
        del W
    K0, Nl = w.linears[0].K, w.linears[-1].N
    i32 = dict(dtype=torch.int32, device="cuda")
    htasks, launches, grads, h2d = [], 0, [], []
    for hi, tasks in enumerate(groups):
        lens = [w.wl.task_lens[t] for t in tasks]
        off = np.concatenate([[0], np.cumsum([len(x) for x in lens])]).astype(np.int32)
        T_h = int(sum(int(x.sum()) for x in lens))
        S_h = int(off[-1])
        blk = 256 if (args.fused_rs or args.fused_ag) else 64
        # every rank owns an equal contiguous row block (sequence parallel); rows are sized once at
        # setup on this workload's packed row count (the step's lengths are fixed, so every step packs
        # the same rows; the timed loop never reads device data on the host)
        cap_h = [w.cap[t] for t in tasks] if w.cap else None
        packed = _packed_rows_once(torch, mux, off, np.concatenate(lens), cap_h)
        max_rows = -(-packed // (blk * world)) * blk * world
        pk = mux.alloc_pack_outputs(len(tasks), S_h, max_rows, max_rows // 64)
        be = Backend()
        be.task_tokens = [w.task_tokens[t] for t in tasks]
        be.pack_info = pk["info"]     # checked after the warm-up (no overflow: every row computed)
        layers = []
        for li, L in enumerate(w.linears):
            ads = []
            for t in tasks:
                r = w.wl.ranks[t]
                B = mux.make_B_storage(L.N, r)
                B.copy_(_gen(torch, seed * 131 + li * 1000 + t, (L.N, r), r ** -0.5))
                ads.append(mux.Adapter(_gen(torch, seed * 137 + li * 1000 + t, (r, L.K), L.K ** -0.5), B, r,
                                       w.wl.scales[t]))
            shard = tp.shard_column if kinds[li] == "col" else tp.shard_row
            _, ap_ = shard(torch.empty(L.N, L.K, dtype=torch.bfloat16, device="meta"), ads, world, rank, mk)
            cls = tp.ColumnParallelMuxLinear if kinds[li] == "col" else tp.RowParallelMuxLinear
            layers.append(cls(be, Wsh[li], ap_, r_cap, fused_rs=args.fused_rs, fused_ag=args.fused_ag))
        rows = max_rows // world
        lo, hi_ = rank * T_h // world, (rank + 1) * T_h // world
        # token-major inputs.  Column-parallel first layer: every rank holds the full buffer and its
        # data loader moves its 1/p token share (Dispatch gathers this rank's packed row block);
        # row-parallel first layer: the rank's column shard of every token (Dispatch packs all rows)
        Xtok = _gen(torch, seed * 7 + hi, (T_h, K0), 1.0)
        if first_row:
            Xtok = Xtok[:, rank * (K0 // world):(rank + 1) * (K0 // world)].contiguous()
        # loss gradient in the last layer's output layout: column-parallel -> this rank's column
        # shard of all rows [R, N/p]; row-parallel -> this rank's row block of full rows [R/p, N]
        dYtok = _gen(torch, seed * 11 + hi, (T_h, Nl), 1.0)
        if not last_row:
            dYtok = dYtok[:, rank * (Nl // world):(rank + 1) * (Nl // world)].contiguous()
        x_shape = (max_rows, K0 // world) if first_row else (rows, K0)
        dy_shape = (rows, Nl) if last_row else (max_rows, Nl // world)
        ht = {"tasks": tasks, "T": T_h, "max_rows": max_rows, "rows": rows, "pk": pk, "layers": layers,
              "tso": torch.tensor(off, **i32), "sl": torch.tensor(np.concatenate(lens).astype(np.int32), **i32),
              "cap": torch.tensor([w.cap[t] for t in tasks], **i32) if w.cap else None, "Xtok": Xtok,
              "x_rows": torch.empty(*x_shape, dtype=torch.bfloat16, device="cuda"),
              "dYtok": dYtok, "dY": torch.empty(*dy_shape, dtype=torch.bfloat16, device="cuda")}
        # host->device bytes per step: this rank's 1/p share of each token-major input
        h2d += [ht["tso"], ht["sl"], Xtok if first_row else Xtok[lo:hi_], dYtok[lo:hi_] if last_row else dYtok]

        def dispatch(e, ht=ht):
            mux.pack_chunks(ht["tso"], ht["sl"], ht["cap"], 0, 64, max_rows=ht["max_rows"],
                            max_chunks=ht["max_rows"] // 64, out=ht["pk"])
            mine = ht["pk"]["row_src"][rank * ht["rows"]:(rank + 1) * ht["rows"]]
            if first_row:
                mux.pack_apply(ht["pk"]["row_src"], ht["Xtok"], ht["max_rows"], out=ht["x_rows"])
            else:
                mux.pack_apply(mine, ht["Xtok"], ht["rows"], out=ht["x_rows"])
            if last_row:
                mux.pack_apply(mine, ht["dYtok"], ht["rows"], out=ht["dY"])
            else:
                mux.pack_apply(ht["pk"]["row_src"], ht["dYtok"], ht["max_rows"], out=ht["dY"])
            return ht["x_rows"]
        lat = [2.0 * max_rows * L.K * L.N / world for L in w.linears]
        ht["ops"] = orchestrate.linear_chain_ops(layers, kinds, ht["pk"]["seg_off"], list(range(len(tasks))),
                                                 dispatch, ht["dY"], lat)
        htasks.append(ht)
        launches += 3 + len(layers) + 2 * len(layers)   # pack + 2 Dispatch + fwd GEMMs + (dX + grads)
        grads.append(layers)
    dags = [orchestrate.build_subgraphs(i, ht["ops"]) for i, ht in enumerate(htasks)]
    schedule = orchestrate.subgraph_schedule(dags)

    def step():
        orchestrate.run_schedule(schedule, [dict() for _ in htasks])

    def result_tensors():
        out = []
        for layers in grads:
            for li, lay in enumerate(layers):
                col = kinds[li] == "col"
                for a in lay.ads:
                    if a.rank == 0:
                        continue
                    out.append(a.dB if col else a.dA)
                    if rank == 0:
                        out.append(a.dA if col else a.dB)
        return out

    names = {"col": "column", "row": "row"}
    desc = {"parallelism": f"tp{world} (" + ", ".join(f"L{i} {names[k]}" for i, k in enumerate(kinds))
            + "; sequence-parallel AG/RS)",
            "htasks": [ht["tasks"] for ht in htasks], "schedule": [f"h{sg.htask}.{sg.index}" for sg, _ in schedule],
            "planner": plan_note, "max_rows": [ht["max_rows"] for ht in htasks],
            "reduce_scatter": "fused into the GEMM epilogue (peer stores)" if args.fused_rs else "NCCL",
            "all_gather": "copy-engine push, consumed per row block by the GEMM" if args.fused_ag else "NCCL"}
    bes = [ht["layers"][0].be for ht in htasks]
    return step, launches, h2d, result_tensors, desc, bes


def _tp_block(args, w, torch, mux, tp, Backend, world, rank):
    """7-linear configs (4: LLaMA-7B block, 16 tasks; 5: LLaMA-70B shapes, 32 tasks): the whole
    decoder block tensor-parallel (tp_block.py): head-sharded attention between column q/k/v and
    row o, SwiGLU between column gate/up and row down, sequence-parallel RMSNorm/residuals."""
    from paper_2603_02885_b200 import tp_block
    from paper_2603_02885_b200.block import LINEARS
    wl = w.wl
    assert [L.name for L in wl.linears] == list(LINEARS), "TP block needs a 7-linear decoder config"
    hidden, ffn = wl.linears[0].K, wl.linears[4].N
    heads, kv_heads = wl.linears[0].N // 128, wl.linears[1].N // 128
    shape = tp_block.TPBlockShape(hidden=hidden, ffn=ffn, heads=heads, kv_heads=kv_heads, p=world)
    seed = wl.seed
    r_cap = 16 * -(-max(wl.ranks) // 16)
    mk = lambda A, B, r, sc: mux.Adapter(A, B, r, sc)  # noqa: E731
    Wfull, afull = {}, {}
    for li, L in enumerate(wl.linears):
        n = L.name
        Wfull[n] = _gen(torch, seed * 97 + li, (L.N, L.K), (0.5 if n in ("q", "k") else 1.0) * L.K ** -0.5)
        afull[n] = []
        for t in range(w.M):
            r = wl.ranks[t]
            B = _gen(torch, seed * 131 + li * 1000 + t, (L.N, r), r ** -0.5)
            A = _gen(torch, seed * 137 + li * 1000 + t, (r, L.K), L.K ** -0.5)
            afull[n].append(mux.Adapter(A, B, r, wl.scales[t]))

    for i in (1, 2):
        Wfull[f"norm{i}"] = (1.0 + 0.1 * torch.randn(hidden, device="cuda",
                                                      generator=torch.Generator(device="cuda").manual_seed(seed + i))
                             ).bfloat16()

    def padded(a):      # B rows need 16-byte alignment: copy into padded storage
        Bs = mux.make_B_storage(a.B.shape[0], a.rank)
        Bs.copy_(a.B)
        return mux.Adapter(a.A.contiguous(), Bs, a.rank, a.scale)
    col_off = None
    fuse = args.fused_proj
    if fuse < 0:            # auto: fuse where a per-rank projection shard is narrow (profiles/r02_fused_ab.jsonl)
        fuse = int(min(L.N // world for L in wl.linears if L.name in tp_block.COLUMN) < FUSE_BELOW_COLS)
    args.fused_proj = fuse
    if fuse:                # q|k|v and gate|up as one column-sliced GEMM each
        Wp, ap, col_off = tp_block.shard_block_fused(Wfull, afull, world, rank, mk)
        ap = {n: [[padded(a) for a in row] if isinstance(row, list) else padded(row) for row in v]
              for n, v in ap.items()}
    else:
        Wp, ap = tp_block.shard_block(Wfull, afull, world, rank, mk)
        ap = {n: [padded(a) for a in v] for n, v in ap.items()}
    del Wfull, afull
    be = Backend()
    be.task_tokens = list(w.task_tokens)
    if args.shared_shrink < 0:   # auto: at N > 1 each rank shrinks 1/N of the rows (tp.py shared_shrink)
        args.shared_shrink = int(world > 1)
    blk = tp_block.TPDecoderBlock(be, shape, Wp, ap, r_cap, col_off=col_off,
                                  shared_shrink=bool(args.shared_shrink))
    i32 = dict(dtype=torch.int32, device="cuda")
    tso, sl = torch.tensor(w.off, **i32), torch.tensor(w.lens, **i32)
    cap = torch.tensor(w.cap, **i32) if w.cap else None
    packed = _packed_rows_once(torch, mux, w.off, w.lens, w.cap)   # sized once at setup (see _tp_chain)
    blk_rows = 256 if args.shared_shrink else 64   # shared shrink: per-rank rows in whole pair row blocks
    max_rows = -(-packed // (blk_rows * world)) * blk_rows * world
    rows = max_rows // world
    pk = mux.alloc_pack_outputs(w.M, w.S, max_rows, max_rows // 64)
    rs = torch.empty(max_rows, **i32)
    Xtok = _gen(torch, seed * 7, (w.T, hidden), 1.0)
    dYtok = _gen(torch, seed * 11, (w.T, hidden), 1.0)
    x_rows = torch.empty(rows, hidden, dtype=torch.bfloat16, device="cuda")
    dy_rows = torch.empty(rows, hidden, dtype=torch.bfloat16, device="cuda")
    st = list(range(w.M))
    mine = slice(rank * rows, (rank + 1) * rows)

    def step():
        mux.pack_chunks(tso, sl, cap, 0, 64, max_rows=max_rows, max_chunks=max_rows // 64, out=pk)
        mux.row_start(sl, pk["seq_row"], max_rows, out=rs)
        mux.pack_apply(pk["row_src"][mine], Xtok, rows, out=x_rows)
        blk.forward(x_rows, pk["seg_off"], st, rs)
        mux.pack_apply(pk["row_src"][mine], dYtok, rows, out=dy_rows)
        blk.backward(dy_rows)

    lo, hi = rank * w.T // world, (rank + 1) * w.T // world
    h2d = [tso, sl, Xtok[lo:hi], dYtok[lo:hi]]

    def result_tensors():
        out = []
        for n, (dA, dB) in blk.adapter_grads().items():
            col = n in tp_block.COLUMN
            for a_, b_ in zip(dA, dB):
                if a_ is None:
                    continue
                out.append(b_ if col else a_)
                if rank == 0:
                    out.append(a_ if col else b_)
        return out

    pairs = sum(int(L) * (int(L) + 1) // 2 for x in wl.task_lens for L in x)
    attn_flops = 12 * 128 * heads * pairs
    desc = {"parallelism": f"tp{world} decoder block (column q/k/v/gate/up, head-sharded attention, row o/down; "
                           "sequence-parallel RMSNorm/residuals; 8 NCCL AG/RS per step)",
            "fused_projections": ("q|k|v and gate|up as one column-sliced GEMM each (per-slice adapters)"
                                  if args.fused_proj else None),
            "shared_shrink": bool(args.shared_shrink),
            "hidden": hidden, "ffn": ffn, "heads": heads, "kv_heads": kv_heads, "max_rows": max_rows,
            "attention_flops": attn_flops}
    lf, lb = blk.launches()
    launches = 4 + lf + lb + (2 if args.shared_shrink else 0)
    be.pack_info = pk["info"]
    return step, launches, h2d, result_tensors, desc, [be]


def tp_arm(args):
    """--mode tp (the default for --gpus N > 1): the workload tensor-parallel over the N ranks
    (strong scaling: the same tokens as N = 1, split over N GPUs).  Config 2 (3 linears): the layer
    stack L0 column / L1 row / L2 column (Megatron pairing; sequence-parallel AG/RS).
    Configs 4/5 (7 linears): the whole decoder block (tp_block.py).  Every rank's compute is the
    fused libmux kernels; collectives are NCCL (or fused into the GEMMs: --fused-rs/--fused-ag).
    Beside it (N > 1) the task-sharded replicas of the same config are timed as a secondary field
    ("weak" scaling: tasks are independent and the backbone frozen, so no collective at all)."""
    if args.comm_ctas:
        os.environ["NCCL_MAX_CTAS"] = str(args.comm_ctas)
    import torch
    from paper_2603_02885_b200 import mux, orchestrate, tp
    dist, world, rank, local, backend = dist_setup(torch)
    mux.lib()
    w = Workload(args.config)
    Backend = timed_backend_cls(tp, torch)
    if len(w.linears) == 7:
        step, launches, h2d_src, result_tensors, desc, bes = _tp_block(args, w, torch, mux, tp, Backend, world, rank)
        flops = w.flops + desc["attention_flops"]
    else:
        step, launches, h2d_src, result_tensors, desc, bes = _tp_chain(args, w, torch, mux, tp, orchestrate,
                                                                       Backend, world, rank)
        flops = w.flops
    stream = torch.cuda.current_stream()
    for _ in range(args.warmup):
        step()
    torch.cuda.synchronize()
    for be in bes:   # setup check outside the timed region: the step's pack fits its buffers
        if getattr(be, "pack_info", None) is not None:
            info = mux.read_info(be.pack_info)
            if info["overflow"]:
                raise RuntimeError(f"bench: the TP step's pack overflowed its buffers: {info}")
    rec = []
    for be in bes:
        be.record = rec
    clocks = ClockSampler(local)
    dist.barrier()
    torch.cuda.synchronize()
    clocks.start()
    s0, s1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    s0.record(stream)
    for _ in range(args.steps):
        step()
    s1.record(stream)
    torch.cuda.synchronize()
    dist.barrier()
    clk = clocks.stop()
    for be in bes:
        be.record = None
    t = torch.tensor([s0.elapsed_time(s1) / args.steps], dtype=torch.float64, device="cuda")
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    ms = float(t.item())
    # dominant kernel: the fused forward GEMM launches on this rank (max time over ranks)
    f_ms = torch.tensor([sum(a.elapsed_time(b) for a, b, _ in rec)], dtype=torch.float64, device="cuda")
    dist.all_reduce(f_ms, op=dist.ReduceOp.MAX)
    f_flops = sum(f for _, _, f in rec)
    pk = peaks()
    achieved = f_flops / (float(f_ms.item()) * 1e-3) / 1e12 if rec else None
    roof = _roofline(achieved, pk, ms * args.steps, clk, len(rec) // max(1, args.steps),
                     "mux_gemm_kernel<fwd> on this rank's shard (events around each forward call; max over ranks)")

    # e2e through the public API with host buffers: each rank copies its share of the inputs
    e2e = None
    if not args.no_e2e:
        e2e = _e2e_generic(torch, dist, stream, step, h2d_src, result_tensors(), args, w.T)
    line = {"metric": METRIC, "value": w.T / (ms * 1e-3), "unit": UNIT, "n_gpus": world, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": ms, "higher_is_better": True, "scaling": "strong",
            "vs_baseline": None, "dtype": "bf16", "data": "synthetic (seeded device normals)", "mode": "tp",
            "config": dict({"workload": f"config {args.config}: " + w.wl.description, "valid_tokens": w.T,
                            "tasks": w.M, "ranks": w.wl.ranks, "dist_backend": backend,
                            "l2": "inputs larger than L2 (weights + activations per step > 126 MB)"}, **desc),
            "tflops_per_gpu_algorithmic": flops / (ms * 1e-3) / 1e12 / world,
            "frac_of_peak_per_gpu": {"measured_burst": flops / (ms * 1e-3) / 1e12 / world / pk["bf16_tflops"],
                                     "measured_sustained": flops / (ms * 1e-3) / 1e12 / world
                                     / pk["bf16_tflops_sustained"]},
            "roofline": roof, "clocks": clk, "gpu_launches": launches * args.steps, "e2e": e2e}
    if world > 1 and not args.no_replicas:
        line["replicas"] = _replicas_secondary(args, torch, dist, world, rank)
    if rank == 0:
        print(json.dumps(line), flush=True)
    dist.destroy_process_group()


def _replicas_secondary(args, torch, dist, world, rank):
    """Task-sharded replicas (no collective): every rank runs its own hTask of the config-2 shape."""
    from paper_2603_02885_b200 import mux
    w = Workload("2", rank_seed=rank)
    ms_ = MuxStep(w, torch, mux)
    for _ in range(args.warmup):
        ms_.step()
    torch.cuda.synchronize()
    dist.barrier()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record()
    for _ in range(args.steps):
        ms_.step()
    b.record()
    torch.cuda.synchronize()
    t = torch.tensor([a.elapsed_time(b) / args.steps], dtype=torch.float64, device="cuda")
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    tt = torch.tensor([w.T], dtype=torch.int64, device="cuda")
    dist.all_reduce(tt)
    return {"value": int(tt.item()) / (float(t.item()) * 1e-3), "unit": UNIT, "ms_per_step": float(t.item()),
            "scaling": "weak", "workload": "config 2 per rank (own seeded tasks), no collective in the data path"}


def traffic_of_this_build():
    """DRAM bytes per forward-GEMM launch from the ncu --set full capture in profiles/gemm_fwd_traffic.json
    (tools/traffic_json.py), used only if it was captured on THIS libmux.so or on a build of the same GEMM
    sources and flags (sha256 match, build.gemm_source_sha16); else null."""
    import hashlib
    tp_ = os.path.join(ROOT, "profiles", "gemm_fwd_traffic.json")
    lib = os.path.join(ROOT, "paper_2603_02885_b200", "libmux.so")
    if not os.path.exists(tp_) or not os.path.exists(lib):
        return None, "no capture"
    tj = json.load(open(tp_))
    sha = hashlib.sha256(open(lib, "rb").read()).hexdigest()[:16]
    from paper_2603_02885_b200.build import gemm_source_sha16
    src = gemm_source_sha16()
    if tj.get("libmux_sha16") != sha and tj.get("gemm_src_sha16") != src:
        return None, (f"capture is of another build (so {tj.get('libmux_sha16')} != {sha}, GEMM sources "
                      f"{tj.get('gemm_src_sha16')} != {src}): not reported")
    return tj.get("mean_bytes_per_launch"), tj.get("source")


def _roofline(achieved, pk, timed_ms, clk, launches_per_step, kernel):
    """frac against the measured BURST bf16 peak unless the clocks were actually held down: the burst
    figure is cuBLAS timed alone for ~ the same duration, the sustained one back to back for 4 s at
    the board's power cap.  A short region (< 1 s) whose MEDIAN SM clock stayed within 10 % of the
    maximum takes burst even if a few samples saw sw_power_cap (the cap then bit only briefly);
    a long region, a median clock well below max or a thermal/hw slowdown takes sustained.  Both
    fractions are reported."""
    reasons = set(clk.get("reasons") or [])
    hard = bool(reasons & {"hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown"})
    sm, sm_max = clk.get("sm_mhz"), clk.get("sm_max_mhz")
    held_down = sm is not None and sm_max and sm < 0.9 * sm_max
    throttled = hard or held_down or (sm is None and "sw_power_cap" in reasons)
    use_burst = timed_ms < 1000.0 and not throttled
    peak = pk["bf16_tflops"] if use_burst else pk["bf16_tflops_sustained"]
    return {"bound": "tensor", "achieved": achieved, "peak": peak, "unit": "TFLOP/s",
            "frac": None if achieved is None else achieved / peak,
            "frac_of_burst": None if achieved is None else achieved / pk["bf16_tflops"],
            "frac_of_sustained": None if achieved is None else achieved / pk["bf16_tflops_sustained"],
            "peak_kind": ("burst" if use_burst else "sustained") + f" (timed region {timed_ms:.0f} ms, "
                                                                   f"throttled={throttled})",
            "peak_source": pk["source"], "kernel": kernel, "launches_per_step": launches_per_step}


def _e2e_generic(torch, dist, stream, step, h2d_src, results, args, tokens):
    """The same step with its inputs copied host->device (pinned, prefetched one step ahead on a copy
    stream into a second slot) and its result read back device->host every step."""
    pin = lambda t: t.detach().cpu().pin_memory()  # noqa: E731
    host = [pin(t) for t in h2d_src]
    slots = [[torch.empty_like(t) for t in h2d_src] for _ in range(2)]
    h_res = [torch.empty(g.shape, dtype=g.dtype, pin_memory=True) for g in results]
    # the step rewrites its results in place: each step's results are staged on the device (one
    # multi-tensor copy, two slots) and read back from the stage, so the next step need not wait for
    # the read-back
    stage = [[torch.empty_like(g) for g in results] for _ in range(2)]
    h2d = sum(x.numel() * x.element_size() for x in host)
    d2h = sum(g.numel() * g.element_size() for g in results)
    # the inputs alternate over two H2D streams by size (separate copy engines), the read-back has its own
    h2ds = [torch.cuda.Stream(), torch.cuda.Stream()]
    cs = torch.cuda.Stream()
    order = sorted(range(len(host)), key=lambda k: -host[k].numel() * host[k].element_size())
    lane_of = {k: j % 2 for j, k in enumerate(order)}
    copied = [[torch.cuda.Event() for _ in range(2)] for _ in range(2)]
    consumed = [torch.cuda.Event() for _ in range(2)]
    done, read = torch.cuda.Event(), [torch.cuda.Event() for _ in range(2)]

    def run(n):
        for ev in consumed + read:
            ev.record(stream)

        def h2d_copy(i):
            for j, hs in enumerate(h2ds):
                with torch.cuda.stream(hs):
                    hs.wait_event(consumed[i % 2])
                    for k, (d_, h_) in enumerate(zip(slots[i % 2], host)):
                        if lane_of[k] == j:
                            d_.copy_(h_, non_blocking=True)
                    copied[i % 2][j].record(hs)
        h2d_copy(0)
        for i in range(n):
            if i + 1 < n:
                h2d_copy(i + 1)
            for ev in copied[i % 2]:
                stream.wait_event(ev)
            for d_, s_ in zip(h2d_src, slots[i % 2]):     # the step reads its inputs from their home
                d_.copy_(s_, non_blocking=True)
            consumed[i % 2].record(stream)
            step()
            if results:
                stream.wait_event(read[i % 2])             # stage slot free (read back two steps ago)
                torch._foreach_copy_(stage[i % 2], results)
            done.record(stream)
            with torch.cuda.stream(cs):
                cs.wait_event(done)
                for g, hg in zip(stage[i % 2], h_res):
                    hg.copy_(g, non_blocking=True)
                read[i % 2].record(cs)

    run(max(1, args.warmup))
    torch.cuda.synchronize()
    dist.barrier()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(stream)
    for s_ in h2ds + [cs]:
        s_.wait_event(e0)
    run(args.steps)
    for s_ in h2ds + [cs]:
        stream.wait_stream(s_)
    e1.record(stream)
    torch.cuda.synchronize()
    te = torch.tensor([e0.elapsed_time(e1) / args.steps], dtype=torch.float64, device="cuda")
    dist.all_reduce(te, op=dist.ReduceOp.MAX)
    e2e_ms = float(te.item())
    return {"value": tokens / (e2e_ms * 1e-3), "unit": UNIT, "h2d_bytes_per_step": int(h2d),
            "d2h_bytes_per_step": int(d2h), "ms_per_step": e2e_ms,
            "what": "per rank: pinned H2D of the sequence metadata and this rank's 1/p share of the token-major "
                    "input and loss gradient (a sharded data loader's bytes; prefetched one step ahead on two copy "
                    "streams, staged into the device buffers the step reads); D2H of this rank's adapter-gradient "
                    "shards (replicated all-reduced gradients only on rank 0), staged on the device and read back "
                    "overlapped with the next step"}


def block_arm(args):
    """--mode block: one LLaMA-7B decoder block (config 4: 16 tasks, ranks
    8/16/32/64, LoRA on all seven linears) fwd+bwd per step, on one GPU:
    pack -> row map -> Dispatch(X) -> block forward (RMSNorm, q/k/v, RoPE,
    causal attention inside packed sequences, o + residual, RMSNorm,
    gate/up, SwiGLU, down + residual) -> Dispatch(dY) -> block backward
    (paper_2603_02885_b200/block.py; every step a libmux kernel).
    Algorithmic FLOPs: each linear 4KN + 6 r_t (K+N) per valid token of task
    t; attention 12 d H per causal (query, key) pair (fwd 2 + bwd 4 matmuls)."""
    import torch
    from paper_2603_02885_b200 import mux
    from paper_2603_02885_b200.block import LINEARS, BlockShape, DecoderBlock

    cfg = "4" if args.config == "2" else args.config
    w = Workload(cfg)
    wl = w.wl
    assert [L.name for L in wl.linears] == list(LINEARS), "block mode needs a 7-linear decoder config"
    hidden, ffn = wl.linears[0].K, wl.linears[4].N
    heads = wl.linears[0].N // 128
    kv_heads = wl.linears[1].N // 128
    shape = BlockShape(hidden=hidden, ffn=ffn, heads=heads, kv_heads=kv_heads)
    h = w.host_tensors()
    dev = "cuda"
    W = {n: _bits_to_dev(h[f"W{li}"], torch) for li, n in enumerate(LINEARS)}
    W["norm1"] = _bits_to_dev(synth.norm_weight(wl, 0), torch)
    W["norm2"] = _bits_to_dev(synth.norm_weight(wl, 1), torch)
    ads = {}
    for li, n in enumerate(LINEARS):
        L = wl.linears[li]
        ads[n] = []
        for t in range(w.M):
            B = mux.make_B_storage(L.N, wl.ranks[t])
            B.copy_(_bits_to_dev(h[f"B{li}_{t}"], torch))
            ads[n].append(mux.Adapter(_bits_to_dev(h[f"A{li}_{t}"], torch), B, wl.ranks[t], wl.scales[t]))
    r_cap = 16 * -(-max(wl.ranks) // 16)
    if args.fused_proj < 0:     # auto (one GPU: full-width projections)
        args.fused_proj = int(min(L.N for L in wl.linears if L.name in ("q", "k", "v", "gate", "up"))
                              < FUSE_BELOW_COLS)
    blk = DecoderBlock(shape, W, ads, r_cap, fused=bool(args.fused_proj))
    blk.overlap_grads = not args.no_overlap_grads
    i32 = dict(dtype=torch.int32, device=dev)
    tso, sl = torch.tensor(w.off, **i32), torch.tensor(w.lens, **i32)
    cap = torch.tensor(w.cap, **i32) if w.cap else None
    max_rows = int(mux.pack_bound_rows(w.T, w.S, 64))
    pk = mux.alloc_pack_outputs(w.M, w.S, max_rows, max_rows // 64)
    rs = torch.empty(max_rows, **i32)
    Xtok = _bits_to_dev(synth.token_input(wl, 0, "X", hidden), torch)
    dYtok = _bits_to_dev(synth.token_input(wl, 6, "dY", hidden), torch)
    X = torch.empty(max_rows, hidden, dtype=torch.bfloat16, device=dev)
    dY = torch.empty(max_rows, hidden, dtype=torch.bfloat16, device=dev)
    st = list(range(w.M))

    def step():
        mux.pack_chunks(tso, sl, cap, 0, 64, max_rows=max_rows, max_chunks=max_rows // 64, out=pk)
        mux.row_start(sl, pk["seq_row"], max_rows, out=rs)
        mux.pack_apply(pk["row_src"], Xtok, max_rows, out=X)
        blk.forward(X, pk["seg_off"], st, rs)
        mux.pack_apply(pk["row_src"], dYtok, max_rows, out=dY)
        return blk.backward(dY)

    for _ in range(args.warmup):
        step()
    torch.cuda.synchronize()
    info = mux.read_info(pk["info"])
    assert info["overflow"] == 0 and info["valid_rows"] == w.T, info
    clk = ClockSampler(int(os.environ.get("LOCAL_RANK", "0")))
    clk.start()
    s0, s1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    torch.cuda.synchronize()
    s0.record()
    for _ in range(args.steps):
        step()
    s1.record()
    torch.cuda.synchronize()
    clocks = clk.stop()
    ms = s0.elapsed_time(s1) / args.steps
    # algorithmic FLOPs
    lin = 0
    for t in range(w.M):
        Tt = int(wl.task_lens[t].sum())
        lin += Tt * sum(flops_per_token(L.K, L.N, wl.ranks[t]) for L in wl.linears)
    pairs = sum(int(L) * (int(L) + 1) // 2 for x in wl.task_lens for L in x)
    attn = 12 * 128 * heads * pairs
    pk_ = peaks()
    tf = (lin + attn) / (ms * 1e-3) / 1e12
    print(json.dumps({"metric": METRIC, "value": w.T / (ms * 1e-3), "unit": UNIT, "n_gpus": 1,
                      "steps": args.steps, "warmup": args.warmup, "ms_per_step": ms, "higher_is_better": True,
                      "scaling": "weak", "vs_baseline": None, "dtype": "bf16", "data": "synthetic", "mode": "block",
                      "config": {"workload": f"config {cfg}: " + wl.description + " - one full decoder block "
                                 "(RMSNorm, q/k/v/o, RoPE, causal attention, SwiGLU MLP) fwd+bwd",
                                 "valid_tokens": w.T, "packed_rows": info["total_rows"], "tasks": w.M,
                                 "hidden": hidden, "ffn": ffn, "heads": heads, "kv_heads": kv_heads,
                                 "l2": "inputs larger than L2 (weights 405 MB)"},
                      "tflops_algorithmic": tf, "frac_of_sustained_peak": tf / pk_["bf16_tflops_sustained"],
                      "flops_split": {"linears": lin, "attention": attn},
                      "fused_projections": bool(args.fused_proj),
                      "gpu_launches": args.steps * (5 + sum(blk.launches())),
                      "clocks": clocks}), flush=True)


def spawn_ranks(n: int) -> int:
    """`python bench.py --gpus N` without torchrun: re-launch this command under torch.distributed.run,
    one process per GPU on this node (rendezvous on 127.0.0.1); rank 0 prints the JSON line.  NCCL's
    INIT/NVLS log goes to stderr (NCCL_DEBUG=INFO), so the rank count and NVLS use are on record."""
    import socket
    import subprocess
    s_ = socket.socket()
    s_.bind(("127.0.0.1", 0))
    port = s_.getsockname()[1]
    s_.close()
    env = dict(os.environ)
    env.setdefault("NCCL_DEBUG", "INFO")
    env.setdefault("NCCL_DEBUG_SUBSYS", "INIT,NVLS")
    env.setdefault("NCCL_DEBUG_FILE", "/dev/stderr")
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={n}",
           "--master-addr", "127.0.0.1", "--master-port", str(port), os.path.abspath(__file__)] + sys.argv[1:]
    return subprocess.call(cmd, env=env)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=50)
    ap.add_argument("--warmup", type=int, default=5)
    ap.add_argument("--impl", default="mux", choices=["mux", "reference"])
    ap.add_argument("--config", default="2")
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--no-overlap-grads", action="store_true",
                    help="run each layer's adapter gradients on the main stream (no side-stream overlap)")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--cpu-seconds", type=float, default=12.0)
    ap.add_argument("--ref-rows", type=int, default=4, help="rows per task per reference-arm step")
    ap.add_argument("--mode", default="auto", choices=["auto", "replicas", "tp", "block"],
                    help="auto: N=1 -> the single-GPU step (replicas x1), N>1 -> tensor parallel (strong scaling, "
                         "the north_star TP path) with the task-sharded replicas as a secondary field")
    ap.add_argument("--no-replicas", action="store_true", help="--mode tp, N>1: skip the secondary replicas timing")
    ap.add_argument("--htasks", type=int, default=-1,
                    help="--mode tp, config 2: hTasks interleaved by Alg. 1 (NEXT-1) so one hTask's collectives "
                         "overlap another's GEMMs; 0 = chosen by the planner (NEXT-4); -1 (default) = 2 for N > 1 "
                         "(at N = 1 the collectives are local copies: 1)")
    ap.add_argument("--chain", default="rcr", choices=("rcr", "crc"),
                    help="--mode tp, config 2: layer kinds of the 3-linear chain; rcr (default) = row, column, row "
                         "(collectives 4096 wide), crc = column, row, column (RS/AG of the 11008-wide intermediate)")
    ap.add_argument("--comm-ctas", type=int, default=0, help="--mode tp: NCCL_MAX_CTAS for the overlapped collectives")
    ap.add_argument("--fused-proj", type=int, default=-1, choices=(-1, 0, 1),
                    help="--mode tp / block, configs 4/5: q|k|v and gate|up as one column-sliced GEMM each (1), "
                         "seven separate linears (0), or auto (-1, default: fused where a per-rank projection "
                         f"shard is narrower than {FUSE_BELOW_COLS} columns)")
    ap.add_argument("--shared-shrink", type=int, default=-1, choices=(-1, 0, 1),
                    help="--mode tp, configs 4/5: column layers shrink only their own rows and all-gather Hs "
                         "(1), recompute every row's shrink on every rank (0), or auto (-1: on for N > 1)")
    ap.add_argument("--fused-rs", action="store_true",
                    help="--mode tp: reduce-scatters fused into the GEMMs (peer stores via symmetric memory)")
    ap.add_argument("--fused-ag", action="store_true",
                    help="--mode tp: all-gathers pushed by the copy engines, consumed inside the GEMMs")
    args = ap.parse_args()
    if args.warmup < 3:
        args.warmup = 3
    if args.gpus > 1 and "WORLD_SIZE" not in os.environ and args.impl != "reference":
        sys.exit(spawn_ranks(args.gpus))
    if args.mode == "auto":
        args.mode = "tp" if int(os.environ.get("WORLD_SIZE", "1")) > 1 else "replicas"
    if args.impl == "reference":
        reference_arm(args)
    elif args.mode == "tp":
        tp_arm(args)
    elif args.mode == "block":
        block_arm(args)
    else:
        main_arm(args)


if __name__ == "__main__":
    main()
