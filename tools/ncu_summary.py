#!/usr/bin/env python
"""Summarise ncu artefacts for profiles/: a launch list (--metrics
gpu__time_duration.sum csv) and/or full-set .ncu-rep captures.

usage: python tools/ncu_summary.py [--launches L.csv] [--rep R.ncu-rep ...] > profiles/rNN_*.md
"""
import argparse
import csv
import io
import subprocess
from collections import OrderedDict, defaultdict

KEYS = [
    "gpu__time_duration.sum", "sm__cycles_elapsed.avg.per_second",
    "sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_elapsed",
    "sm__throughput.avg.pct_of_peak_sustained_elapsed",
    "dram__bytes_read.sum", "dram__bytes_write.sum",
    "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed",
    "dram__throughput.avg.pct_of_peak_sustained_elapsed",
    "lts__throughput.avg.pct_of_peak_sustained_elapsed",
    "lts__t_sector_hit_rate.pct",
    "l1tex__throughput.avg.pct_of_peak_sustained_elapsed",
    "launch__grid_size", "launch__block_size", "launch__registers_per_thread",
    "launch__shared_mem_per_block_dynamic",
]


def launches(path):
    rows = list(csv.reader(open(path)))
    hdr = None
    agg = OrderedDict()
    for r in rows:
        if r and r[0] == "ID":
            hdr = r
            continue
        if not hdr or len(r) != len(hdr):
            continue
        d = dict(zip(hdr, r))
        if d["Metric Name"] != "gpu__time_duration.sum":
            continue
        name = d["Kernel Name"].split("(")[0]
        v = float(d["Metric Value"].replace(",", ""))
        if d["Metric Unit"] == "us":
            v *= 1e3
        elif d["Metric Unit"] == "ms":
            v *= 1e6
        agg.setdefault(name, []).append(v)
    tot = sum(sum(v) for v in agg.values())
    out = ["| kernel | launches | mean us | total us | share |", "|---|---|---|---|---|"]
    for k, v in sorted(agg.items(), key=lambda kv: -sum(kv[1])):
        out.append(f"| `{k}` | {len(v)} | {sum(v)/len(v)/1e3:.1f} | {sum(v)/1e3:.1f} | {sum(v)/tot:.3f} |")
    return "\n".join(out)


def rep(path):
    raw = subprocess.run(["ncu", "-i", path, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(raw)))
    hdr, units = rows[0], rows[1]
    out = []
    for vals in rows[2:]:
        d = dict(zip(hdr, vals))
        u = dict(zip(hdr, units))
        out.append(f"### `{d.get('Kernel Name', '?')}` (ID {d.get('ID', '?')})\n")
        out.append("| metric | value | unit |\n|---|---|---|")
        for k in KEYS:
            if k in d:
                out.append(f"| {k} | {d[k]} | {u.get(k, '')} |")
        out.append("")
    return "\n".join(out)


if __name__ == "__main__":
    ap = argparse.ArgumentParser()
    ap.add_argument("--launches")
    ap.add_argument("--rep", nargs="*", default=[])
    a = ap.parse_args()
    if a.launches:
        print("## Launch list (ncu --metrics gpu__time_duration.sum, cold-cache, serialised)\n")
        print(launches(a.launches))
        print()
    for r in a.rep:
        print(f"## Full-set capture: {r}\n")
        print(rep(r))
