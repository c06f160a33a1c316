#!/usr/bin/env python
"""Write profiles/gemm_fwd_traffic.json from an ncu --set full capture of the
forward GEMM launches of one bench step (dram__bytes_read.sum +
dram__bytes_write.sum per launch).  usage: tools/traffic_json.py REP.ncu-rep"""
import csv
import io
import json
import subprocess
import sys

rep = sys.argv[1]
raw = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(raw)))
hdr, units = rows[0], rows[1]
scale = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}
per = []
for vals in rows[2:]:
    d = dict(zip(hdr, vals))
    if "<0>" not in d["Kernel Name"]:  # forward launches only (the capture may hold the dX GEMMs too)
        continue
    u = dict(zip(hdr, units))
    b = sum(float(d[k]) * scale[u[k]] for k in ("dram__bytes_read.sum", "dram__bytes_write.sum"))
    per.append({"kernel": d["Kernel Name"], "grid": d.get("launch__grid_size"), "dram_bytes": b,
                "duration_us": float(d["gpu__time_duration.sum"]) * (1e-3 if u["gpu__time_duration.sum"] == "ns"
                                                                      else 1.0)})
out = {"source": f"ncu --set full ({rep}), forward GEMM launches of one bench step", "per_launch": per,
       "mean_bytes_per_launch": sum(x["dram_bytes"] for x in per) / max(1, len(per))}
json.dump(out, open("profiles/gemm_fwd_traffic.json", "w"), indent=1)
print(json.dumps(out, indent=1))
