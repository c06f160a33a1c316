#!/usr/bin/env python
"""Write profiles/gemm_fwd_traffic.json from an ncu --set full capture of the
forward GEMM launches of one bench step (dram__bytes_read.sum +
dram__bytes_write.sum per launch), tagged with the sha256 of the libmux.so it
was captured on (bench.py reports the traffic only for that build).
usage: tools/traffic_json.py REP.ncu-rep [path/to/libmux.so]"""
import csv
import hashlib
import os
import io
import json
import subprocess
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2603_02885_b200.build import gemm_source_sha16  # noqa: E402

rep = sys.argv[1]
raw = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(raw)))
hdr, units = rows[0], rows[1]
scale = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}
per = []
for vals in rows[2:]:
    d = dict(zip(hdr, vals))
    name = d["Kernel Name"]
    # forward launches only (the capture may hold the dX GEMMs too): mux_gemm_kernel<kBwd = false, ...>
    if "mux_gemm_kernel<false" not in name and "mux_gemm_kernel<0" not in name:
        continue
    u = dict(zip(hdr, units))
    b = sum(float(d[k]) * scale[u[k]] for k in ("dram__bytes_read.sum", "dram__bytes_write.sum"))
    per.append({"kernel": d["Kernel Name"], "grid": d.get("launch__grid_size"), "dram_bytes": b,
                "duration_us": float(d["gpu__time_duration.sum"]) * (1e-3 if u["gpu__time_duration.sum"] == "ns"
                                                                      else 1.0)})
lib = sys.argv[2] if len(sys.argv) > 2 else os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))),
                                                          "paper_2603_02885_b200", "libmux.so")
out = {"source": f"ncu --set full ({rep}), forward GEMM launches of one bench step", "per_launch": per,
       "libmux_sha16": hashlib.sha256(open(lib, "rb").read()).hexdigest()[:16],
       "gemm_src_sha16": gemm_source_sha16(),
       "mean_bytes_per_launch": sum(x["dram_bytes"] for x in per) / max(1, len(per))}
json.dump(out, open("profiles/gemm_fwd_traffic.json", "w"), indent=1)
print(json.dumps(out, indent=1))
