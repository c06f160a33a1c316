# L2 cache policies on the main-tile TMA loads (MUX_L2HINT 0 / a / 1 / 2): DRAM bytes (ncu), interleaved
# launch times, and the sustained / default-length bench
timeout 600 ncu -k regex:mux_gemm --metrics dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum --csv \
  python tools/raster_ab.py --var MUX_L2HINT --modes 0,a,1,2 --once > gpurun_out/r02_l2hint_ncu.csv 2>/dev/null
python - <<'PY'
import csv, io
rows = [r for r in csv.reader(open("gpurun_out/r02_l2hint_ncu.csv")) if len(r) > 10]
hdr = rows[0]; data = rows[1:]
iN, iM, iV, iU = hdr.index("Kernel Name"), hdr.index("Metric Name"), hdr.index("Metric Value"), hdr.index("Metric Unit")
per = {}
order = []
for r in data:
    key = r[0]
    if key not in per: per[key] = {}; order.append(key)
    per[key][r[iM]] = (r[iV], r[iU])
modes = ["0", "a", "1", "2"]
i = 0
for shp in ["4096x4096", "4096x11008", "11008x4096"]:
    for ps in ["fwd", "dx"]:
        for m in modes:
            d = per[order[i]]; i += 1
            print(shp, ps, m, {k: v for k, v in d.items()})
PY
timeout 900 python tools/raster_ab.py --var MUX_L2HINT --modes 0,a,1,2 > gpurun_out/r02_l2hint_ab.jsonl
cat gpurun_out/r02_l2hint_ab.jsonl
for i in 1 2; do
for h in 0 a; do
MUX_L2HINT=$h timeout 600 python bench.py --steps 300 --warmup 10 --no-cpu-baseline --no-e2e 2>/dev/null | tail -1 | python -c "
import json,sys; d=json.loads(sys.stdin.read()); print(json.dumps({'l2hint':'$h','steps':300,'value':d['value'],'ms':d['ms_per_step'],'sm_mhz':d['clocks']['sm_mhz'],'pw':d['clocks'].get('power_w_max'),'reasons':d['clocks']['reasons']}))" >> gpurun_out/r02_l2hint_bench.jsonl
done
done
for i in 1 2 3; do
for h in 0 a; do
MUX_L2HINT=$h timeout 600 python bench.py --no-cpu-baseline --no-e2e 2>/dev/null | tail -1 | python -c "
import json,sys; d=json.loads(sys.stdin.read()); print(json.dumps({'l2hint':'$h','steps':50,'value':d['value'],'ms':d['ms_per_step'],'sm_mhz':d['clocks']['sm_mhz'],'pw':d['clocks'].get('power_w_max'),'reasons':d['clocks']['reasons']}))" >> gpurun_out/r02_l2hint_bench.jsonl
done
done
cat gpurun_out/r02_l2hint_bench.jsonl
