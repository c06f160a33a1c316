# config-2 TP chain after the row-sizing fix (cap passed to the setup pack): rcr vs crc at world 1
timeout 900 python -m pytest -q tests/test_gpu_tp.py tests/test_gpu_tp_block.py -k "orchestrated or bench_gpus2" > gpurun_out/r02_t35.log 2>&1
tail -5 gpurun_out/r02_t35.log
rm -f gpurun_out/r02_chain_ab.jsonl
for c in rcr crc rcr crc; do
timeout 600 python bench.py --mode tp --gpus 1 --chain $c --steps 30 --warmup 5 --no-cpu-baseline 2>/dev/null | tail -1 >> gpurun_out/r02_chain_ab.jsonl
done
python - <<'PY'
import json
for l in open("gpurun_out/r02_chain_ab.jsonl"):
    d = json.loads(l); print(d["config"].get("parallelism"), round(d["value"]), d["ms_per_step"], d["e2e"]["value"], d["roofline"]["frac_of_burst"])
PY
