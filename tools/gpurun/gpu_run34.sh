# config-2 TP chain pairing: rcr (row, col, row; default) vs crc, functional + world-1 timing
python -m paper_2603_02885_b200.build > /dev/null 2>&1 || python -c "import paper_2603_02885_b200.build as b; b.build()"
timeout 900 python -m pytest -q tests/test_gpu_tp.py tests/test_gpu_tp_block.py -k "orchestrated or bench_gpus2" > gpurun_out/r02_t34.log 2>&1
tail -5 gpurun_out/r02_t34.log
for c in rcr crc rcr crc; do
timeout 600 python bench.py --mode tp --gpus 1 --chain $c --steps 30 --warmup 5 --no-cpu-baseline 2>/dev/null | tail -1 >> gpurun_out/r02_chain_ab.jsonl
done
python - <<'PY'
import json
for l in open("gpurun_out/r02_chain_ab.jsonl"):
    d = json.loads(l); print(d["config"].get("parallelism"), round(d["value"]), d["ms_per_step"], d["e2e"]["value"])
PY
