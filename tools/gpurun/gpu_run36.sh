# e2e with device-staged results (generic path: TP / block arms); per-part times of the fused TP shard calls
for c in rcr crc; do
timeout 600 python bench.py --mode tp --gpus 1 --chain $c --steps 30 --warmup 5 --no-cpu-baseline 2>/dev/null | tail -1 >> gpurun_out/r02_chain_ab_e2e.jsonl
done
python - <<'PY'
import json
for l in open("gpurun_out/r02_chain_ab_e2e.jsonl"):
    d = json.loads(l); print(d["config"].get("parallelism"), round(d["value"]), d["ms_per_step"], d["e2e"]["value"], d["e2e"]["ms_per_step"])
PY
timeout 900 python tools/tp_shard_profile.py --points 4:8,5:8,4:4 --fused --shared-shrink --parts > gpurun_out/r02_tp_shard_parts.jsonl 2>gpurun_out/tp_shard.err
cat gpurun_out/r02_tp_shard_parts.jsonl; tail -3 gpurun_out/tp_shard.err
