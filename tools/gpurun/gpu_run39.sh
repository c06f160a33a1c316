# where the TP-8 shard GEMMs (config 4) spend their time: per-part times + role wait fractions
timeout 900 python tools/tp_shard_profile.py --points 4:8 --fused --shared-shrink --parts > gpurun_out/r02_tp_shard_parts_v4.jsonl 2>gpurun_out/tp_shard.err
python - <<'PY'
import json
for l in open("gpurun_out/r02_tp_shard_parts_v4.jsonl"):
    d = json.loads(l)
    print(d["config"], d["tp"], d["compute_ms_per_rank"], d["tflops_per_rank"], [(x["linear"], x["ms"], x.get("parts_ms")) for x in d["linears"]])
PY
MUX_ROWS=21504 MUX_TASKS=16 MUX_MIXED=1 timeout 600 python tools/gemm_waits.py 64 512x4096,1376x4096,4096x1536,4096x2752 > gpurun_out/r02_waits_tp8.jsonl 2>&1
cat gpurun_out/r02_waits_tp8.jsonl
