# multi-slice gradients, per-slice epilogue (16-column TMEM loads): parity + per-part times
timeout 1200 python -m pytest -q -x tests/test_gpu_sliced.py tests/test_gpu_linear.py tests/test_gpu_wide.py > gpurun_out/r02_t38.log 2>&1
tail -3 gpurun_out/r02_t38.log
timeout 900 python tools/tp_shard_profile.py --points 4:8,5:8,4:4 --fused --shared-shrink --parts > gpurun_out/r02_tp_shard_parts_v3.jsonl 2>gpurun_out/tp_shard.err
python - <<'PY'
import json
for l in open("gpurun_out/r02_tp_shard_parts_v3.jsonl"):
    d = json.loads(l)
    print(d["config"], d["tp"], d["compute_ms_per_rank"], d["tflops_per_rank"], [(x["linear"], x["ms"], x.get("parts_ms")) for x in d["linears"]])
PY
tail -3 gpurun_out/tp_shard.err
