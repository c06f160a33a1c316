set -x
timeout 900 python tools/op_profile.py --out gpurun_out/r02_op_profile.json > gpurun_out/op_profile.log 2>&1
timeout 900 python tools/sweep.py --out gpurun_out/r02_sweep.jsonl > gpurun_out/sweep.log 2>&1
timeout 900 python tools/alignment_sweep.py --out gpurun_out/r02_alignment_sweep.jsonl > gpurun_out/align.log 2>&1
timeout 300 python -m pytest -q tests/test_c_example.py tests/test_gpu_tp_block.py > gpurun_out/r02s2_t19.log 2>&1
tail -2 gpurun_out/r02s2_t19.log
