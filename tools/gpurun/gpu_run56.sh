# Carrier NaN-isolation test, then the §8(d) sweeps, the planner's operator profile and the alignment
# sweep re-measured on the final (carrier) build
timeout 900 python -m pytest tests/test_gpu_carry.py -m gpu -q > gpurun_out/r02_carry6_tests.log 2>&1; echo "pytest rc=$?" >> gpurun_out/r02_carry6_tests.log
tail -2 gpurun_out/r02_carry6_tests.log
timeout 900 python tools/sweep.py --out gpurun_out/r02_sweep_carry.jsonl > gpurun_out/sweep.log 2>&1
timeout 900 python tools/op_profile.py --out gpurun_out/r02_op_profile_carry.json > gpurun_out/op_profile.log 2>&1
timeout 900 python tools/alignment_sweep.py --out gpurun_out/r02_alignment_sweep_carry.jsonl > gpurun_out/align.log 2>&1
tail -3 gpurun_out/sweep.log gpurun_out/op_profile.log gpurun_out/align.log
