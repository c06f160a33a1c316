# Carrier fuzz on the final build
timeout 1200 python -m pytest tests/test_gpu_carry.py -m gpu -q > gpurun_out/r02_carry_fuzz.log 2>&1; echo "pytest rc=$?" >> gpurun_out/r02_carry_fuzz.log
tail -3 gpurun_out/r02_carry_fuzz.log
