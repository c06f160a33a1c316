# Carriers vs side tiles on the same build (MUX_CARRY=2 forces carriers everywhere they are legal, 0 = side
# tiles), config-2 and TP-8 shard shapes, interleaved; then the default bench against MUX_CARRY=0
timeout 900 python -m pytest tests/test_gpu_carry.py tests/test_gpu_linear.py -m gpu -x -q > gpurun_out/r02_carry4_tests.log 2>&1; echo "pytest rc=$?" >> gpurun_out/r02_carry4_tests.log
tail -2 gpurun_out/r02_carry4_tests.log
timeout 900 python tools/gemm_ab.py --env-ab MUX_CARRY=2,0 --no-cublas > gpurun_out/r02_carry4_envab_cfg2.jsonl 2>&1
timeout 900 python tools/gemm_ab.py --env-ab MUX_CARRY=2,0 --no-cublas --rows 21504 --tasks 16 --shapes 4096x512,4096x1536,512x4096,1376x4096,4096x2752 > gpurun_out/r02_carry4_envab_tp.jsonl 2>&1
cat gpurun_out/r02_carry4_envab_cfg2.jsonl gpurun_out/r02_carry4_envab_tp.jsonl
for i in 1 2 3; do
timeout 300 python bench.py --no-cpu-baseline > gpurun_out/r02_carry4_bench_$i.json 2>/dev/null; tail -1 gpurun_out/r02_carry4_bench_$i.json | cut -c1-200
MUX_CARRY=0 timeout 300 python bench.py --no-cpu-baseline > gpurun_out/r02_nocarry4_bench_$i.json 2>/dev/null; tail -1 gpurun_out/r02_nocarry4_bench_$i.json | cut -c1-200
done
