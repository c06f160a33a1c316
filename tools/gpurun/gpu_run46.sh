# Carrier shrink, forward and backward (map_shrink; bwd B_t MN-major 32 B swizzle): parity, A/B, bench
timeout 900 python -m pytest tests/test_gpu_carry.py tests/test_gpu_linear.py tests/test_gpu_fullsize.py tests/test_gpu_graph.py tests/test_gpu_autograd.py tests/test_gpu_sliced.py -m gpu -x -q > gpurun_out/r02_carry2_tests.log 2>&1; echo "pytest rc=$?" >> gpurun_out/r02_carry2_tests.log
tail -3 gpurun_out/r02_carry2_tests.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke(); print('smoke ok')" > gpurun_out/r02_carry2_smoke.log 2>&1; tail -1 gpurun_out/r02_carry2_smoke.log
if grep -q "pytest rc=0" gpurun_out/r02_carry2_tests.log; then
timeout 600 python tools/gemm_ab.py --libs paper_2603_02885_b200/libmux_old.so paper_2603_02885_b200/libmux.so > gpurun_out/r02_carry2_ab_cfg2.jsonl 2>&1
timeout 600 python tools/gemm_ab.py --libs paper_2603_02885_b200/libmux_old.so paper_2603_02885_b200/libmux.so --rows 21504 --tasks 16 --shapes 4096x512,4096x1536,512x4096,1376x4096,4096x2752 --no-cublas > gpurun_out/r02_carry2_ab_tp.jsonl 2>&1
cat gpurun_out/r02_carry2_ab_cfg2.jsonl gpurun_out/r02_carry2_ab_tp.jsonl
MUX_CARRY=0 timeout 600 python tools/gemm_ab.py --libs paper_2603_02885_b200/libmux_old.so paper_2603_02885_b200/libmux.so --no-cublas > gpurun_out/r02_carry2_ab_cfg2_carry0.jsonl 2>&1
cat gpurun_out/r02_carry2_ab_cfg2_carry0.jsonl
timeout 600 python tools/shrink_cost.py --label config2-carry > gpurun_out/r02_shrink_cost_carry.jsonl 2>&1
cat gpurun_out/r02_shrink_cost_carry.jsonl
for i in 1 2; do
timeout 300 python bench.py --no-cpu-baseline > gpurun_out/r02_carry2_bench_$i.json 2>/dev/null; tail -1 gpurun_out/r02_carry2_bench_$i.json | cut -c1-300
MUX_CARRY=0 timeout 300 python bench.py --no-cpu-baseline > gpurun_out/r02_nocarry2_bench_$i.json 2>/dev/null; tail -1 gpurun_out/r02_nocarry2_bench_$i.json | cut -c1-300
done
fi
