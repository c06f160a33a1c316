# Carrier shrink (forward): parity first, then interleaved A/B vs the previous build and the bench
timeout 900 python -m pytest tests/test_gpu_linear.py tests/test_gpu_fullsize.py tests/test_gpu_graph.py tests/test_gpu_sliced.py tests/test_gpu_autograd.py -m gpu -x -q > gpurun_out/r02_carry_tests.log 2>&1; echo "pytest rc=$?" >> gpurun_out/r02_carry_tests.log
tail -3 gpurun_out/r02_carry_tests.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke(); print('smoke ok')" > gpurun_out/r02_carry_smoke.log 2>&1; tail -1 gpurun_out/r02_carry_smoke.log
if grep -q "pytest rc=0" gpurun_out/r02_carry_tests.log; then
timeout 600 python tools/gemm_ab.py --libs paper_2603_02885_b200/libmux_old.so paper_2603_02885_b200/libmux.so --fwd-only > gpurun_out/r02_carry_ab_cfg2.jsonl 2>&1
timeout 600 python tools/gemm_ab.py --libs paper_2603_02885_b200/libmux_old.so paper_2603_02885_b200/libmux.so --fwd-only --rows 21504 --tasks 16 --shapes 4096x512,4096x1536,512x4096,1376x4096,4096x2752 --no-cublas > gpurun_out/r02_carry_ab_tp.jsonl 2>&1
cat gpurun_out/r02_carry_ab_cfg2.jsonl gpurun_out/r02_carry_ab_tp.jsonl
timeout 600 python tools/shrink_cost.py --label config2-carry > gpurun_out/r02_shrink_cost_carry.jsonl 2>&1
for i in 1 2; do
timeout 300 python bench.py --no-cpu-baseline > gpurun_out/r02_carry_bench_$i.json 2>/dev/null; tail -1 gpurun_out/r02_carry_bench_$i.json | cut -c1-400
MUX_CARRY=0 timeout 300 python bench.py --no-cpu-baseline > gpurun_out/r02_nocarry_bench_$i.json 2>/dev/null; tail -1 gpurun_out/r02_nocarry_bench_$i.json | cut -c1-400
done
fi
