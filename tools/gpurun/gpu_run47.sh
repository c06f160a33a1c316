# Carrier shrink with counter flags (red.release.add, last-CTA reset): parity, wait profile, A/B
timeout 900 python -m pytest tests/test_gpu_carry.py tests/test_gpu_linear.py tests/test_gpu_streamk.py tests/test_gpu_rs.py tests/test_gpu_graph.py -m gpu -x -q > gpurun_out/r02_carry3_tests.log 2>&1; echo "pytest rc=$?" >> gpurun_out/r02_carry3_tests.log
tail -3 gpurun_out/r02_carry3_tests.log
if grep -q "pytest rc=0" gpurun_out/r02_carry3_tests.log; then
for c in 1 0; do MUX_CARRY=$c timeout 300 python tools/gemm_waits.py 16 > gpurun_out/r02_waits_carry$c.jsonl 2>&1; done
cat gpurun_out/r02_waits_carry1.jsonl gpurun_out/r02_waits_carry0.jsonl
timeout 900 python tools/gemm_ab.py --libs paper_2603_02885_b200/libmux_old.so paper_2603_02885_b200/libmux.so paper_2603_02885_b200/libmux_noflag.so > gpurun_out/r02_carry3_ab_cfg2.jsonl 2>&1
cat gpurun_out/r02_carry3_ab_cfg2.jsonl
timeout 600 python tools/shrink_cost.py --label config2-carry-redflags > gpurun_out/r02_shrink_cost_carry3.jsonl 2>&1
cat gpurun_out/r02_shrink_cost_carry3.jsonl
fi
