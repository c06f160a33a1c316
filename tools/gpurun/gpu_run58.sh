# Final build (fixed-size flag region): carrier suite incl. the shared-workspace regression, full GPU
# suite, smoke, the §8(d) sweeps / planner profile / alignment sweep, then the final evidence (ncu
# launch list, full capture -> traffic json, bench line, TP shard profile, oracle arm)
timeout 900 python -m pytest tests/test_gpu_carry.py -m gpu -x -q > gpurun_out/r02_carry7_tests.log 2>&1; echo "pytest rc=$?" >> gpurun_out/r02_carry7_tests.log
tail -2 gpurun_out/r02_carry7_tests.log
grep -q "pytest rc=0" gpurun_out/r02_carry7_tests.log || exit 1
timeout 1800 python -m pytest tests -m gpu -q > gpurun_out/r02_gpu_tests_final2.log 2>&1; echo "pytest rc=$?" >> gpurun_out/r02_gpu_tests_final2.log
tail -3 gpurun_out/r02_gpu_tests_final2.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke(); print('smoke ok')" > gpurun_out/r02_smoke_final2.log 2>&1; tail -1 gpurun_out/r02_smoke_final2.log
timeout 900 python tools/sweep.py --out gpurun_out/r02_sweep_final.jsonl > gpurun_out/sweep.log 2>&1
timeout 900 python tools/op_profile.py --out gpurun_out/r02_op_profile_final.json > gpurun_out/op_profile.log 2>&1; tail -2 gpurun_out/op_profile.log
timeout 900 python tools/alignment_sweep.py --out gpurun_out/r02_alignment_sweep_final.jsonl > gpurun_out/align.log 2>&1
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/r02_launches_final2.csv python bench.py --steps 2 --warmup 1 --no-e2e --no-cpu-baseline > /dev/null 2>&1
timeout 1200 ncu --set full --clock-control none --import-source on -k regex:mux_gemm_kernel --launch-skip 6 --launch-count 3 -o gpurun_out/r02_prof_gemm_final2 python bench.py --steps 1 --warmup 1 --no-e2e --no-cpu-baseline > gpurun_out/r02_ncu_full_final2.log 2>&1
python tools/traffic_json.py gpurun_out/r02_prof_gemm_final2.ncu-rep > gpurun_out/r02_traffic_final2.log 2>&1; cp profiles/gemm_fwd_traffic.json gpurun_out/gemm_fwd_traffic.json
timeout 600 python bench.py > gpurun_out/r02_bench_final2.json 2> gpurun_out/r02_bench_final2.err; tail -1 gpurun_out/r02_bench_final2.json | cut -c1-300
timeout 900 python tools/tp_shard_profile.py --points 4:8,5:8 --fused --shared-shrink > gpurun_out/r02_tp_shard_final2.jsonl 2>gpurun_out/tp_shard_final.err
timeout 900 python bench.py --impl reference --steps 2 --warmup 1 > gpurun_out/r02_bench_reference2.json 2> gpurun_out/r02_bench_reference.err
