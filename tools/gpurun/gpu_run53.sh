# Final round-2 evidence on the final build: full GPU suite, smoke, ncu launch list of the bench step,
# ncu --set full of the timed step's three forward GEMM launches -> profiles/gemm_fwd_traffic.json,
# then the bench line (which now reports that traffic) and the reference (oracle) arm
timeout 1800 python -m pytest tests -m gpu -q > gpurun_out/r02_gpu_tests_final.log 2>&1; echo "pytest rc=$?" >> gpurun_out/r02_gpu_tests_final.log
tail -3 gpurun_out/r02_gpu_tests_final.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke(); print('smoke ok')" > gpurun_out/r02_smoke_final.log 2>&1; tail -1 gpurun_out/r02_smoke_final.log
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/r02_launches_final.csv python bench.py --steps 2 --warmup 1 --no-e2e --no-cpu-baseline > /dev/null 2>&1
timeout 1200 ncu --set full --clock-control none --import-source on -k regex:mux_gemm_kernel --launch-skip 6 --launch-count 3 -o gpurun_out/r02_prof_gemm_final python bench.py --steps 1 --warmup 1 --no-e2e --no-cpu-baseline > gpurun_out/r02_ncu_full_final.log 2>&1
python tools/traffic_json.py gpurun_out/r02_prof_gemm_final.ncu-rep > gpurun_out/r02_traffic_final.log 2>&1; cp profiles/gemm_fwd_traffic.json gpurun_out/gemm_fwd_traffic.json
timeout 600 python bench.py > gpurun_out/r02_bench_final.json 2> gpurun_out/r02_bench_final.err; tail -1 gpurun_out/r02_bench_final.json | cut -c1-300
timeout 900 python tools/tp_shard_profile.py --points 4:8,5:8 --fused --shared-shrink > gpurun_out/r02_tp_shard_final.jsonl 2>gpurun_out/tp_shard_final.err; cut -c1-200 gpurun_out/r02_tp_shard_final.jsonl
timeout 900 python bench.py --impl reference --steps 2 --warmup 1 > gpurun_out/r02_bench_reference.json 2> gpurun_out/r02_bench_reference.err; tail -1 gpurun_out/r02_bench_reference.json | cut -c1-300
