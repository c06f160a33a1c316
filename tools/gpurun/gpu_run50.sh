# Round-2 evidence on the carrier build: full GPU suite, smoke, default bench, ncu launch list of the
# bench step, ncu --set full of the timed step's three forward GEMM launches (traffic, tensor pipe)
timeout 1800 python -m pytest tests -m gpu -q > gpurun_out/r02_gpu_tests_v4.log 2>&1; echo "pytest rc=$?" >> gpurun_out/r02_gpu_tests_v4.log
tail -3 gpurun_out/r02_gpu_tests_v4.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke(); print('smoke ok')" > gpurun_out/r02_smoke_v4.log 2>&1; tail -1 gpurun_out/r02_smoke_v4.log
timeout 600 python bench.py > gpurun_out/r02_bench_main_v5.json 2> gpurun_out/r02_bench_main_v5.err; tail -1 gpurun_out/r02_bench_main_v5.json | cut -c1-300
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/r02_launches_v2.csv python bench.py --steps 2 --warmup 1 --no-e2e --no-cpu-baseline > /dev/null 2>&1
timeout 1200 ncu --set full --clock-control none --import-source on -k regex:mux_gemm_kernel --launch-skip 6 --launch-count 3 -o gpurun_out/r02_prof_gemm_v2 python bench.py --steps 1 --warmup 1 --no-e2e --no-cpu-baseline > gpurun_out/r02_ncu_full_v2.log 2>&1
ls -la gpurun_out | tail -5
