# Round-2 re-entry check: full GPU suite, smoke, default bench (config 2), launch list
timeout 1500 python -m pytest tests -m gpu -x -q > gpurun_out/r02_gpu_tests_v3.log 2>&1; echo "pytest rc=$?" >> gpurun_out/r02_gpu_tests_v3.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke(); print('smoke ok')" > gpurun_out/r02_smoke_v3.log 2>&1
timeout 600 python bench.py > gpurun_out/r02_bench_main_v4.json 2> gpurun_out/r02_bench_main_v4.err
tail -1 gpurun_out/r02_bench_main_v4.json
