python -c "import __graft_entry__ as g; g.build(); g.smoke()" > gpurun_out/r02_final_smoke.log 2>&1
tail -1 gpurun_out/r02_final_smoke.log
timeout 2400 python -m pytest tests -m gpu -q > gpurun_out/r02_final_gputests.log 2>&1
tail -3 gpurun_out/r02_final_gputests.log
python bench.py > gpurun_out/r02_final_bench.json 2> gpurun_out/r02_final_bench.err
tail -c 400 gpurun_out/r02_final_bench.json
