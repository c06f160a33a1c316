# Sanitizers on the carrier path: memcheck + synccheck over the carrier suite (fwd and bwd carriers, the
# fallbacks) and smoke(); racecheck over smoke() (which runs a carrier launch)
timeout 1200 compute-sanitizer --tool memcheck --print-limit 10 python -m pytest -q tests/test_gpu_carry.py -k "not normal_values and not spanning and not more_row_blocks" > gpurun_out/r02_memcheck_carry.log 2>&1; tail -3 gpurun_out/r02_memcheck_carry.log
timeout 1200 compute-sanitizer --tool synccheck --print-limit 10 python -m pytest -q tests/test_gpu_carry.py -k "not normal_values and not spanning and not more_row_blocks" > gpurun_out/r02_synccheck_carry.log 2>&1; tail -3 gpurun_out/r02_synccheck_carry.log
timeout 900 compute-sanitizer --tool memcheck --print-limit 10 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/r02_memcheck_smoke.log 2>&1; tail -3 gpurun_out/r02_memcheck_smoke.log
timeout 900 compute-sanitizer --tool racecheck --print-limit 10 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/r02_racecheck_smoke_v3.log 2>&1; tail -5 gpurun_out/r02_racecheck_smoke_v3.log
