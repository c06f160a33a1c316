set -x
timeout 900 python -m pytest -q tests/test_gpu_tp_block.py tests/test_gpu_decoder_block.py > gpurun_out/r02s2_t4.log 2>&1
tail -3 gpurun_out/r02s2_t4.log
timeout 900 python tools/fused_ab.py --sets qkv1,gu1,qkv2,gu2,qkv4,gu4,qkv8,gu8,qkv70b8,gu70b8 --out gpurun_out/r02_fused_ab.jsonl > /dev/null 2> gpurun_out/fused_ab.err
for fp in 1 0; do
  timeout 600 python bench.py --mode tp --config 4 --fused-proj $fp --steps 10 --warmup 3 --no-cpu-baseline > gpurun_out/r02_bench_tp4_fp$fp.json 2>gpurun_out/bench_tp4_fp$fp.err
  timeout 600 python bench.py --mode block --config 4 --fused-proj $fp --steps 10 --warmup 3 > gpurun_out/r02_bench_block4_fp$fp.json 2>gpurun_out/bench_block4_fp$fp.err
done
timeout 300 compute-sanitizer --tool racecheck tools/probe/racecheck_probe > gpurun_out/r02_racecheck_probe.log 2>&1
timeout 600 compute-sanitizer --tool racecheck --print-limit 10 python __graft_entry__.py smoke > gpurun_out/r02_racecheck_smoke.log 2>&1
timeout 900 compute-sanitizer --tool memcheck --print-limit 10 python -m pytest -q tests/test_gpu_sliced.py -k "not full_size" > gpurun_out/r02_memcheck_sliced.log 2>&1
tail -2 gpurun_out/r02_racecheck_probe.log gpurun_out/r02_racecheck_smoke.log gpurun_out/r02_memcheck_sliced.log
