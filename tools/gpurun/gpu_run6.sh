set -x
timeout 300 compute-sanitizer --tool racecheck tools/probe/racecheck_probe > gpurun_out/r02_racecheck_probe.log 2>&1
for fp in 1 0 1 0; do
  timeout 600 python bench.py --mode tp --config 4 --fused-proj $fp --steps 20 --warmup 5 --no-cpu-baseline >> gpurun_out/r02_bench_tp4_ab.jsonl 2>>gpurun_out/bench_ab.err
  timeout 600 python bench.py --mode block --config 4 --fused-proj $fp --steps 20 --warmup 5 >> gpurun_out/r02_bench_block4_ab.jsonl 2>>gpurun_out/bench_ab.err
done
timeout 600 python bench.py --mode tp --config 5 --steps 10 --warmup 3 --no-cpu-baseline >> gpurun_out/r02_bench_tp5.jsonl 2>>gpurun_out/bench_ab.err
timeout 900 python tools/tp_shard_profile.py --points 4:8,5:8 --fused --shared-shrink >> gpurun_out/r02_tp_shard_fused_v2.jsonl 2>>gpurun_out/tp_shard.err
