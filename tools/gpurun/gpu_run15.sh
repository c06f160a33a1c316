set -x
timeout 900 python tools/tp_shard_profile.py --points 4:8,5:8,4:4,4:2,4:1 --fused --shared-shrink > gpurun_out/r02_tp_shard_fused_v3.jsonl 2>gpurun_out/tp_shard.err
timeout 900 python tools/tp_shard_profile.py --points 4:8,5:8 > gpurun_out/r02_tp_shard_sep_v3.jsonl 2>>gpurun_out/tp_shard.err
timeout 600 python bench.py --mode block --config 4 --steps 20 --warmup 5 > gpurun_out/r02_bench_block4_v3.json 2>gpurun_out/b.err
timeout 600 python bench.py --mode tp --config 4 --steps 20 --warmup 5 --no-cpu-baseline > gpurun_out/r02_bench_tp4_v3.json 2>>gpurun_out/b.err
