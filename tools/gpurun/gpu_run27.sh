for c in 3a 3b 3c; do timeout 600 python bench.py --config $c --steps 20 --warmup 5 --no-cpu-baseline >> gpurun_out/r02_bench_config3.jsonl 2>>gpurun_out/c3.err; done
timeout 900 python bench.py --mode tp --config 5 --steps 10 --warmup 3 --no-cpu-baseline > gpurun_out/r02_bench_tp5_v2.json 2>>gpurun_out/c3.err
