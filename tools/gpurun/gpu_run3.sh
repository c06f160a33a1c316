set -x
timeout 900 python -m pytest -q tests/test_gpu_raster.py tests/test_gpu_tp_block.py tests/test_gpu_sliced.py "tests/test_gpu_streamk.py::test_linear_and_rs_suites_under_forced_streamk" > gpurun_out/r02s2_t3.log 2>&1
tail -3 gpurun_out/r02s2_t3.log
timeout 600 python tools/raster_ab.py --out gpurun_out/r02_raster_ab.jsonl > /dev/null 2>gpurun_out/raster_ab.err
timeout 600 ncu --metrics dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum,lts__t_sector_hit_rate.pct -k regex:mux_gemm --csv python tools/raster_ab.py --once > gpurun_out/r02_raster_ncu.csv 2>gpurun_out/raster_ncu.err
for f in "" "--fused" "--fused --shared-shrink" "--shared-shrink"; do timeout 600 python tools/tp_shard_profile.py --points 4:8,5:8,4:1 $f >> gpurun_out/r02_tp_shard_fused.jsonl 2>>gpurun_out/tp_shard.err; done
for fp in 1 0; do timeout 600 python bench.py --mode tp --config 4 --fused-proj $fp --steps 10 --warmup 3 --no-cpu-baseline > gpurun_out/r02_bench_tp4_fp$fp.json 2>gpurun_out/bench_tp4_fp$fp.err; done
ls -la gpurun_out
