# Final-build bench lines of the other arms: the config-4 decoder block (NEXT-3) and the TP arm at world 1
timeout 900 python bench.py --mode block --config 4 > gpurun_out/r02_bench_block_final.json 2> gpurun_out/block_final.err; tail -1 gpurun_out/r02_bench_block_final.json | cut -c1-250
timeout 900 python bench.py --mode tp --config 4 > gpurun_out/r02_bench_tp4_world1_final.json 2> gpurun_out/tp4_final.err; tail -1 gpurun_out/r02_bench_tp4_world1_final.json | cut -c1-250
timeout 900 python bench.py --mode tp --config 2 > gpurun_out/r02_bench_tp2_world1_final.json 2> gpurun_out/tp2_final.err; tail -1 gpurun_out/r02_bench_tp2_world1_final.json | cut -c1-250
