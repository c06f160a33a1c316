for fp in 1 0; do
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/r02_block_launches_fp$fp.csv python bench.py --mode block --config 4 --fused-proj $fp --steps 2 --warmup 1 > /dev/null 2>&1
done
ls -la gpurun_out/r02_block_launches_fp*.csv
