set -x
timeout 900 python -m pytest -q tests/test_gpu_wide.py tests/test_gpu_linear.py > gpurun_out/r02s2_t14.log 2>&1
tail -3 gpurun_out/r02s2_t14.log
timeout 900 python tools/raster_ab.py --var MUX_TILE_N --modes 256,512 --rounds 11 --out gpurun_out/r02_tile_ab_cfg2.jsonl > /dev/null 2> gpurun_out/tile_ab.err
timeout 900 python tools/raster_ab.py --var MUX_TILE_N --modes 256,512 --rounds 11 --rows 21504 --tasks 16 --rank 32 --shapes 512x4096,1376x4096,4096x1536,4096x2752,1536x4096 --out gpurun_out/r02_tile_ab_tp.jsonl > /dev/null 2>> gpurun_out/tile_ab.err
