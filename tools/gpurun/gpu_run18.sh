set -x
timeout 600 python -m pytest -q -x tests/test_gpu_wide.py > gpurun_out/r02s2_t18.log 2>&1
tail -3 gpurun_out/r02s2_t18.log
timeout 900 python tools/raster_ab.py --var MUX_TILE_N --modes 256,512 --rounds 11 --out gpurun_out/r02_tile_ab_cfg2_v2.jsonl > /dev/null 2> gpurun_out/tile_ab.err
timeout 900 python tools/raster_ab.py --var MUX_TILE_N --modes 256,512 --rounds 11 --rows 21504 --tasks 16 --rank 32 --shapes 512x4096,1376x4096,4096x1536,4096x2752,1536x4096 --out gpurun_out/r02_tile_ab_tp_v2.jsonl > /dev/null 2>> gpurun_out/tile_ab.err
