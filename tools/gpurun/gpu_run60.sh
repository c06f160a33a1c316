# Narrow (256 x 128) vs standard (256 x 256) pair tiles on tensor-parallel shard shapes with narrow outputs
# (o-proj dX at TP-8: 512 output columns = 2 standard tiles per row block, 168 tiles on 74 pairs)
timeout 1200 python tools/raster_ab.py --var MUX_TILE_N --modes 256,128 --rounds 11 --rows 21504 --tasks 16 --rank 16 --shapes 512x4096,4096x512,4096x1024,1024x4096,4096x1536,1376x4096 --out gpurun_out/r02_narrow_ab_tp.jsonl > /dev/null 2> gpurun_out/narrow_ab.err
cat gpurun_out/r02_narrow_ab_tp.jsonl
