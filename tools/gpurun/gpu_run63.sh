# Block step (config 4, ~1 s timed, at the power cap): row bands (m, default) vs the DRAM-traffic-model raster (a)
for i in 1 2 3; do
for r in m a; do
MUX_RASTER=$r timeout 600 python bench.py --mode block --config 4 --no-cpu-baseline --no-e2e 2>/dev/null | tail -1 | python -c "
import json,sys; d=json.loads(sys.stdin.read()); print(json.dumps({'raster':'$r','value':d['value'],'ms':d['ms_per_step'],'sm_mhz':d['clocks']['sm_mhz'],'pw':d['clocks'].get('power_w_max'),'reasons':d['clocks']['reasons']}))" >> gpurun_out/r02_block_raster_ab.jsonl
done
done
cat gpurun_out/r02_block_raster_ab.jsonl
