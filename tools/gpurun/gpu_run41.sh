# default-length bench (config 2, 1 GPU): raster m (default) vs a (traffic model), interleaved
for i in 1 2 3 4; do
for r in m a; do
MUX_RASTER=$r timeout 600 python bench.py --no-cpu-baseline 2>/dev/null | tail -1 | python -c "
import json,sys; d=json.loads(sys.stdin.read()); print(json.dumps({'raster':'$r','value':d['value'],'e2e':d['e2e']['value'],'ms':d['ms_per_step'],'sm_mhz':d['clocks']['sm_mhz'],'sm_min':d['clocks'].get('sm_mhz_min'),'pw':d['clocks'].get('power_w_max'),'reasons':d['clocks']['reasons'],'fwd_ms':d['kernels']['fwd_calls_ms_per_step'],'bwd_ms':d['kernels']['bwd_calls_ms_per_step']}))" >> gpurun_out/r02_raster_default.jsonl
done
done
cat gpurun_out/r02_raster_default.jsonl
