# sustained bench (config 2, 1 GPU) with the row-band raster (m, default) vs the traffic-model raster (a):
# does less DRAM traffic buy clock under the power cap?
for i in 1 2 3; do
for r in m a; do
MUX_RASTER=$r timeout 600 python bench.py --steps 300 --warmup 10 --no-cpu-baseline --no-e2e 2>/dev/null | tail -1 | python -c "
import json,sys; d=json.loads(sys.stdin.read()); print(json.dumps({'raster':'$r','value':d['value'],'ms':d['ms_per_step'],'sm_mhz':d['clocks']['sm_mhz'],'sm_min':d['clocks'].get('sm_mhz_min'),'pw':d['clocks'].get('power_w_max'),'reasons':d['clocks']['reasons'],'fwd_ms':d['kernels']['fwd_calls_ms_per_step'],'bwd_ms':d['kernels']['bwd_calls_ms_per_step']}))" >> gpurun_out/r02_raster_sustained.jsonl
done
done
cat gpurun_out/r02_raster_sustained.jsonl
nvidia-smi -q -d POWER | grep -i -A3 "limit" | head -20
