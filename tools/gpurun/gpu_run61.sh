# Carriers vs side tiles under a sustained load (300-step bench, ~1.2 s timed), interleaved pairs
for i in 1 2; do
for c in 1 0; do
MUX_CARRY=$c timeout 600 python bench.py --steps 300 --warmup 10 --no-cpu-baseline --no-e2e 2>/dev/null | tail -1 | python -c "
import json,sys; d=json.loads(sys.stdin.read()); print(json.dumps({'carry':'$c','steps':300,'value':d['value'],'ms':d['ms_per_step'],'sm_mhz':d['clocks']['sm_mhz'],'sm_min':d['clocks'].get('sm_mhz_min'),'pw':d['clocks'].get('power_w_max'),'reasons':d['clocks']['reasons'],'frac':d['roofline']['frac'],'peak_kind':d['roofline']['peak_kind']}))" >> gpurun_out/r02_carry_sustained.jsonl
done
done
cat gpurun_out/r02_carry_sustained.jsonl
