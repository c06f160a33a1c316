# Multi-wave carriers (MUX_CARRY=3) on the config-4 decoder block (22 592 rows = 89 row blocks > 74 pairs)
timeout 300 python -c "import __graft_entry__ as g; g.smoke(); print('smoke ok')" > gpurun_out/r02_smoke_v5.log 2>&1; tail -1 gpurun_out/r02_smoke_v5.log
timeout 900 python -m pytest tests/test_gpu_carry.py -m gpu -x -q > gpurun_out/r02_carry5_tests.log 2>&1; echo "pytest rc=$?" >> gpurun_out/r02_carry5_tests.log
tail -2 gpurun_out/r02_carry5_tests.log
if grep -q "pytest rc=0" gpurun_out/r02_carry5_tests.log; then
timeout 900 python tools/gemm_ab.py --env-ab MUX_CARRY=3,1 --no-cublas --rows 22592 --tasks 16 --shapes 4096x4096,4096x11008,11008x4096 > gpurun_out/r02_carry5_envab_rows22k.jsonl 2>&1
cat gpurun_out/r02_carry5_envab_rows22k.jsonl
for i in 1 2 3; do
for c in 3 1; do
MUX_CARRY=$c timeout 600 python bench.py --mode block --config 4 --no-cpu-baseline --no-e2e > gpurun_out/r02_block_carry${c}_$i.json 2>/dev/null; tail -1 gpurun_out/r02_block_carry${c}_$i.json | python -c "
import json,sys; d=json.loads(sys.stdin.read()); print(json.dumps({'carry':'$c','value':d['value'],'ms':d['ms_per_step'],'sm_mhz':d['clocks']['sm_mhz'],'reasons':d['clocks']['reasons']}))" >> gpurun_out/r02_block_carry_ab.jsonl
done
done
cat gpurun_out/r02_block_carry_ab.jsonl
fi
