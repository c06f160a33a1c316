set -x
timeout 900 python tools/fused_ab.py --sets qkv1,gu1,qkv2,gu2,qkv4,gu4,qkv8,gu8,qkv70b8,gu70b8,o8,down8 --out gpurun_out/r02_fused_ab_v2.jsonl > /dev/null 2> gpurun_out/fused_ab.err
timeout 900 python tools/tp_shard_profile.py --points 4:2,4:4 >> gpurun_out/r02_tp_shard_fused_24.jsonl 2>>gpurun_out/tp_shard.err
timeout 900 python tools/tp_shard_profile.py --points 4:2,4:4 --fused >> gpurun_out/r02_tp_shard_fused_24.jsonl 2>>gpurun_out/tp_shard.err
timeout 600 compute-sanitizer --tool racecheck --print-limit 10 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/r02_racecheck_smoke.log 2>&1
timeout 600 compute-sanitizer --tool synccheck --print-limit 10 python -m pytest -q tests/test_gpu_sliced.py -k "not full_size" > gpurun_out/r02_synccheck_sliced.log 2>&1
