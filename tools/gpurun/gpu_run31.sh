timeout 600 python -m pytest -q tests/test_gpu_linear.py -k "given_gs or given_hs" tests/test_gpu_tp_block.py > gpurun_out/r02s2_t31.log 2>&1
tail -3 gpurun_out/r02s2_t31.log
timeout 900 python tools/tp_shard_profile.py --points 4:8,5:8,4:4 --fused --shared-shrink > gpurun_out/r02_tp_shard_fused_v4.jsonl 2>gpurun_out/tp_shard.err
