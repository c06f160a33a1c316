# one-launch multi-slice adapter gradients: parity + per-part times of the fused TP shard calls
timeout 1200 python -m pytest -q -x tests/test_gpu_sliced.py tests/test_gpu_linear.py tests/test_gpu_wide.py tests/test_gpu_grad_simt.py tests/test_gpu_fullsize.py > gpurun_out/r02_t37.log 2>&1
tail -5 gpurun_out/r02_t37.log
timeout 900 python tools/tp_shard_profile.py --points 4:8,5:8,4:4 --fused --shared-shrink --parts > gpurun_out/r02_tp_shard_parts_v2.jsonl 2>gpurun_out/tp_shard.err
cat gpurun_out/r02_tp_shard_parts_v2.jsonl; tail -3 gpurun_out/tp_shard.err
