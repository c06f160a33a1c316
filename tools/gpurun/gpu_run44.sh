# Re-entry check, part 2: the GPU tests after test_gpu_streamk (the first run stopped there), the
# shrink's cost inside the fused GEMM (D2 upper bound), and an ncu capture of the attention kernels
timeout 1200 python -m pytest tests/test_gpu_streamk.py tests/test_gpu_tp.py tests/test_gpu_tp_2proc.py tests/test_gpu_tp_block.py tests/test_gpu_wide.py -m gpu -x -q > gpurun_out/r02_gpu_tests_v3b.log 2>&1; echo "pytest rc=$?" >> gpurun_out/r02_gpu_tests_v3b.log
timeout 600 python tools/shrink_cost.py --label config2 > gpurun_out/r02_shrink_cost.jsonl 2>&1
timeout 600 python tools/shrink_cost.py --label tp8 --rows 21504 --tasks 16 --shapes 4096x512,4096x1536,512x4096,1376x4096 >> gpurun_out/r02_shrink_cost.jsonl 2>&1
cat gpurun_out/r02_shrink_cost.jsonl
timeout 600 ncu --set full --import-source on -k regex:mux_attn -c 5 -o gpurun_out/r02_attn_full -f python tools/attn_ab.py --rounds 1 --iters 1 > gpurun_out/r02_attn_ncu.log 2>&1
ls -la gpurun_out
