set -x
python bench.py > gpurun_out/r02_bench_main_v2.json 2> gpurun_out/bench_main.err
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/r02_launches.csv python bench.py --steps 2 --warmup 1 --no-e2e --no-cpu-baseline > /dev/null 2>&1
timeout 1200 ncu --set full --clock-control none --import-source on -k regex:mux_gemm_kernel --launch-skip 6 --launch-count 6 -o gpurun_out/r02_prof_gemm python bench.py --steps 1 --warmup 1 --no-e2e --no-cpu-baseline > gpurun_out/ncu_full.log 2>&1
timeout 300 ncu --metrics launch__grid_size,launch__block_size,launch__cluster_dim_x,launch__cluster_dim_y,launch__shared_mem_per_block_dynamic,launch__registers_per_thread,gpu__time_duration.sum --csv python -c "
import torch
a=torch.randn(11648,4096,device='cuda').bfloat16(); b=torch.randn(4096,4096,device='cuda').bfloat16(); c=torch.randn(11648,11008,device='cuda').bfloat16(); w2=torch.randn(11008,4096,device='cuda').bfloat16()
for _ in range(2):
    a@b.t(); c@w2; torch.cuda.synchronize()
" > gpurun_out/r02_cublas_kernels.csv 2>&1
