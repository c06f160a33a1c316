set -x
MUX_ROWS=21504 MUX_TASKS=16 MUX_MIXED=1 timeout 600 python tools/gemm_waits.py 32 512x4096,4096x512,4096x1536,1536x4096,4096x4096,1376x4096 > gpurun_out/r02_gemm_waits_tp.jsonl 2> gpurun_out/waits.err
MUX_ROWS=11648 MUX_TASKS=4 timeout 600 python tools/gemm_waits.py 16 4096x4096,4096x11008,11008x4096 > gpurun_out/r02_gemm_waits_cfg2.jsonl 2>> gpurun_out/waits.err
