set -x
timeout 900 python -m pytest -q tests/test_gpu_linear.py tests/test_gpu_sliced.py tests/test_gpu_streamk.py tests/test_gpu_raster.py -k "not forced_streamk" > gpurun_out/r02s2_t12.log 2>&1
tail -2 gpurun_out/r02s2_t12.log
MUX_ROWS=21504 MUX_TASKS=16 MUX_MIXED=1 timeout 600 python tools/gemm_waits.py 32 512x4096,4096x512,4096x1536,1536x4096,4096x4096 > gpurun_out/r02_gemm_waits_tp_v5.jsonl 2> gpurun_out/waits.err
timeout 900 python tools/gemm_ab.py --libs paper_2603_02885_b200/libmux.so paper_2603_02885_b200/libmux_old.so --rows 21504 --tasks 16 --rank 32 --shapes 512x4096,4096x512,1376x4096,4096x1376,4096x1536,1536x4096 --rounds 11 > gpurun_out/r02_gemm_ab_flagcount2_tp.jsonl 2>gpurun_out/ab.err
timeout 900 python tools/gemm_ab.py --libs paper_2603_02885_b200/libmux.so paper_2603_02885_b200/libmux_old.so --rounds 11 > gpurun_out/r02_gemm_ab_flagcount2_cfg2.jsonl 2>>gpurun_out/ab.err
