MUX_LIB_FILE=libmux_direct.so timeout 600 python -m pytest -q tests/test_gpu_linear.py tests/test_gpu_sliced.py -k "not rs and not debug" > gpurun_out/r02s2_t26.log 2>&1
tail -2 gpurun_out/r02s2_t26.log
timeout 900 python tools/gemm_ab.py --libs paper_2603_02885_b200/libmux.so paper_2603_02885_b200/libmux_direct.so --rounds 11 --no-cublas > gpurun_out/r02_gemm_ab_direct_cfg2.jsonl 2>gpurun_out/ab.err
timeout 900 python tools/gemm_ab.py --libs paper_2603_02885_b200/libmux.so paper_2603_02885_b200/libmux_direct.so --rows 21504 --tasks 16 --rank 32 --shapes 512x4096,1376x4096,4096x1536,4096x2752,1536x4096,4096x512 --no-cublas --rounds 11 > gpurun_out/r02_gemm_ab_direct_tp.jsonl 2>>gpurun_out/ab.err
