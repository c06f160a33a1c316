set -x
timeout 300 compute-sanitizer --tool racecheck tools/probe/racecheck_probe > gpurun_out/r02_racecheck_probe.log 2>&1
timeout 900 python tools/gemm_ab.py --libs paper_2603_02885_b200/libmux.so paper_2603_02885_b200/libmux_noprefetch.so --rows 21504 --tasks 16 --rank 32 --shapes 512x4096,4096x512,1376x4096,4096x1376,4096x1536 --no-cublas --rounds 11 > gpurun_out/r02_gemm_ab_flagprefetch_tp.jsonl 2>gpurun_out/ab.err
timeout 900 python tools/gemm_ab.py --libs paper_2603_02885_b200/libmux.so paper_2603_02885_b200/libmux_noprefetch.so --no-cublas --rounds 11 > gpurun_out/r02_gemm_ab_flagprefetch_cfg2.jsonl 2>>gpurun_out/ab.err
timeout 1800 python -m pytest tests -m gpu -q > gpurun_out/r02s2_gpu_full.log 2>&1
tail -3 gpurun_out/r02s2_gpu_full.log
