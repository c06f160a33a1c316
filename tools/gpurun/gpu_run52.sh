# W as 128-row TMA boxes (fewer producer TMA issues): parity on every tile width, then interleaved A/B
timeout 1200 python -m pytest tests/test_gpu_wide.py tests/test_gpu_linear.py tests/test_gpu_carry.py tests/test_gpu_streamk.py tests/test_gpu_sliced.py tests/test_gpu_fullsize.py -m gpu -x -q > gpurun_out/r02_wbox_tests.log 2>&1; echo "pytest rc=$?" >> gpurun_out/r02_wbox_tests.log
tail -2 gpurun_out/r02_wbox_tests.log
if grep -q "pytest rc=0" gpurun_out/r02_wbox_tests.log; then
timeout 900 python tools/gemm_ab.py --libs paper_2603_02885_b200/libmux_wbox64.so paper_2603_02885_b200/libmux.so --no-cublas > gpurun_out/r02_wbox_ab_cfg2.jsonl 2>&1
timeout 900 python tools/gemm_ab.py --libs paper_2603_02885_b200/libmux_wbox64.so paper_2603_02885_b200/libmux.so --no-cublas --rows 21504 --tasks 16 --shapes 4096x512,512x4096,1376x4096,4096x1536 > gpurun_out/r02_wbox_ab_tp.jsonl 2>&1
cat gpurun_out/r02_wbox_ab_cfg2.jsonl gpurun_out/r02_wbox_ab_tp.jsonl
fi
