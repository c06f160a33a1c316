# Warp-3 shrink-flag poller (flag hand-over through an mbarrier): parity, A/B vs the previous build and
# the no-flag diagnostic, wait profile
timeout 1200 python -m pytest tests/test_gpu_carry.py tests/test_gpu_linear.py tests/test_gpu_streamk.py tests/test_gpu_rs.py tests/test_gpu_graph.py tests/test_gpu_tp.py tests/test_gpu_sliced.py -m gpu -x -q > gpurun_out/r02_fok_tests.log 2>&1; echo "pytest rc=$?" >> gpurun_out/r02_fok_tests.log
tail -2 gpurun_out/r02_fok_tests.log
if grep -q "pytest rc=0" gpurun_out/r02_fok_tests.log; then
timeout 900 python tools/gemm_ab.py --libs paper_2603_02885_b200/libmux_c4.so paper_2603_02885_b200/libmux.so paper_2603_02885_b200/libmux_noflag.so --no-cublas > gpurun_out/r02_fok_ab_cfg2.jsonl 2>&1
timeout 900 python tools/gemm_ab.py --libs paper_2603_02885_b200/libmux_c4.so paper_2603_02885_b200/libmux.so --no-cublas --rows 21504 --tasks 16 --shapes 4096x512,512x4096,1376x4096,4096x2752 > gpurun_out/r02_fok_ab_tp.jsonl 2>&1
cat gpurun_out/r02_fok_ab_cfg2.jsonl gpurun_out/r02_fok_ab_tp.jsonl
timeout 300 python tools/gemm_waits.py 16 > gpurun_out/r02_waits_fok.jsonl 2>&1
fi
