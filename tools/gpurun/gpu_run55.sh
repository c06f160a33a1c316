# Diagnostic: what the producer's reader-side proxy fence (after the shrink-flag acquire) costs:
# current build vs the same without that fence (libmux_nofence.so, timing only) vs no flag wait at all
timeout 900 python tools/gemm_ab.py --libs paper_2603_02885_b200/libmux.so paper_2603_02885_b200/libmux_nofence.so paper_2603_02885_b200/libmux_noflag.so --no-cublas > gpurun_out/r02_fence_ab_cfg2.jsonl 2>&1
cat gpurun_out/r02_fence_ab_cfg2.jsonl
