timeout 900 python tools/attn_ab.py --libs paper_2603_02885_b200/libmux.so paper_2603_02885_b200/libmux_dq2.so paper_2603_02885_b200/libmux_dk2.so paper_2603_02885_b200/libmux_dqdk2.so --rounds 9 > gpurun_out/r02_attn_stages_ab.jsonl 2> gpurun_out/attn.err
for l in libmux_dq2.so libmux_dk2.so; do MUX_LIB_FILE=$l timeout 600 python -m pytest -q tests/test_gpu_block.py -k attention >> gpurun_out/r02s2_t29.log 2>&1; done
tail -4 gpurun_out/r02s2_t29.log
