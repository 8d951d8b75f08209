#!/bin/bash
mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_gpu_attention.py -q -x -k tcgen05 2>&1 | grep -v "^    " | tail -30 > gpurun_out/r2_t21.log
TLT_ATTN_TREE_TC=1 python tools/probe_attn.py 1:1024:65 5:700:49 16:700:17 31:700:17 31:2000:17 8:1024:33 > gpurun_out/r2_probe_tree_tc.txt 2>&1
TLT_ATTN_TREE_TC=0 python tools/probe_attn.py 1:1024:65 5:700:49 16:700:17 31:700:17 31:2000:17 8:1024:33 > gpurun_out/r2_probe_tree_tma.txt 2>&1
timeout 900 python -m pytest tests/test_spot.py -q -x 2>&1 | grep -v "^    " | tail -30 >> gpurun_out/r2_t21.log
