#!/bin/bash
mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_gpu_attention.py -q -x -k tcgen05 2>&1 | tail -3 > gpurun_out/r2_t26.log
TLT_ATTN_TREE_TC=1 python tools/probe_attn.py 1:1024:65 5:700:49 16:700:17 31:700:17 31:2000:17 8:1024:33 > gpurun_out/r2_probe_tree_tc2.txt 2>&1
TLT_ATTN_TREE_TC=0 python tools/probe_attn.py 1:1024:65 5:700:49 16:700:17 31:700:17 31:2000:17 8:1024:33 > gpurun_out/r2_probe_tree_tma2.txt 2>&1
for tc in 1 0; do
  TLT_ATTN_TREE_TC=$tc timeout 900 python bench.py --steps 1 --warmup 1 --cpu-rows 0 --ar-baseline 0 --len-median 400 --max-len 2048 > gpurun_out/r2_ab2_treetc$tc.json 2> gpurun_out/r2_ab2_treetc$tc.err
done
