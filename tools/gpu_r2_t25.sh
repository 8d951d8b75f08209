#!/bin/bash
mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_gpu_attention.py -q -x 2>&1 | tail -3 > gpurun_out/r2_t25.log
for tc in 1 0; do
  TLT_ATTN_TREE_TC=$tc timeout 900 python bench.py --steps 1 --warmup 1 --cpu-rows 0 --ar-baseline 0 --len-median 400 --max-len 2048 > gpurun_out/r2_ab_treetc$tc.json 2> gpurun_out/r2_ab_treetc$tc.err
done
