#!/bin/bash
mkdir -p gpurun_out
( python tools/debug_pool.py 11 6,8,32 0 ; echo "exact rc=$?"
  python tools/debug_pool.py 11 6,8,32 1 ; echo "pooled rc=$?"
  TLT_ATTN_TREE_DYN=0 python tools/debug_pool.py 11 6,8,32 1 ; echo "pooled tree-dyn-off rc=$?"
  timeout 600 compute-sanitizer --tool memcheck --print-limit 5 python tools/debug_pool.py 11 6,8,32 1 ) > gpurun_out/r2_t5.log 2>&1
