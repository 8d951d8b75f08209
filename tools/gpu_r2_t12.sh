#!/bin/bash
mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_gpu_attention.py -q -x -k "tiny" 2>&1 | grep -v "^    " | tail -30 > gpurun_out/r2_t12.log
TLT_ATTN_TMA=0 python tools/debug_exp.py >> gpurun_out/r2_t12.log 2>&1
