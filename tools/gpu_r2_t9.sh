#!/bin/bash
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_attention.py -q -x 2>&1 | tail -25 > gpurun_out/r2_t9.log
python tools/probe_attn.py 1:1024:1 8:1024:1 32:1024:1 64:1024:1 1:1024:65 5:700:49 16:700:17 31:700:17 > gpurun_out/r2_probe_attn_tma.txt 2>&1
TLT_ATTN_TMA=0 python tools/probe_attn.py 1:1024:1 8:1024:1 32:1024:1 64:1024:1 1:1024:65 5:700:49 16:700:17 31:700:17 > gpurun_out/r2_probe_attn_notma.txt 2>&1
timeout 900 python -m pytest tests -q -m gpu -x 2>&1 | tail -5 >> gpurun_out/r2_t9.log
