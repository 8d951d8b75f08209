#!/bin/bash
mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_ngram.py -q -x -k lossless 2>&1 | tail -3 > gpurun_out/r2_t18.log
timeout 600 python -m pytest tests/test_gpu_attention.py -q -x 2>&1 | tail -2 >> gpurun_out/r2_t18.log
TLT_ATTN_TMA_TREE=1 timeout 600 python -m pytest tests/test_gpu_attention.py -q -x 2>&1 | tail -2 >> gpurun_out/r2_t18.log
python tools/probe_attn.py 1:1024:65 5:700:49 16:700:17 31:700:17 31:2000:17 8:1024:33 > gpurun_out/r2_probe_tree_v0.txt 2>&1
TLT_ATTN_TMA_TREE=1 python tools/probe_attn.py 1:1024:65 5:700:49 16:700:17 31:700:17 31:2000:17 8:1024:33 > gpurun_out/r2_probe_tree_v1.txt 2>&1
for mc in 64 128 256; do for fc in -1 1; do echo "min_chunk=$mc fused=$fc"; TLT_ATTN_DEC_MIN_CHUNK=$mc TLT_ATTN_FUSED_COMBINE=$fc python tools/probe_attn.py 1:1024:1 4:1024:1 8:2048:1 32:1024:1 64:1024:1 64:2048:1; done; done > gpurun_out/r2_probe_dec_sweep.txt 2>&1
