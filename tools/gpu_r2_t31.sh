#!/bin/bash
mkdir -p gpurun_out
for c in 4 8 16 32 64 296; do for mc in 64 256; do echo "== DEC_CTAS=$c MIN_CHUNK=$mc"; TLT_ATTN_DEC_CTAS=$c TLT_ATTN_DEC_MIN_CHUNK=$mc python tools/probe_attn.py 1:256:1 1:1024:1 1:2048:1 2:1024:1 4:1024:1; done; done > gpurun_out/r2_dec_b1_sweep.txt 2>&1
