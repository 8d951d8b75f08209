#!/bin/bash
mkdir -p gpurun_out
for c in 296 444 592 888 1184; do
  TLT_ATTN_DEC_CTAS=$c timeout 300 python tools/probe_attn_ctas.py 2>&1 | grep ctas
done | tee gpurun_out/attn_ctas.txt
