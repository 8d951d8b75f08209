#!/bin/bash
# flash-decode: fused split combine x split floor, per-layer probe times
mkdir -p gpurun_out
for fc in 0 1; do for mc in 64 128 256; do
  TLT_ATTN_FUSED_COMBINE=$fc TLT_ATTN_DEC_MIN_CHUNK=$mc timeout 300 python tools/probe_attn_ctas.py 2>&1 | grep ctas | sed "s/^/fc=$fc mc=$mc /"
done; done | tee gpurun_out/attn_fc.txt
