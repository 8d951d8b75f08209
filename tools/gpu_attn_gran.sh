#!/bin/bash
mkdir -p gpurun_out
for g in 256 128 64; do
  TLT_ATTN_DEC_GRAN=$g timeout 300 python tools/probe_attn_ctas.py 2>&1 | grep ctas | sed "s/^/gran=$g /"
done | tee gpurun_out/attn_gran.txt
for g in 256 64; do
  TLT_ATTN_DEC_GRAN=$g timeout 300 python tools/profile_step.py --model qwen2.5-7b --b 1 --ar 6 --sd 0 --ctx 1536 --prompt 1024 --graphs 1 2>&1 | tail -3 | sed "s/^/gran=$g /"
done | tee -a gpurun_out/attn_gran.txt
