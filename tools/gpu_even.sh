#!/bin/bash
# even key splits (TLT_ATTN_DEC_EVEN) A/B: probe, decode step time, attention tests
mkdir -p gpurun_out
for e in 0 1; do
  TLT_ATTN_DEC_EVEN=$e timeout 300 python tools/probe_attn_ctas.py 2>&1 | grep ctas | sed "s/^/even=$e /"
  TLT_ATTN_DEC_EVEN=$e timeout 300 python tools/profile_step.py --model qwen2.5-7b --b 1 --ar 5 --sd 0 --ctx 1536 --prompt 256 2>&1 | tail -2 | sed "s/^/even=$e /"
done | tee gpurun_out/attn_even.txt
timeout 600 python -m pytest tests/test_gpu_attention.py tests/test_gpu_parity_tiny.py -q 2>&1 | tail -2 | tee -a gpurun_out/attn_even.txt
