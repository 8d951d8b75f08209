#!/bin/bash
timeout 600 python -m pytest tests -m gpu -x -q 2>&1 | tail -1
S="5:700:49 31:700:17 16:700:33 1:700:65 2:700:49 8:1500:33 1:1500:65"
for t in 0 1; do echo "== TC $t"; TLT_ATTN_TC=$t timeout 200 python tools/probe_attn.py $S; done
for t in 0 1; do echo "== TC $t steps"; for b in 1 5 16 31; do
  TLT_ATTN_TC=$t timeout 120 python tools/profile_step.py --model qwen2.5-7b --b $b --ar 0 --sd 3 --strategy 6,8,$([ $b = 5 ] && echo 48 || echo 16) --ctx 2400 --prompt 700 2>&1 | tail -1 | cut -c1-24; done; done
