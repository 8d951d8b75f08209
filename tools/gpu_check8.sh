#!/bin/bash
for v in 256 64 16; do echo "== cluster norm max M $v"; for b in 1 5 16 31; do
  TLT_CLUSTER_NORM_MAX_M=$v timeout 120 python tools/profile_step.py --model qwen2.5-7b --b $b --ar 3 --sd 3 --strategy 6,8,$([ $b = 5 ] && echo 48 || echo 16) --ctx 2400 --prompt 700 2>&1 | grep -E "ar ms|sd ms" | tail -2 | cut -c1-30 | tr '\n' ' '; echo; done; done
