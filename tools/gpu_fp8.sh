#!/bin/bash
for v in 0 1; do echo "== drafter fp8 $v"; for bs in "1 16" "5 48" "11 32" "31 16"; do set -- $bs
  TLT_DRAFTER_FP8=$v timeout 120 python tools/profile_step.py --model qwen2.5-7b --b $1 --ar 0 --sd 3 --strategy 6,8,$2 --ctx 2400 --prompt 700 2>&1 | tail -1 | cut -c1-50; done; done
