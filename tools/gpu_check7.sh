#!/bin/bash
timeout 600 python -m pytest tests -m gpu -x -q 2>&1 | tail -1
for b in 1 5 16 31; do
  timeout 120 python tools/profile_step.py --model qwen2.5-7b --b $b --ar 0 --sd 3 --strategy 6,8,$([ $b = 5 ] && echo 48 || echo 16) --ctx 2400 --prompt 700 2>&1 | tail -1 | cut -c1-40; done
