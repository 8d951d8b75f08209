#!/bin/bash
timeout 600 python -m pytest tests -m gpu -x -q 2>&1 | tail -1
S="64:1024:1 48:700:1 40:700:1 32:700:1 16:700:1 1:1024:1 64:300:1"
timeout 200 python tools/probe_attn.py $S
for b in 64 48 32; do timeout 120 python tools/profile_step.py --model qwen2.5-7b --b $b --ar 4 --sd 0 --ctx 2400 --prompt 700 2>&1 | tail -1; done
