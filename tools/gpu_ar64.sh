#!/bin/bash
mkdir -p gpurun_out
timeout 300 ncu --metrics gpu__time_duration.sum --cache-control none --clock-control none --csv --log-file gpurun_out/launches_ar64.csv \
  python tools/profile_step.py --model qwen2.5-7b --b 64 --ar 2 --sd 0 --ctx 2048 --prompt 800 > gpurun_out/launches_ar64.log 2>&1; echo "ncu rc=$?"
timeout 300 python tools/profile_step.py --model qwen2.5-7b --b 64 --ar 4 --sd 0 --ctx 2048 --prompt 800 2>&1 | tail -2
timeout 300 python tools/profile_step.py --model qwen2.5-7b --b 32 --ar 4 --sd 0 --ctx 2048 --prompt 800 2>&1 | tail -2
