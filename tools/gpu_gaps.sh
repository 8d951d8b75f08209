#!/bin/bash
mkdir -p gpurun_out
timeout 600 python -m pytest tests -m gpu -x -q 2>&1 | tail -2
timeout 300 ncu --metrics gpu__time_duration.sum --cache-control none --clock-control none --csv --log-file gpurun_out/launches_warm_b1.csv \
  python tools/profile_step.py --model qwen2.5-7b --b 1 --ar 2 --sd 2 --strategy 6,8,16 > gpurun_out/launches_warm_b1.log 2>&1; echo "ncu rc=$?"
cat gpurun_out/launches_warm_b1.log | tail -4
TLT_PDL=0 timeout 300 python tools/profile_step.py --model qwen2.5-7b --b 1 --ar 4 --sd 3 --strategy 6,8,16 2>&1 | tail -4
timeout 300 python tools/profile_step.py --model qwen2.5-7b --b 1 --ar 4 --sd 3 --strategy 6,8,16 2>&1 | tail -4
