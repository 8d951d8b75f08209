#!/bin/bash
mkdir -p gpurun_out
timeout 600 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu.log 2>&1; tail -2 gpurun_out/pytest_gpu.log
timeout 300 python tools/sweep.py --batches 1 4 16 31 --depths 6 --topks 8 --budgets 16 --steps 3 --out gpurun_out/sweep_iter.jsonl > gpurun_out/sweep.log 2>&1; cat gpurun_out/sweep_iter.jsonl; tail -2 gpurun_out/sweep.log
timeout 300 ncu --metrics gpu__time_duration.sum --cache-control none --clock-control none --csv --log-file gpurun_out/launches_warm_b1.csv \
  python tools/profile_step.py --model qwen2.5-7b --b 1 --ar 2 --sd 2 --strategy 6,8,16 > gpurun_out/launches_warm_b1.log 2>&1; echo "ncu rc=$?"
