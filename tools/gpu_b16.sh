#!/bin/bash
mkdir -p gpurun_out
timeout 300 python tools/sweep.py --batches 16 31 --depths 6 --topks 8 --budgets 16 --steps 3 --out gpurun_out/sweep_iter.jsonl > gpurun_out/sweep.log 2>&1; echo "sweep rc=$?"; cat gpurun_out/sweep.log | tail -5
timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_b16.csv \
  python tools/profile_step.py --model qwen2.5-7b --b 16 --ar 1 --sd 2 --strategy 6,8,16 > gpurun_out/launches_b16.log 2>&1; echo "ncu rc=$?"
timeout 900 python bench.py > gpurun_out/bench.json 2> gpurun_out/bench.err; echo "bench rc=$?"; cat gpurun_out/bench.json; tail -3 gpurun_out/bench.err
