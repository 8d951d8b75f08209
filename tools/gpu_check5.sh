#!/bin/bash
mkdir -p gpurun_out
timeout 600 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu.log 2>&1; tail -1 gpurun_out/pytest_gpu.log
for b in 64 32; do timeout 300 python tools/profile_step.py --model qwen2.5-7b --b $b --ar 4 --sd 0 --ctx 2048 --prompt 800 2>&1 | tail -1; done
timeout 300 python tools/sweep.py --batches 1 4 16 31 --depths 6 --topks 8 --budgets 16 --steps 3 --out gpurun_out/sweep_iter.jsonl > gpurun_out/sweep.log 2>&1; cat gpurun_out/sweep_iter.jsonl
