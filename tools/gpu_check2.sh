#!/bin/bash
mkdir -p gpurun_out
timeout 600 python -m pytest tests -m gpu -x -q 2>&1 | tail -4
timeout 300 python tools/sweep.py --batches 1 4 16 31 --depths 6 --topks 8 --budgets 16 --steps 3 --out gpurun_out/sweep_iter.jsonl > gpurun_out/sweep.log 2>&1; cat gpurun_out/sweep_iter.jsonl; tail -2 gpurun_out/sweep.log
B=31 BENCH=0 bash tools/gpu_prof.sh
