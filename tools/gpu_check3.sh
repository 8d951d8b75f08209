#!/bin/bash
mkdir -p gpurun_out
timeout 600 python -m pytest tests -m gpu -x -q 2>&1 | tail -2
timeout 300 python tools/sweep.py --batches 1 16 31 --depths 6 --topks 8 --budgets 16 --steps 3 --out gpurun_out/sweep_iter.jsonl > gpurun_out/sweep.log 2>&1; cat gpurun_out/sweep_iter.jsonl; tail -2 gpurun_out/sweep.log
B=31 BENCH=0 bash tools/gpu_prof.sh
timeout 300 ncu --set full --clock-control none --import-source on -k regex:k_row_topk_chunk -c 1 -s 3 -o gpurun_out/topk_chunk -f \
  python tools/profile_step.py --model qwen2.5-7b --b 31 --ar 0 --sd 1 --strategy 6,8,16 > gpurun_out/ncu_topk.log 2>&1; echo "ncu rc=$?"
