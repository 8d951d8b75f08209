#!/bin/bash
# Iteration check: GPU tests, GEMM shape times, a short strategy sweep, bench.
mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_gpu.log
tail -3 gpurun_out/pytest_gpu.log
for m in ${GEMM_MS:-1 17 128 272 528 1024 2048}; do
  for kn in "3584 37888 3" "18944 3584 0" "3584 4608 0" "3584 3584 0" "3584 152064 0"; do
    echo "M=$m KN=$kn $(timeout 60 python tools/time_gemm.py $m $kn)"; done; done > gpurun_out/gemm_times.txt 2>&1
cat gpurun_out/gemm_times.txt
timeout 600 python tools/sweep.py --batches ${SWEEP_B:-1 16 31} --depths 6 --topks 8 --budgets 16 --steps 3 \
  --out gpurun_out/sweep_iter.jsonl > gpurun_out/sweep.log 2>&1; cat gpurun_out/sweep_iter.jsonl
if [ "${BENCH:-1}" = 1 ]; then timeout 900 python bench.py > gpurun_out/bench.json 2> gpurun_out/bench.err; cat gpurun_out/bench.json; tail -3 gpurun_out/bench.err; fi
