#!/bin/bash
# GEMM shape sweep + default-arm strategy sweep + ncu full capture of gate_up.
mkdir -p gpurun_out
for m in 17 128 256 528 1024 2048 4096; do
  for kn in "3584 37888 3" "18944 3584 0" "3584 4608 0" "3584 152064 0"; do
    echo "M=$m KN=$kn $(timeout 60 python tools/time_gemm.py $m $kn)"; done; done > gpurun_out/gemm_times.txt 2>&1
timeout 900 python tools/sweep.py --batches 1 4 16 31 --depths 6 10 --topks 8 --budgets 16 32 64 --steps 3 \
  --out gpurun_out/sweep_default_arms.jsonl > gpurun_out/sweep.log 2>&1
timeout 300 ncu --set full --clock-control none --import-source on -k k_gemm_swapab -c 1 -s 3 \
  -o gpurun_out/gateup_m1024 -f python tools/one_gemm.py 1024 3584 37888 3 > gpurun_out/ncu1.log 2>&1
timeout 300 ncu --set full --clock-control none --import-source on -k k_gemm_swapab -c 1 -s 3 \
  -o gpurun_out/gateup_m17 -f python tools/one_gemm.py 17 3584 37888 3 > gpurun_out/ncu2.log 2>&1
cat gpurun_out/gemm_times.txt; cat gpurun_out/sweep_default_arms.jsonl
