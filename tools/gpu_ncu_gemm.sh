#!/bin/bash
# GPU parity tests, then ncu --set full of the gate_up GEMM at verify/decode M.
mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_gpu.log; tail -3 gpurun_out/pytest_gpu.log
for m in ${NCU_MS:-272 17}; do
timeout 300 ncu --set full --clock-control none --import-source on -k regex:k_gemm_swapab -c 1 -s 2 \
  -o gpurun_out/gateup_m$m -f python tools/one_gemm.py $m 3584 37888 3 > gpurun_out/ncu_m$m.log 2>&1; echo "ncu m=$m rc=$?"
done
timeout 300 python tools/sweep.py --batches 1 16 31 --depths 6 --topks 8 --budgets 16 --steps 3 --out gpurun_out/sweep_iter.jsonl > gpurun_out/sweep.log 2>&1; cat gpurun_out/sweep_iter.jsonl
