#!/bin/bash
mkdir -p gpurun_out
timeout 120 python -m pytest tests/test_gpu_gemm.py -x -q > gpurun_out/pytest_gemm.log 2>&1; echo "rc=$?" >> gpurun_out/pytest_gemm.log
tail -15 gpurun_out/pytest_gemm.log
grep -q "rc=0" gpurun_out/pytest_gemm.log || exit 1
GEMM_MS="272 528 1024 2048" SWEEP_B="1 16 31" BENCH=1 bash tools/gpu_iter.sh
