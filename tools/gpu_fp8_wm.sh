#!/bin/bash
# e4m3 drafter LM head: one-CTA-per-row quantiser + TLT_FP8_WM (256 weight rows per CTA) A/B
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_gemm_e4m3.py tests/test_gpu_parity_tiny.py -q -x -p no:cacheprovider > gpurun_out/fp8_tests.log 2>&1; tail -3 gpurun_out/fp8_tests.log
for wm in 1 2; do echo "== TLT_FP8_WM=$wm"; TLT_FP8_WM=$wm timeout 300 python tools/probe.py 6:8 6:64 6:128 6:248 2>&1 | grep kind; done > gpurun_out/fp8_probe.txt
bash tools/gpu_ab_bench.sh TLT_FP8_WM "2 1" 1 > gpurun_out/fp8_ab.log 2>&1
