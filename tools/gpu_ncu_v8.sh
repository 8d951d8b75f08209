#!/bin/bash
# ncu --set full of the gate_up GEMM at M = 272 under plan variants 8 and 0 (profiles/r2_ncu_gemm_v{0,8}_m272).
mkdir -p gpurun_out
TLT_GEMM_FORCE_VARIANT=8 timeout 300 ncu --set full --clock-control none --import-source on -k "regex:k_gemm" -s 2 -c 1 \
  -o gpurun_out/ncu_v8_m272 -f python tools/one_gemm.py 272 3584 37888 3 > gpurun_out/ncu_v8.log 2>&1
TLT_GEMM_FORCE_VARIANT=0 timeout 300 ncu --set full --clock-control none --import-source on -k "regex:k_gemm" -s 2 -c 1 \
  -o gpurun_out/ncu_v0_m272 -f python tools/one_gemm.py 272 3584 37888 3 > gpurun_out/ncu_v0.log 2>&1
