#!/bin/bash
mkdir -p gpurun_out
run() { echo "== $*"; timeout 120 env "$@" python tools/profile_step.py --b 16 --ar 1 --sd 3 --strategy 6,8,16 --graphs 0 2>&1 | tail -4; echo "rc=$?"; }
{
run TLT_GEMM_PAIR_MIN_M=0
run TLT_GEMM_PAIR_MIN_M=192 TLT_PDL=0
run TLT_GEMM_PAIR_MIN_M=192
run TLT_GEMM_PAIR_MIN_M=192 TLT_GEMM_PAIR_CPS=1
} > gpurun_out/diag.log 2>&1
cat gpurun_out/diag.log
