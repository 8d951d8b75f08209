#!/bin/bash
# GEMM config sweep at one shape: M K N kind
for cfg in "0 0 256" "1 0 256" "2 0 256" "1 0 128" "2 0 128" "1 0 64" "2 0 64" "1 3 256" "1 6 128" "2 2 256"; do
  set -- $cfg
  echo "wm=$1 stages=$2 bnmax=$3 :: $(TLT_GEMM_WM=$1 TLT_GEMM_STAGES=$2 TLT_GEMM_BN_MAX=$3 python tools/time_gemm.py $M $K $N $KIND)"
done
