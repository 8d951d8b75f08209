#!/bin/bash
S="1:245 1:527 5:245 5:527 2:527"
echo "== default"; timeout 200 python tools/probe.py $S
echo "== pure pair"; TLT_GEMM_PAIR_MIN_CTAS=1 TLT_GEMM_PAIR_SPLIT=0 timeout 200 python tools/probe.py $S
echo "== pure pair persistent"; TLT_GEMM_PAIR_MIN_CTAS=1 TLT_GEMM_PAIR_SPLIT=0 TLT_GEMM_PAIR_PERSIST_MIN_M=200 timeout 200 python tools/probe.py $S
echo "== 1cta bn256"; TLT_GEMM_PAIR_MIN_M=100000 TLT_GEMM_BN_MAX=256 timeout 200 python tools/probe.py $S
