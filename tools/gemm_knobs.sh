#!/bin/bash
S="527:3584:4608:0 527:3584:3584:2 527:18944:3584:2 272:3584:4608:0 272:3584:3584:2 272:18944:3584:2 1024:18944:3584:2"
cfg() { echo "== $*"; env "$@" timeout 120 python tools/time_gemms.py $S; }
{
cfg TLT_GEMM_PAIR_MIN_CTAS=148
cfg TLT_GEMM_PAIR_MIN_CTAS=1
cfg TLT_GEMM_PAIR_MIN_CTAS=1 TLT_GEMM_PAIR_BN_MAX=128
cfg TLT_GEMM_PAIR_MIN_CTAS=1 TLT_GEMM_PAIR_BN_MAX=96
cfg TLT_GEMM_PAIR_MIN_CTAS=1 TLT_GEMM_PAIR_BN_MAX=64
cfg TLT_GEMM_PAIR_MIN_M=100000 TLT_GEMM_BN_MAX=64
cfg TLT_GEMM_PAIR_MIN_M=100000 TLT_GEMM_BN_MAX=256
} > gpurun_out/gemm_knobs.txt 2>&1
cat gpurun_out/gemm_knobs.txt
timeout 300 ncu --set full --clock-control none --import-source on -k regex:k_row_topk_chunk -c 1 -s 8 -o gpurun_out/topk_chunk -f \
  python tools/profile_step.py --model qwen2.5-7b --b 31 --ar 0 --sd 1 --strategy 6,8,16 > gpurun_out/ncu_topk.log 2>&1; echo "ncu rc=$?"
