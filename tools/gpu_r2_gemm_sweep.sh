#!/bin/bash
# mid-M GEMM knob sweep (verify / drafter shapes of the 7B model)
mkdir -p gpurun_out
S="272:3584:37888:3 528:3584:37888:3 1040:3584:37888:3 272:18944:3584:2 528:18944:3584:2 1040:18944:3584:2 496:3584:152064:0 248:3584:152064:0 528:3584:4608:0 528:3584:3584:2"
cfg() { echo "== $*"; env "$@" timeout 180 python tools/time_gemms.py $S; }
{
cfg TLT_GEMM_X=0
cfg TLT_GEMM_PAIR_CPS=1
cfg TLT_GEMM_PAIR_BN_MAX=128
cfg TLT_GEMM_PAIR_PERSIST_MIN_M=256
cfg TLT_GEMM_PAIR_WM2=1
cfg TLT_GEMM_PAIR_MIN_CTAS=296
cfg TLT_GEMM_PAIR_MIN_M=100000
} > gpurun_out/r2_gemm_sweep.txt 2>&1
