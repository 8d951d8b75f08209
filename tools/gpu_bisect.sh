#!/bin/bash
run() { echo "== $*"; timeout 90 env "$@" python tools/profile_step.py --model qwen2.5-7b --b 5 --ar 1 --sd 2 --strategy 10,8,48 --ctx 2400 --prompt 256 2>&1 | tail -2; echo "rc=$?"; }
run TLT_GEMM_PAIR_SPLIT=0
run TLT_GEMM_PAIR_SPLIT=1
run TLT_GEMM_PAIR_SPLIT=1 TLT_PDL=0
run TLT_GEMM_PAIR_SPLIT=1 TLT_ATTN_FUSED_COMBINE=0
