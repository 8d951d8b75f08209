#!/bin/bash
run() { echo "== $*"; env "$@" TLT_TRACE=1 timeout 300 python bench.py --steps 1 --warmup 1 --ar-baseline 0 --cpu-gen 0 > gpurun_out/b.json 2> gpurun_out/b.err; echo "rc=$?"; tail -2 gpurun_out/b.err; head -c 300 gpurun_out/b.json; echo; }
run TLT_GEMM_PAIR_SPLIT=0
run TLT_ATTN_FUSED_COMBINE=0
