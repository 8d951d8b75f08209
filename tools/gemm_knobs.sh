#!/bin/bash
timeout 180 python -m pytest tests/test_gpu_gemm.py -x -q 2>&1 | tail -3
TLT_GEMM_PERSIST=0 timeout 180 python -m pytest tests/test_gpu_gemm.py -x -q 2>&1 | tail -3
timeout 600 python -m pytest tests -m gpu -x -q 2>&1 | tail -3
S="1:3584:37888:3 17:3584:37888:3 64:3584:37888:3 128:3584:37888:3 272:3584:37888:3 528:3584:37888:3 1024:3584:37888:3 528:3584:152064:0 272:3584:152064:0 272:18944:3584:0 528:18944:3584:0 1024:18944:3584:0 2048:18944:3584:0 1024:3584:4608:0 2048:3584:4608:0"
cfg() { echo "== $*"; env "$@" timeout 120 python tools/time_gemms.py $S; }
{
cfg TLT_GEMM_PERSIST=0
cfg TLT_GEMM_PERSIST=2
cfg TLT_GEMM_PERSIST=2 TLT_GEMM_PERSIST1_MIN_M=1
} > gpurun_out/gemm_knobs.txt 2>&1
cat gpurun_out/gemm_knobs.txt
timeout 300 python tools/sweep.py --batches 1 4 16 31 --depths 6 --topks 8 --budgets 16 --steps 3 --out gpurun_out/sweep_iter.jsonl > gpurun_out/sweep.log 2>&1; cat gpurun_out/sweep_iter.jsonl
