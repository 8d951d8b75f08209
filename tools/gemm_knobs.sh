#!/bin/bash
# GEMM tests, then tools/time_gemm.py at the verify shapes under each GEMM planner knob.
timeout 300 python -m pytest tests/test_gpu_gemm.py -x -q 2>&1 | tail -2
S="527:3584:4608:0 527:3584:3584:2 527:18944:3584:2 272:3584:4608:0 272:3584:3584:2 272:18944:3584:2 128:18944:3584:2 1040:18944:3584:2"
cfg() { echo "== $*"; env "$@" timeout 120 python tools/time_gemms.py $S; }
cfg TLT_GEMM_PAIR_SPLIT=0
cfg TLT_GEMM_PAIR_SPLIT=1
