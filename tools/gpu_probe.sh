#!/bin/bash
timeout 600 python -m pytest tests -m gpu -x -q 2>&1 | tail -1
S="1:1 1:16 1:48 1:100 1:245 1:343 5:1 5:48 5:245 5:527 2:1 2:48 2:245 2:527 0:245"
cfg() { echo "== $*"; env "$@" timeout 200 python tools/probe.py $S; }
cfg X=1
cfg TLT_GEMM_PAIR_SPLIT=0
