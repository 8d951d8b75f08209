#!/bin/bash
timeout 300 python -m pytest tests/test_gpu_gemm.py -x -q 2>&1 | tail -1
TLT_GEMM_MAX_SPLITS=16 timeout 300 python -m pytest tests/test_gpu_gemm.py -x -q 2>&1 | tail -1
for v in 8 10 12 16; do echo "== max splits $v"; TLT_GEMM_MAX_SPLITS=$v timeout 200 python tools/probe.py 5:1 5:17 5:48 2:1 2:17 2:48 0:1 0:17; done
