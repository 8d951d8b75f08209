#!/bin/bash
timeout 300 python -m pytest tests/test_gpu_gemm.py -x -q 2>&1 | tail -1
for v in 0 1; do echo "== wm2 $v"; TLT_GEMM_PAIR_WM2=$v timeout 200 python tools/probe.py 0:384 0:496 0:527 0:768 0:1040 3:496 3:1040; done
