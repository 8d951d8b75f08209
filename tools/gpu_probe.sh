#!/bin/bash
timeout 300 python -m pytest tests/test_gpu_gemm.py tests/test_gpu_parity_tiny.py -x -q 2>&1 | tail -1
timeout 200 python tools/probe.py 0:17 0:245 0:272 0:527 0:1040 2:17 2:245 2:527 5:245 1:245 3:240 3:496 4:17 4:272
