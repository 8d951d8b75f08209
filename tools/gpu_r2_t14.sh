#!/bin/bash
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_parity_tiny.py tests/test_gpu_neural_7b.py -q -x 2>&1 | grep -v "^    " | tail -40 > gpurun_out/r2_t14.log
