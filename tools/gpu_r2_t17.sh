#!/bin/bash
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_attention.py -q -x 2>&1 | grep -v "^    " | tail -20 > gpurun_out/r2_t17.log
timeout 1800 python -m pytest tests -q -m gpu 2>&1 | tail -8 >> gpurun_out/r2_t17.log
