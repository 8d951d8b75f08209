#!/bin/bash
mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_experiment.py -q -x 2>&1 | grep -v "^    " | tail -30 > gpurun_out/r2_t10.log
bash tools/gpu_r2_gemm_sweep.sh
