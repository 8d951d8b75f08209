#!/bin/bash
mkdir -p gpurun_out
timeout 1800 python -m pytest tests -q -m gpu -x 2>&1 | grep -v "^    " | tail -40 > gpurun_out/r2_t34.log
