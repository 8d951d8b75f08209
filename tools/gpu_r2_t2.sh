#!/bin/bash
mkdir -p gpurun_out
timeout 900 python -m pytest tests -q -m gpu -x -k "rollout_result or handback" 2>&1 | tail -30 > gpurun_out/r2_t2.log
