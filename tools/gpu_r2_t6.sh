#!/bin/bash
mkdir -p gpurun_out
timeout 900 compute-sanitizer --tool memcheck --print-limit 3 python -m pytest tests/test_gpu_graph_pool.py -q -x 2>&1 | grep -v "^    " | head -80 > gpurun_out/r2_t6.log
timeout 900 python -m pytest tests/test_gpu_attention.py -q -x 2>&1 | tail -20 >> gpurun_out/r2_t6.log
