#!/bin/bash
mkdir -p gpurun_out
timeout 900 compute-sanitizer --tool memcheck --print-limit 3 python -m pytest tests/test_gpu_graph_pool.py -q -x 2>&1 | grep -v "^    " | tail -30 > gpurun_out/r2_t7.log
timeout 900 python -m pytest tests/test_gpu_attention.py -q -x 2>&1 | tail -20 >> gpurun_out/r2_t7.log
timeout 1800 python -m pytest tests -q -m gpu 2>&1 | tail -20 >> gpurun_out/r2_t7.log
python tools/sweep_attn.py > gpurun_out/r2_attn_sweep.txt 2>&1
