#!/bin/bash
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_graph_pool.py -q -x -s 2>&1 | tail -30 > gpurun_out/r2_t3.log
timeout 1500 python -m pytest tests/test_gpu_parity_graphs.py -q -x 2>&1 | tail -30 >> gpurun_out/r2_t3.log
timeout 1500 python -m pytest tests -q -m gpu 2>&1 | tail -15 >> gpurun_out/r2_t3.log
