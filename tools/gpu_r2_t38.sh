#!/bin/bash
mkdir -p gpurun_out
{
echo "== all variants, graph pool tests x12"
for r in $(seq 12); do TLT_GEMM_AUTOTUNE_ALL=1 timeout 300 python -m pytest tests/test_gpu_graph_pool.py -q -x -p no:cacheprovider 2>&1 | tail -1; done
echo "== forced multicast variant tests x10"
for r in $(seq 10); do timeout 300 python -m pytest tests/test_gpu_gemm.py -q -x -p no:cacheprovider -k "variants and (6 or 7)" 2>&1 | tail -1; done
echo "== default, graph pool tests x12"
for r in $(seq 12); do timeout 300 python -m pytest tests/test_gpu_graph_pool.py -q -x -p no:cacheprovider 2>&1 | tail -1; done
} > gpurun_out/r2_t38.log 2>&1
