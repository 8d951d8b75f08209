#!/bin/bash
# multicast-cluster skip fix: live-row GEMM tests, pool loop with all variants;
# fused top-8 drafter LM head A/B on the bench
mkdir -p gpurun_out
{
timeout 600 python -m pytest tests/test_gpu_gemm.py -q -x -p no:cacheprovider 2>&1 | tail -3
echo "== all variants, graph pool tests x12"
for r in $(seq 12); do TLT_GEMM_AUTOTUNE_ALL=1 timeout 300 python -m pytest tests/test_gpu_graph_pool.py -q -x -p no:cacheprovider 2>&1 | tail -1; done
echo "== bench default"
timeout 900 python bench.py --steps 2 --warmup 3 2>&1 | tail -1
echo "== bench fused top-8"
TLT_FUSED_TOPK_K=8 timeout 900 python bench.py --steps 2 --warmup 3 2>&1 | tail -1
} > gpurun_out/r2_t39.log 2>&1
