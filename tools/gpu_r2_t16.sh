#!/bin/bash
mkdir -p gpurun_out
T="tests/test_gpu_parity_tiny.py tests/test_gpu_neural_7b.py"
( echo "== default"; timeout 600 python -m pytest $T -q -x 2>&1 | tail -1
  echo "== autotune off"; TLT_GEMM_AUTOTUNE=0 timeout 600 python -m pytest $T -q -x 2>&1 | tail -1
  echo "== tma off"; TLT_ATTN_TMA=0 timeout 600 python -m pytest $T -q -x 2>&1 | tail -1
  echo "== tree dyn off"; TLT_ATTN_TREE_DYN=0 timeout 600 python -m pytest $T -q -x 2>&1 | tail -1
  echo "== only 7b after one tiny test"; timeout 600 python -m pytest tests/test_gpu_parity_tiny.py::test_rollout_tokens_match_oracle tests/test_gpu_neural_7b.py -q -x 2>&1 | tail -1
) > gpurun_out/r2_t16.log 2>&1
