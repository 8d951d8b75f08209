#!/bin/bash
mkdir -p gpurun_out
T=tests/test_gpu_neural_7b.py::test_7b_logits_rows_and_hidden_states_match_oracle
( echo "== default"; TLT_GEMM_AUTOTUNE_LOG=1 timeout 600 python -m pytest $T -q -x 2>&1 | grep -E "passed|failed|autotune" | head -40
  echo "== autotune off"; TLT_GEMM_AUTOTUNE=0 timeout 600 python -m pytest $T -q -x 2>&1 | tail -1
  echo "== tma off"; TLT_ATTN_TMA=0 timeout 600 python -m pytest $T -q -x 2>&1 | tail -1 ) > gpurun_out/r2_t15.log 2>&1
