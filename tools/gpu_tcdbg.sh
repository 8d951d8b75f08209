#!/bin/bash
for s in 1 2 4 0; do echo "== stage $s"; TLT_ATTN_TC_DBG=$s timeout 60 python -m pytest tests/test_gpu_attention.py -x -q -k "1-2-17-300" 2>&1 | tail -2; echo "rc=$?"; done
