#!/bin/bash
timeout 200 python -m pytest tests/test_gpu_attention.py -x -q 2>&1 | tail -1
S="5:700:49 31:700:17 16:700:33 1:700:65 8:1500:33"
for t in 0 1; do echo "== TC $t"; TLT_ATTN_TC=$t timeout 200 python tools/probe_attn.py $S; done
