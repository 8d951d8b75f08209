#!/bin/bash
S="1:1 1:17 1:48 1:100 5:1 5:17 5:48"
for c in 4 8 2; do echo "== qkv max splits $c"; TLT_QKV_MAX_SPLITS=$c timeout 200 python tools/probe.py $S; done
for c in 8 4; do echo "== global max splits $c"; TLT_GEMM_MAX_SPLITS=$c timeout 200 python tools/probe.py 5:1 5:17 5:48 2:1 2:17 2:48; done
