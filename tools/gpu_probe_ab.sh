#!/bin/bash
# Engine GEMM-site probes (graph-replayed) under TLT_PDL=0 / TLT_GEMM_AUTOTUNE=0 against the defaults.
S="1:17 5:17 0:17 2:17 0:272 2:272 1:527 5:527 0:527 2:527 4:527"
echo "== default"; python tools/probe.py $S 2>&1 | grep kind
echo "== PDL=0"; TLT_PDL=0 python tools/probe.py $S 2>&1 | grep kind
echo "== AUTOTUNE=0"; TLT_GEMM_AUTOTUNE=0 python tools/probe.py $S 2>&1 | grep kind
