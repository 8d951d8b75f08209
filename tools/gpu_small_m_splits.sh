#!/bin/bash
# split-K cap sweep for the small-M QKV / O-proj / down GEMMs (graph-replayed engine probes)
for s in 8 4 2 16; do echo "== TLT_GEMM_MAX_SPLITS=$s"; TLT_GEMM_MAX_SPLITS=$s timeout 300 python tools/probe.py 1:17 5:17 2:17 1:65 5:65 2:65 2>&1 | grep kind; done
