#!/bin/bash
# GEMM diagnostics: per plan variant, full / loads-only (TLT_GEMM_DBG=1) /
# no-epilogue (2) / neither (3) timings at the verify shapes.
#   bash tools/gpu_gemm_diag.sh "0 1 2 8" > gpurun_out/gemm_diag.txt
vars=${1:-"0 1 2 8"}
shapes="272:3584:37888:3 528:3584:37888:3 528:18944:3584:2 528:3584:4608:0 528:3584:3584:2 496:3584:152064:0"
for v in $vars; do for d in 0 1 2; do
  echo "== variant $v dbg $d"
  TLT_GEMM_FORCE_VARIANT=$v TLT_GEMM_DBG=$d timeout 120 python tools/time_gemms.py $shapes 2>&1 | grep -v Warn
done; done
