#!/bin/bash
mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_gpu_gemm.py -q -x -k variants 2>&1 | grep -v "^    " | tail -25 > gpurun_out/r2_t32.log
S="272:3584:37888:3 528:3584:37888:3 1024:3584:37888:3 528:3584:4608:0 528:18944:3584:2 512:3584:152064:0 256:3584:152064:0"
{ for v in 0 7; do echo "== variant $v"; TLT_GEMM_FORCE_VARIANT=$v timeout 180 python tools/time_gemms.py $S; done; } > gpurun_out/r2_gemm_mc.txt 2>&1
