#!/bin/bash
mkdir -p gpurun_out
S="272:3584:37888:3 528:3584:37888:3 272:18944:3584:2 528:18944:3584:2 528:3584:4608:0 272:3584:4608:0 528:3584:3584:2 272:3584:3584:2 496:3584:152064:0 248:3584:152064:0 196:3584:37888:3 196:18944:3584:2"
{
for v in 0 1 2 3 4 6; do echo "== variant $v"; TLT_GEMM_FORCE_VARIANT=$v timeout 180 python tools/time_gemms.py $S; done
} > gpurun_out/r2_gemm_variants.txt 2>&1
