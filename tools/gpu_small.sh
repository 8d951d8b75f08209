#!/bin/bash
# warm per-launch times of the small decode GEMM sites, PDL off / on
for p in 0 gemm; do echo "TLT_PDL=$p"; TLT_PDL=$p python tools/probe.py 1:1 5:1 0:1 2:1 4:1 1:17 5:17 0:17 2:17 $EXTRA; done
