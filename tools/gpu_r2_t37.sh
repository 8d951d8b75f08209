#!/bin/bash
mkdir -p gpurun_out
for r in 1 2 3 4 5; do
  timeout 1500 python -m pytest tests -q -m gpu -p no:cacheprovider -x 2>&1 > gpurun_out/r2_t37_full$r.log
  tail -1 gpurun_out/r2_t37_full$r.log
done > gpurun_out/r2_t37.log
