#!/bin/bash
mkdir -p gpurun_out
for r in 1 2 3; do
  timeout 1500 python -m pytest tests -q -m gpu -x -p no:cacheprovider 2>&1 | grep -v "^    " | tail -60 > gpurun_out/r2_t35_run$r.log
done
