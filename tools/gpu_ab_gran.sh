#!/bin/bash
# same-box A/B of the flash-decode split granularity on the full bench
mkdir -p gpurun_out
for arm in old new old new; do
  if [ $arm = old ]; then export TLT_ATTN_DEC_GRAN=256; else unset TLT_ATTN_DEC_GRAN; fi
  timeout 600 python bench.py > gpurun_out/bench_$arm.json 2>/dev/null
  python -c "import json;d=json.load(open('gpurun_out/bench_$arm.json'));print('$arm',d['value'],d['e2e']['value'],d['ar_baseline']['value'],d['clocks']['sm_mhz'])" | tee -a gpurun_out/ab_gran.txt
done
