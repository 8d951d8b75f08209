#!/bin/bash
# auto fused-combine: probe, GPU suite, then same-box bench A/B (auto vs off)
mkdir -p gpurun_out
timeout 300 python tools/probe_attn_ctas.py 2>&1 | grep ctas | sed "s/^/auto /" | tee gpurun_out/fc_auto.txt
timeout 900 python -m pytest tests -m gpu -q > gpurun_out/pytest_gpu.log 2>&1; tail -2 gpurun_out/pytest_gpu.log
for arm in off auto off auto; do
  if [ $arm = off ]; then export TLT_ATTN_FUSED_COMBINE=0; else unset TLT_ATTN_FUSED_COMBINE; fi
  timeout 600 python bench.py > gpurun_out/bench_$arm.json 2>/dev/null
  python -c "import json;d=json.load(open('gpurun_out/bench_$arm.json'));print('$arm',d['value'],d['e2e']['value'],d['ar_baseline']['value'],d['clocks']['sm_mhz'])" | tee -a gpurun_out/fc_auto.txt
done
