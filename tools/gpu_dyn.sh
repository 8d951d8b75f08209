#!/bin/bash
# per-request decode split sizing (TLT_ATTN_DEC_DYN): tests, probe, same-box bench A/B
mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu.log 2>&1; tail -2 gpurun_out/pytest_gpu.log | tee gpurun_out/dyn.txt
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; tail -1 gpurun_out/smoke.log | tee -a gpurun_out/dyn.txt
for e in 0 1; do TLT_ATTN_DEC_DYN=$e timeout 300 python tools/probe_attn_ctas.py 2>&1 | grep ctas | sed "s/^/dyn=$e /"; done | tee -a gpurun_out/dyn.txt
for arm in 0 1 0 1; do
  TLT_ATTN_DEC_DYN=$arm timeout 600 python bench.py > gpurun_out/bench_dyn$arm.json 2>/dev/null
  python -c "import json;d=json.load(open('gpurun_out/bench_dyn$arm.json'));print('dyn=$arm',d['value'],d['e2e']['value'],d['ar_baseline']['value'],d['clocks']['sm_mhz'])" | tee -a gpurun_out/dyn.txt
done
