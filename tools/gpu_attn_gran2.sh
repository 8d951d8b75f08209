#!/bin/bash
# new default (64-key granularity, 256-key floor) vs the old fixed 256-key splits, then tests + bench
mkdir -p gpurun_out
timeout 300 python tools/probe_attn_ctas.py 2>&1 | grep ctas | sed "s/^/new /" | tee gpurun_out/attn_gran2.txt
TLT_ATTN_DEC_GRAN=256 timeout 300 python tools/probe_attn_ctas.py 2>&1 | grep ctas | sed "s/^/old /" | tee -a gpurun_out/attn_gran2.txt
timeout 900 python -m pytest tests -m gpu -q > gpurun_out/pytest_gpu.log 2>&1; tail -2 gpurun_out/pytest_gpu.log
timeout 900 python bench.py > gpurun_out/bench.json 2> gpurun_out/bench.err; echo "bench rc=$?"
python -c "import json;d=json.load(open('gpurun_out/bench.json'));print(d['value'],d['e2e']['value'],d['ar_baseline'],d['clocks'])"
