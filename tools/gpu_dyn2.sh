#!/bin/bash
mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu.log 2>&1; tail -2 gpurun_out/pytest_gpu.log | tee gpurun_out/dyn2.txt
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; tail -1 gpurun_out/smoke.log | tee -a gpurun_out/dyn2.txt
timeout 300 python tools/probe_attn_ctas.py 2>&1 | grep ctas | sed "s/^/dyn=1 floor256 /" | tee -a gpurun_out/dyn2.txt
timeout 600 python bench.py > gpurun_out/bench.json 2> gpurun_out/bench.err; echo "bench rc=$?" | tee -a gpurun_out/dyn2.txt
python -c "import json;d=json.load(open('gpurun_out/bench.json'));print(d['value'],d['e2e']['value'],d['ar_baseline']['value'],d['clocks']['sm_mhz'])" | tee -a gpurun_out/dyn2.txt
