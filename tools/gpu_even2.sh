#!/bin/bash
mkdir -p gpurun_out
timeout 300 python tools/probe_attn_ctas.py 2>&1 | grep ctas | sed "s/^/short1 /" | tee gpurun_out/attn_even2.txt
timeout 900 python -m pytest tests -m gpu -q > gpurun_out/pytest_gpu.log 2>&1; tail -2 gpurun_out/pytest_gpu.log | tee -a gpurun_out/attn_even2.txt
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; tail -1 gpurun_out/smoke.log
