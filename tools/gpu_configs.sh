#!/bin/bash
# Config 4 (32B stochastic rollout, tools/config4.py) and the config-5 strategy sweep (tools/sweep.py).
mkdir -p gpurun_out
timeout 1500 python tools/config4.py > gpurun_out/config4.json 2> gpurun_out/config4.err; echo "config4 rc=$?"; tail -4 gpurun_out/config4.err; cat gpurun_out/config4.json
timeout 1500 python tools/sweep.py --batches 1 8 32 128 --steps 3 --out gpurun_out/sweep_full.jsonl > gpurun_out/sweep_full.log 2>&1; echo "sweep rc=$?"; wc -l gpurun_out/sweep_full.jsonl
