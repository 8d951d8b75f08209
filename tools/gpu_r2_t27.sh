#!/bin/bash
mkdir -p gpurun_out
timeout 2400 python -m pytest tests -q -m gpu 2>&1 | tail -8 > gpurun_out/r2_t27.log
timeout 420 ncu --set full --clock-control none --import-source on -k "regex:attention_tree_tc" -s 20 -c 1 \
  -o gpurun_out/r2_ncu_tree_tc_b31 -f python tools/probe_attn.py 31:700:17 > gpurun_out/r2_ncu_tree_tc.log 2>&1
for nm in 256 0; do
  TLT_CLUSTER_NORM_MAX_M=$nm timeout 900 python bench.py --steps 1 --warmup 1 --cpu-rows 0 --len-median 400 --max-len 2048 > gpurun_out/r2_ab_norm$nm.json 2> gpurun_out/r2_ab_norm$nm.err
done
