#!/bin/bash
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_experiment.py tests/test_gpu_attention.py tests/test_gpu_graph_pool.py -q -x 2>&1 | tail -5 > gpurun_out/r2_t8.log
python tools/probe_attn.py 1:1024:1 8:1024:1 32:1024:1 64:1024:1 1:1024:65 5:700:49 16:700:17 31:700:17 > gpurun_out/r2_probe_attn_graph.txt 2>&1
timeout 1500 python bench.py --steps 2 --warmup 1 > gpurun_out/r2_bench_pool.json 2> gpurun_out/r2_bench_pool.err
timeout 1500 python bench.py --steps 2 --warmup 1 --graph-pool 0 --cpu-rows 0 --bucket-steps 0 > gpurun_out/r2_bench_nopool.json 2> gpurun_out/r2_bench_nopool.err
