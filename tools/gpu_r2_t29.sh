#!/bin/bash
mkdir -p gpurun_out
timeout 1500 python bench.py --steps 2 --warmup 2 --cpu-rows 0 --bucket-steps 0 > gpurun_out/r2_spot_off.json 2> gpurun_out/r2_spot_off.err
timeout 1800 python bench.py --steps 2 --warmup 2 --cpu-rows 0 --bucket-steps 0 --spot-train-iters 20 > gpurun_out/r2_spot_on.json 2> gpurun_out/r2_spot_on.err
