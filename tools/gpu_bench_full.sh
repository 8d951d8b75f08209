#!/bin/bash
# Round checkpoint: GPU tests, bench line, launch list, ncu --set full of the rooflined GEMMs.
mkdir -p gpurun_out
timeout 600 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu.log 2>&1; tail -1 gpurun_out/pytest_gpu.log
timeout 900 python bench.py > gpurun_out/bench.json 2> gpurun_out/bench.err; echo "bench rc=$?"; tail -2 gpurun_out/bench.err
for spec in "17 3584 37888 3" "527 3584 37888 3" "1 3584 37888 3" "17 18944 3584 0" "527 18944 3584 0" "496 3584 152064 0"; do
  set -- $spec
  timeout 300 ncu --set full --clock-control none --import-source on -k regex:k_gemm -c 1 -s 2 \
    -o gpurun_out/gemm_m$1_k$2_n$3 -f python tools/one_gemm.py $1 $2 $3 $4 > gpurun_out/ncu_gemm_m$1_k$2.log 2>&1; echo "ncu $spec rc=$?"
done
timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_b1.csv \
  python tools/profile_step.py --model qwen2.5-7b --b 1 --ar 1 --sd 2 --strategy 6,8,16 > gpurun_out/launches_b1.log 2>&1; echo "ncu launches rc=$?"
