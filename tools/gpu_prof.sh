#!/bin/bash
mkdir -p gpurun_out
B=${B:-31}
timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_b$B.csv \
  python tools/profile_step.py --model qwen2.5-7b --b $B --ar 1 --sd 2 --strategy ${STRAT:-6,8,16} > gpurun_out/launches_b$B.log 2>&1; echo "ncu rc=$?"
if [ "${BENCH:-1}" = 1 ]; then timeout 900 python bench.py > gpurun_out/bench.json 2> gpurun_out/bench.err; echo "bench rc=$?"; cat gpurun_out/bench.json; tail -3 gpurun_out/bench.err; fi
