#!/bin/bash
# Round-2 closing pass: the default bench line, launch lists of whole SD / AR
# steps (b = 1, 8, 32) and per-launch DRAM traffic of every GEMM site at the
# two roofline M's (-> profiles/).
mkdir -p gpurun_out
timeout 1500 python bench.py > gpurun_out/fin_bench.json 2> gpurun_out/fin_bench.err
ll() {  # name -- profile_step args
  local name=$1; shift
  timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file "gpurun_out/fin_launches_$name.csv" \
    python tools/profile_step.py "$@" > "gpurun_out/fin_launches_$name.log" 2>&1
}
ll sd_b1 --b 1 --ar 1 --sd 2 --strategy 6,8,64 --prompt 512 --ctx 1200
ll sd_b8 --b 8 --ar 1 --sd 2 --strategy 6,8,32 --prompt 512 --ctx 1200
ll sd_b32 --b 32 --ar 1 --sd 2 --strategy 6,8,16 --prompt 512 --ctx 1200
# DRAM bytes per launch of each GEMM site (probe kinds) at M = 17 and 527:
# launches 4..6 of the eager warm-up pass (successive layers' weights)
for spec in 1:17 5:17 0:17 2:17 4:17 1:527 5:527 0:527 2:527 4:527; do
  timeout 300 ncu --metrics dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum --clock-control none \
    -k regex:k_gemm -s 3 -c 3 --csv --log-file "gpurun_out/fin_traffic_${spec/:/_}.csv" \
    python tools/probe.py $spec > /dev/null 2>&1
done
