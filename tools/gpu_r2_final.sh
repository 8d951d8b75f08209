#!/bin/bash
# Round-2 final pass: GPU tests, the bench line, launch lists of whole steps
# and ncu --set full captures of the dominant kernels (summaries -> profiles/).
mkdir -p gpurun_out
timeout 2400 python -m pytest tests -q -m gpu -p no:cacheprovider > gpurun_out/r2f_tests_full.log 2>&1; tail -12 gpurun_out/r2f_tests_full.log > gpurun_out/r2f_tests.log
export TLT_GEMM_AUTOTUNE_CACHE=$PWD/gpurun_out/r2f_autotune.txt; rm -f $TLT_GEMM_AUTOTUNE_CACHE
timeout 1800 python bench.py > gpurun_out/r2f_bench.json 2> gpurun_out/r2f_bench.err
# profile steps of the same shapes with the bench's autotuned plans (bucket rows + rollouts covered them)
timeout 600 python tools/profile_step.py --b 1 --ar 1 --sd 2 --strategy 6,8,64 --prompt 512 --ctx 1200 > /dev/null 2>&1
timeout 600 python tools/profile_step.py --b 8 --ar 1 --sd 2 --strategy 6,8,32 --prompt 512 --ctx 1200 > /dev/null 2>&1
timeout 600 python tools/profile_step.py --b 32 --ar 1 --sd 2 --strategy 6,8,16 --prompt 512 --ctx 1200 > /dev/null 2>&1
ll() {  # name -- profile_step args
  local name=$1; shift
  timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file "gpurun_out/r2f_launches_$name.csv" \
    python tools/profile_step.py "$@" > "gpurun_out/r2f_launches_$name.log" 2>&1
}
ll sd_b1 --b 1 --ar 1 --sd 2 --strategy 6,8,64 --prompt 512 --ctx 1200
ll sd_b8 --b 8 --ar 1 --sd 2 --strategy 6,8,32 --prompt 512 --ctx 1200
ll sd_b32 --b 32 --ar 1 --sd 2 --strategy 6,8,16 --prompt 512 --ctx 1200
timeout 600 ncu --set full --clock-control none --import-source on -k "regex:k_gemm" -s 1 -c 1 \
  -o gpurun_out/r2f_ncu_gemm_m527 -f python tools/one_gemm.py 527 3584 37888 3 > gpurun_out/r2f_ncu_gemm.log 2>&1
timeout 420 ncu --set full --clock-control none --import-source on -k "regex:attention" -s 20 -c 1 \
  -o gpurun_out/r2f_ncu_attn_tree_b31 -f python tools/probe_attn.py 31:700:17 > gpurun_out/r2f_ncu_attn.log 2>&1
