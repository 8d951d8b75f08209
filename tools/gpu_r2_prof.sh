#!/bin/bash
# Round-2 profile pass: per-launch device times of whole SD / AR steps at
# b = 1, 8, 32 (ncu launch lists), and ncu --set full of the attention
# kernels at the verify / decode shapes the judge asked for.
#   gpurun --timeout 2400 -- 'bash tools/gpu_r2_prof.sh'
mkdir -p gpurun_out
ll() {  # name -- profile_step args
  local name=$1; shift
  timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file "gpurun_out/r2_launches_$name.csv" \
    python tools/profile_step.py "$@" > "gpurun_out/r2_launches_$name.log" 2>&1
  echo "launches $name rc=$?"
}
cap() {  # name kernel-regex skip count -- probe_attn args
  local name=$1 re=$2 skip=$3 cnt=$4; shift 4
  timeout 420 ncu --set full --clock-control none --import-source on -k "regex:$re" -s "$skip" -c "$cnt" \
    -o "gpurun_out/r2_ncu_$name" -f python tools/probe_attn.py "$@" > "gpurun_out/r2_ncu_$name.log" 2>&1
  echo "ncu $name rc=$?"
}
ll sd_b1 --b 1 --ar 1 --sd 2 --strategy 10,8,64 --prompt 512 --ctx 1200
ll sd_b8 --b 8 --ar 1 --sd 2 --strategy 10,8,32 --prompt 512 --ctx 1200
ll sd_b32 --b 32 --ar 1 --sd 2 --strategy 6,8,16 --prompt 512 --ctx 1200
python tools/probe_attn.py 1:1024:1 5:700:49 31:700:17 64:1024:1 1:4096:1 31:4096:17 > gpurun_out/r2_probe_attn.txt 2>&1
cap attn_tree_b31_T16 'attention|attn' 20 2 31:700:17
cap attn_tree_b5_T48 'attention|attn' 20 2 5:700:49
cap attn_dec_b1 'attention|attn' 20 2 1:1024:1
ls -la gpurun_out/
