#!/bin/bash
# ncu --set full of the decode-phase (HBM / latency bound) kernels of the 7B
# path: flash-decode attention (AR b=32), tree attention (verify b=16), KV
# compaction, tree select, drafter top-k. One GPU, one process per capture.
#   gpurun --timeout 1800 -- 'bash tools/gpu_ncu_decode.sh'
mkdir -p gpurun_out
cap() {  # name kernel-regex skip count -- profile_step args
  local name=$1 re=$2 skip=$3 cnt=$4; shift 4
  timeout 420 ncu --set full --clock-control none --import-source on -k "regex:$re" -s "$skip" -c "$cnt" \
    -o "gpurun_out/$name" -f python tools/profile_step.py "$@" > "gpurun_out/ncu_$name.log" 2>&1
  echo "ncu $name rc=$?"
}
cap attn_dec_b32 'k_attention_dec' 28 1 --b 32 --ar 2 --sd 0 --ctx 1536 --prompt 1024
cap attn_tree_b16 'k_attention_tree' 28 1 --b 16 --ar 0 --sd 2 --strategy 6,8,16 --ctx 1536 --prompt 1024
cap commit_b16 'k_commit$' 0 1 --b 16 --ar 0 --sd 2 --strategy 6,8,16 --ctx 1536 --prompt 1024
cap tree_level_b16 'k_tree_level' 6 1 --b 16 --ar 0 --sd 2 --strategy 6,8,16 --ctx 1536 --prompt 1024
cap row_topk_b16 'k_row_topk_chunk' 6 1 --b 16 --ar 0 --sd 2 --strategy 6,8,16 --ctx 1536 --prompt 1024
ls -la gpurun_out/*.ncu-rep
