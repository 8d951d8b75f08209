#!/bin/bash
mkdir -p gpurun_out
timeout 1800 python -m pytest tests -q -m gpu 2>&1 | tail -15 > gpurun_out/r2_t13.log
timeout 1500 python bench.py --steps 2 --warmup 1 > gpurun_out/r2_bench_v13.json 2> gpurun_out/r2_bench_v13.err
TLT_GEMM_AUTOTUNE=0 timeout 1500 python bench.py --steps 2 --warmup 1 --cpu-rows 0 --bucket-steps 0 > gpurun_out/r2_bench_v13_noat.json 2> gpurun_out/r2_bench_v13_noat.err
cap() {  # name kernel-regex skip count -- probe_attn args
  local name=$1 re=$2 skip=$3 cnt=$4; shift 4
  timeout 420 ncu --set full --clock-control none --import-source on -k "regex:$re" -s "$skip" -c "$cnt" \
    -o "gpurun_out/r2_ncu_$name" -f python tools/probe_attn.py "$@" > "gpurun_out/r2_ncu_$name.log" 2>&1
  echo "ncu $name rc=$?" >> gpurun_out/r2_t13.log
}
cap tma_tree_b31_T16 'attention_tma' 20 1 31:700:17
cap tma_tree_b5_T48 'attention_tma' 20 1 5:700:49
cap tma_dec_b64 'attention_tma' 20 1 64:1024:1
cap tma_dec_b1 'attention_tma' 20 1 1:1024:1
