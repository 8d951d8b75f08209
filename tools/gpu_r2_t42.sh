#!/bin/bash
# b=1 plain-decode attention: ncu full captures of the attention and combine kernels
mkdir -p gpurun_out
timeout 420 ncu --set full --clock-control none --import-source on -k "regex:k_attention_tma" -s 20 -c 1 \
  -o gpurun_out/r2_ncu_dec_b1 -f python tools/probe_attn.py 1:700:1 > gpurun_out/r2_ncu_dec_b1.log 2>&1
timeout 420 ncu --set full --clock-control none --import-source on -k "regex:k_attn_combine" -s 20 -c 1 \
  -o gpurun_out/r2_ncu_comb_b1 -f python tools/probe_attn.py 1:700:1 > gpurun_out/r2_ncu_comb_b1.log 2>&1
timeout 300 ncu --metrics gpu__time_duration.sum,launch__grid_size --clock-control none --csv --log-file gpurun_out/r2_dec_b1_launches.csv \
  python tools/probe_attn.py 1:700:1 1:256:1 > /dev/null 2>&1
timeout 300 python -m pytest tests/test_gpu_topk.py -q -x -p no:cacheprovider -k "fused and 130" 2>&1 | grep -E "Error|assert|passed|failed" | head -20 > gpurun_out/r2_t42_topk.log
for f in 1 8; do
TLT_FUSED_TOPK_K=$f timeout 600 ncu --metrics gpu__time_duration.sum,launch__grid_size --clock-control none --csv --log-file gpurun_out/r2_t42_sd_b8_f$f.csv \
  python tools/profile_step.py --b 8 --ar 1 --sd 2 --strategy 6,8,32 --prompt 512 --ctx 1200 > /dev/null 2>&1
done
