#!/bin/bash
# tcgen05 tree-attention split target (148 planned CTAs for >= 2 requests) vs the old 296: tests + bench A/B
mkdir -p gpurun_out
timeout 1200 python -m pytest tests/test_gpu_attention.py tests/test_gpu_parity_graphs.py tests/test_gpu_parity_7b.py -q -x -p no:cacheprovider > gpurun_out/asplit_tests.log 2>&1; tail -2 gpurun_out/asplit_tests.log
for v in new 296; do
  echo "== TLT_ATTN_TREE_CTAS=$v"
  if [ $v = new ]; then timeout 900 python bench.py --steps 2 --warmup 3 > gpurun_out/asplit_$v.json 2> gpurun_out/asplit_$v.err
  else TLT_ATTN_TREE_CTAS=$v timeout 900 python bench.py --steps 2 --warmup 3 > gpurun_out/asplit_$v.json 2> gpurun_out/asplit_$v.err; fi
  python - "gpurun_out/asplit_$v.json" <<'PY'
import json, sys
d = json.loads(open(sys.argv[1]).read().strip().splitlines()[-1])
print(d["value"], d["e2e"]["value"], d["mean_accept_len"], d["ar_baseline"]["value"], d["ar_baseline"]["speedup"], d["clocks"])
for b in d["per_bucket"]:
    print(b["b"], b["ar_ms_per_step"], [(a["strategy"], a["ms_per_step"]) for a in b["arms"]])
PY
done
