#!/bin/bash
# fused top-k LM-head epilogue (extraction rounds + running bound): parity, timing, bench A/B
mkdir -p gpurun_out
{
timeout 900 python -m pytest tests/test_gpu_topk.py -q -x -p no:cacheprovider 2>&1 | tail -3
timeout 300 python tools/time_lm_topk.py 2>&1 | tail -6
echo "== bench fused top-8"
TLT_FUSED_TOPK_K=8 timeout 900 python bench.py --steps 2 --warmup 3 > gpurun_out/r2_t43_bench_f8.json 2>gpurun_out/r2_t43_bench_f8.err
python - <<PY
import json
d=json.loads(open("gpurun_out/r2_t43_bench_f8.json").read().strip().splitlines()[-1])
print(d["value"], d["e2e"]["value"], d["ar_baseline"], d["clocks"])
for r in d["per_bucket"]: print(r["b"], r["ar_ms_per_step"], [(a["strategy"], a["ms_per_step"]) for a in r["arms"]])
PY
} > gpurun_out/r2_t43.log 2>&1
