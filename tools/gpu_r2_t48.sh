#!/bin/bash
# e4m3 drafter LM head (TLT_DRAFTER_FP8=1) in the rollout: throughput and acceptance
mkdir -p gpurun_out
{
for fp8 in 1 0; do
echo "== TLT_DRAFTER_FP8=$fp8 bench"
TLT_DRAFTER_FP8=$fp8 timeout 900 python bench.py --steps 2 --warmup 3 > gpurun_out/r2_t48_bench_$fp8.json 2>gpurun_out/r2_t48_bench_$fp8.err
python - <<PY
import json
d=json.loads(open("gpurun_out/r2_t48_bench_$fp8.json").read().strip().splitlines()[-1])
print(d["value"], d["e2e"]["value"], d["mean_accept_len"], d["ar_baseline"]["value"], d["ar_baseline"]["speedup"], d["clocks"])
for r in d["per_bucket"]: print(r["b"], r["ar_ms_per_step"], [(a["strategy"], a["ms_per_step"], a["mean_accept_len"]) for a in r["arms"]])
PY
done
} > gpurun_out/r2_t48.log 2>&1
