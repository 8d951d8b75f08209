#!/bin/bash
# one-wave deep-ring weight-streaming GEMM plans (TLT_GEMM_ONE_WAVE) A/B
mkdir -p gpurun_out
{
TLT_GEMM_ONE_WAVE=1 timeout 900 python -m pytest tests/test_gpu_gemm.py tests/test_gpu_graph_pool.py -q -x -p no:cacheprovider 2>&1 | tail -2
for r in 1 2; do for ow in 1 0; do
echo "== TLT_GEMM_ONE_WAVE=$ow bench run $r"
TLT_GEMM_ONE_WAVE=$ow timeout 900 python bench.py --steps 2 --warmup 3 > gpurun_out/r2_t47_bench_${ow}_$r.json 2>gpurun_out/r2_t47_bench_${ow}_$r.err
python - <<PY
import json
d=json.loads(open("gpurun_out/r2_t47_bench_${ow}_$r.json").read().strip().splitlines()[-1])
print(d["value"], d["e2e"]["value"], d["ar_baseline"]["value"], d["ar_baseline"]["speedup"], d["clocks"])
print("M17", d["roofline"]["frac"], [(x["site"][:6], x["avg_launch_us"]) for x in d["roofline"]["sites"]])
for r in d["per_bucket"]: print(r["b"], r["ar_ms_per_step"], [(a["strategy"], a["ms_per_step"]) for a in r["arms"]])
PY
done; done
} > gpurun_out/r2_t47.log 2>&1
