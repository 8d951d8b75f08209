#!/bin/bash
# PDL on every kernel (TMEM kernels release dependents only after allocating) vs GEMM-only PDL
mkdir -p gpurun_out
{
timeout 600 python -m pytest tests/test_gpu_attention.py -q -x -p no:cacheprovider 2>&1 | tail -2
for pdl in 1 gemm; do
echo "== TLT_PDL=$pdl probes"
TLT_PDL=$pdl timeout 300 python tools/probe_attn.py 1:256:1 1:1024:1 8:1024:1 64:1024:1 1:700:65 5:700:49 31:700:17 2>&1 | grep b=
done
for r in 1 2 3; do for pdl in 1 gemm; do
echo "== TLT_PDL=$pdl bench run $r"
TLT_PDL=$pdl timeout 900 python bench.py --steps 2 --warmup 3 > gpurun_out/r2_t46_bench_${pdl}_$r.json 2>gpurun_out/r2_t46_bench_${pdl}_$r.err
echo "rc=$?"
python - <<PY
import json
d=json.loads(open("gpurun_out/r2_t46_bench_${pdl}_$r.json").read().strip().splitlines()[-1])
print(d["value"], d["e2e"]["value"], d["ar_baseline"]["value"], d["ar_baseline"]["speedup"], d["clocks"])
for r in d["per_bucket"]: print(r["b"], r["ar_ms_per_step"], [(a["strategy"], a["ms_per_step"]) for a in r["arms"]])
PY
done; done
} > gpurun_out/r2_t46.log 2>&1
