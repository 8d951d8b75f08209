#!/bin/bash
# shared-memory carveout A/B: attention probes and the bench
mkdir -p gpurun_out
{
for c in 0 1; do
echo "== TLT_SMEM_CARVEOUT=$c probes"
TLT_SMEM_CARVEOUT=$c timeout 300 python tools/probe_attn.py 1:256:1 1:1024:1 8:1024:1 64:1024:1 1:700:65 5:700:49 31:700:17 2>&1 | grep b=
done
for c in 1 0; do
echo "== TLT_SMEM_CARVEOUT=$c bench"
TLT_SMEM_CARVEOUT=$c timeout 900 python bench.py --steps 2 --warmup 3 > gpurun_out/r2_t40_bench_c$c.json 2>gpurun_out/r2_t40_bench_c$c.err
python - <<PY
import json
d=json.loads(open("gpurun_out/r2_t40_bench_c$c.json").read().strip().splitlines()[-1])
print(d["value"], d["e2e"]["value"], d["ar_baseline"].get("value"), d["clocks"])
for r in d["per_bucket"]: print(r["b"], r["ar_ms_per_step"], [(a["strategy"], a["ms_per_step"]) for a in r["arms"]])
PY
done
} > gpurun_out/r2_t40.log 2>&1
