#!/bin/bash
# variant 8 fix + batched combine loads: GEMM/attention tests, probes, bench
mkdir -p gpurun_out
{
timeout 900 python -m pytest tests/test_gpu_gemm.py tests/test_gpu_attention.py -q -x -p no:cacheprovider 2>&1 | tail -3
timeout 300 python tools/probe_attn.py 1:256:1 1:1024:1 8:1024:1 64:1024:1 1:700:65 5:700:49 31:700:17 2>&1 | grep b=
echo "== bench"
timeout 900 python bench.py --steps 2 --warmup 3 > gpurun_out/r2_t45_bench.json 2>gpurun_out/r2_t45_bench.err
python - <<PY
import json
d=json.loads(open("gpurun_out/r2_t45_bench.json").read().strip().splitlines()[-1])
print(d["value"], d["e2e"]["value"], d["ar_baseline"]["value"], d["ar_baseline"]["speedup"], d["clocks"])
for r in d["per_bucket"]: print(r["b"], r["ar_ms_per_step"], [(a["strategy"], a["ms_per_step"]) for a in r["arms"]])
PY
} > gpurun_out/r2_t45.log 2>&1
