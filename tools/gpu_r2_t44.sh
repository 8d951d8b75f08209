#!/bin/bash
# token sub-tile GEMM plan (variant 8): parity, timing per variant, bench with the autotuner offered it
mkdir -p gpurun_out
{
timeout 900 python -m pytest tests/test_gpu_gemm.py tests/test_gpu_topk.py -q -x -p no:cacheprovider 2>&1 | tail -3
S="272:3584:37888:3 528:3584:37888:3 1040:3584:37888:3 272:18944:3584:2 528:18944:3584:2 264:3584:4608:1 528:3584:4608:1 528:3584:3584:2 496:3584:152064:0 300:3584:37888:3 400:18944:3584:2"
for v in 0 2 4 8; do echo "== variant $v"; TLT_GEMM_FORCE_VARIANT=$v timeout 300 python tools/time_gemms.py $S 2>&1 | grep M=; done
echo "== bench"
TLT_GEMM_AUTOTUNE_LOG=1 timeout 900 python bench.py --steps 2 --warmup 3 > gpurun_out/r2_t44_bench.json 2>gpurun_out/r2_t44_bench.err
grep autotune gpurun_out/r2_t44_bench.err | sort | uniq | head -60
python - <<PY
import json
d=json.loads(open("gpurun_out/r2_t44_bench.json").read().strip().splitlines()[-1])
print(d["value"], d["e2e"]["value"], d["ar_baseline"]["value"], d["ar_baseline"]["speedup"], d["clocks"])
print(d["roofline_tensor_class"]["sites"])
for r in d["per_bucket"]: print(r["b"], r["ar_ms_per_step"], [(a["strategy"], a["ms_per_step"]) for a in r["arms"]])
PY
} > gpurun_out/r2_t44.log 2>&1
