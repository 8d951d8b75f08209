#!/bin/bash
# A/B of an environment knob on the bench (the recipe behind the profiles/r2_*_ab*.txt
# and r2_pdl_all_vs_gemm.txt style comparisons):
#   bash tools/gpu_ab_bench.sh TLT_PDL "1 gemm" 3 > gpurun_out/ab.log
# prints per run: value, e2e, AR baseline, SD/AR speedup, clocks, per-bucket step times.
var=$1; vals=$2; runs=${3:-1}
mkdir -p gpurun_out
for r in $(seq "$runs"); do for v in $vals; do
  echo "== $var=$v run $r"
  env "$var=$v" timeout 900 python bench.py --steps 2 --warmup 3 > "gpurun_out/ab_${v}_$r.json" 2> "gpurun_out/ab_${v}_$r.err"
  echo "rc=$?"
  python - "gpurun_out/ab_${v}_$r.json" <<'PY'
import json, sys
d = json.loads(open(sys.argv[1]).read().strip().splitlines()[-1])
print(d["value"], d["e2e"]["value"], d["mean_accept_len"], d["ar_baseline"]["value"], d["ar_baseline"]["speedup"], d["clocks"])
for b in d["per_bucket"]:
    print(b["b"], b["ar_ms_per_step"], [(a["strategy"], a["ms_per_step"]) for a in b["arms"]])
PY
done; done
