#!/bin/bash
# A/B of an env knob on the mini rollout bench: VAR, VALS, RUNS
timeout 600 python -m pytest tests -m gpu -x -q 2>&1 | tail -2
for v in $VALS; do for i in $(seq 1 ${RUNS:-3}); do
  env $VAR=$v TLT_TRACE=1 timeout 150 python bench.py --steps 1 --warmup 1 --ar-baseline 0 --cpu-gen 0 > gpurun_out/ab_${v}_$i.json 2> gpurun_out/ab_${v}_$i.err
  echo "$VAR=$v run $i rc=$? $(python -c "import json;d=json.loads(open('gpurun_out/ab_${v}_$i.json').read().strip().splitlines()[-1]);print(d['value'])" 2>&1 | tail -1)"
done; done
