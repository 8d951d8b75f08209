"""profiles/r2_traffic.json from the ncu DRAM-traffic launch lists of
tools/gpu_r2_s3_final.sh: mean dram__bytes_read + dram__bytes_write per
launch of each engine GEMM site (key 'probe kind:M', as bench.py PROBES)."""
import csv
import glob
import json
import os
import sys
from collections import defaultdict

src = sys.argv[1] if len(sys.argv) > 1 else "gpurun_out"
out = {"_comment": "dram__bytes_read.sum + dram__bytes_write.sum per launch (bytes), mean of 3 launches of the "
                   "engine's own GEMM site (tools/probe.py under ncu, successive layers' weights, eager warm-up "
                   "pass; tools/gpu_r2_s3_final.sh); key = 'probe kind:M'"}
for path in sorted(glob.glob(os.path.join(src, "fin_traffic_*.csv"))):
    key = os.path.basename(path)[len("fin_traffic_"):-4].replace("_", ":")
    with open(path) as f:
        rows = list(csv.DictReader([l for l in f if not l.startswith("==")]))
    per = defaultdict(float)
    scale = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "KB": 1e3, "MB": 1e6, "GB": 1e9}
    for r in rows:
        if r["Metric Name"] in ("dram__bytes_read.sum", "dram__bytes_write.sum"):
            per[r["ID"]] += float(r["Metric Value"].replace(",", "")) * scale.get(r["Metric Unit"], 1)
    if per:
        out[key] = int(sum(per.values()) / len(per))
json.dump(out, open("profiles/r2_traffic.json", "w"), indent=1)
print(json.dumps(out, indent=1))
