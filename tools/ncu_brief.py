"""Print the key metrics of an ncu --set full report (details page)."""
import csv
import subprocess
import sys

KEYS = ["Duration", "Elapsed Cycles", "DRAM Throughput", "Memory Throughput", "Compute (SM) Throughput",
        "Registers Per Thread", "Achieved Occupancy", "Theoretical Occupancy", "Waves Per SM", "L2 Hit Rate",
        "Dynamic Shared Memory Per Block", "Grid Size", "Cluster Size", "Block Limit Shared Mem", "Block Limit Registers",
        "Issue Slots Busy", "Executed Ipc Active", "Max Bandwidth", "L1/TEX Hit Rate", "Mem Busy", "SM Busy",
        "One or More Eligible", "No Eligible"]


def main(path):
    out = subprocess.run(["ncu", "-i", path, "--page", "details", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(out.splitlines()))
    hdr = rows[0]
    ki, si, ni, ui, vi = (hdr.index(x) for x in ("Kernel Name", "Section Name", "Metric Name", "Metric Unit",
                                                  "Metric Value"))
    seen = set()
    for r in rows[1:]:
        if len(r) <= vi:
            continue
        if any(k == r[ni] or r[ni].startswith(k) for k in KEYS) and (r[si], r[ni]) not in seen:
            seen.add((r[si], r[ni]))
            print(f"{r[si][:28]:28s} | {r[ni]:40s} {r[vi]:>14s} {r[ui]}")
    print("kernel:", rows[1][ki][:120])


if __name__ == "__main__":
    main(sys.argv[1])
