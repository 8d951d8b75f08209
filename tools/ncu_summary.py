"""Summarise an ncu --metrics gpu__time_duration.sum launch list (CSV)."""
import csv
import sys
from collections import OrderedDict, defaultdict


def load(path):
    rows = []
    with open(path) as f:
        lines = [l for l in f if not l.startswith("==")]
    for r in csv.DictReader(lines):
        if r.get("Metric Name") != "gpu__time_duration.sum":
            continue
        v = float(r["Metric Value"].replace(",", ""))
        unit = r.get("Metric Unit", "nsecond")
        scale = {"nsecond": 1e-3, "usecond": 1.0, "msecond": 1e3}.get(unit, 1e-3)
        rows.append((int(r["ID"]), r["Kernel Name"], v * scale))
    return rows


def short(name):
    n = name.split("(")[0]
    return n.replace("void ", "").replace("tlt::", "")


def summarize(rows, lo, hi, title):
    agg = defaultdict(lambda: [0, 0.0])
    for _, n, us in rows[lo:hi]:
        a = agg[short(n)]
        a[0] += 1
        a[1] += us
    tot = sum(a[1] for a in agg.values())
    print(f"== {title}: {hi - lo} launches, {tot:.1f} us total (serialised, cold)")
    for n, (c, us) in sorted(agg.items(), key=lambda kv: -kv[1][1]):
        print(f"  {us:9.1f} us {100 * us / tot:5.1f}%  x{c:4d}  {n}")


if __name__ == "__main__":
    rows = load(sys.argv[1])
    spans = [tuple(int(x) for x in s.split(":")) for s in sys.argv[2:]] or [(0, len(rows))]
    for lo, hi in spans:
        summarize(rows, lo if lo >= 0 else len(rows) + lo, hi if hi > 0 else len(rows), f"[{lo}:{hi}]")
