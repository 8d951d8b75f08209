"""Aggregate TLT_TRACE step lines of a bench rollout: device time by mode and batch bucket."""
import collections
import re
import sys

agg = collections.defaultdict(lambda: [0, 0.0, 0, 0])  # steps, ms, tokens(emitted approx), rows
for line in open(sys.argv[1]):
    m = re.match(r"\[tlt\] sd_ms ([\d.]+) b=(\d+) D=(\d+) k=(\d+) T=(\d+) acc=(\d+)", line)
    if m:
        ms, b, D, k, T, acc = float(m[1]), int(m[2]), int(m[3]), int(m[4]), int(m[5]), int(m[6])
        bucket = 1 if b == 1 else 2 if b < 8 else 8 if b < 16 else 16
        key = f"SD bucket>={bucket:2d} ({D},{k},{T})"
        a = agg[key]
        a[0] += 1; a[1] += ms; a[2] += acc + b; a[3] += b
        continue
    m = re.match(r"\[tlt\] prefill_ms ([\d.]+) n=(\d+)", line)
    if m:
        a = agg["prefill"]
        a[0] += 1; a[1] += float(m[1]); a[3] += int(m[2])
        continue
    m = re.match(r"\[tlt\] ar_ms ([\d.]+) b=(\d+)", line)
    if m:
        ms, b = float(m[1]), int(m[2])
        key = "AR b>=48" if b >= 48 else "AR b>=32" if b >= 32 else f"AR b<32"
        a = agg[key]
        a[0] += 1; a[1] += ms; a[2] += b; a[3] += b
tot = sum(a[1] for a in agg.values())
for k, (n, ms, tok, rows) in sorted(agg.items()):
    print(f"{k:32s} steps={n:5d} ms={ms:9.1f} ({100 * ms / tot:4.1f}%) ms/step={ms / max(n, 1):6.2f} tok/s={1e3 * tok / ms:8.0f}")
print(f"total device ms {tot:.1f}")
