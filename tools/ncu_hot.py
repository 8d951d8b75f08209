"""Top SASS instructions by warp-stall samples from an ncu report's source page."""
import csv
import subprocess
import sys


def main(path, n=25):
    out = subprocess.run(["ncu", "-i", path, "--page", "source", "--csv", "--print-source", "sass"],
                         capture_output=True, text=True).stdout
    lines = out.splitlines()
    start = next(i for i, l in enumerate(lines) if l.startswith('"Address"'))
    rows = list(csv.reader(lines[start:]))
    h = rows[0]
    ai, si, ci = h.index("Address"), h.index("Source"), h.index("Warp Stall Sampling (All Samples)")
    data = [(int(r[ci] or 0), r[ai], r[si].strip()) for r in rows[1:] if len(r) > ci]
    tot = sum(d[0] for d in data) or 1
    for c, a, s in sorted(data, reverse=True)[:n]:
        print(f"{100 * c / tot:5.1f}%  {a[-5:]}  {s[:90]}")


if __name__ == "__main__":
    main(sys.argv[1], int(sys.argv[2]) if len(sys.argv) > 2 else 25)
