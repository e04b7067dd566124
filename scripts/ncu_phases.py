"""Per-source-range instruction / stall shares of one kernel in an ncu report (dev tool).

usage: python scripts/ncu_phases.py x.ncu-rep file.cu name:a-b [name:a-b ...]
Line ranges are half-open [a, b) in `file.cu`; other files/lines are grouped
per file.
"""
import csv
import io
import subprocess
import sys


def fl(x):
    try:
        return float(x)
    except ValueError:
        return 0.0


rep, fname = sys.argv[1], sys.argv[2]
groups = []
for g in sys.argv[3:]:
    n, r = g.split(":")
    a, b = r.split("-")
    groups.append((n, int(a), int(b)))
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "cuda,sass"],
                     capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(out)))
hdr, f, recs = None, "?", []
for r in rows:
    if r and r[0] == "File Path":
        f = r[1].rsplit("/", 1)[-1]
    elif r and r[0] == "Line No":
        hdr = r
    elif hdr and r and r[0].isdigit():
        recs.append((f, int(r[0]), fl(r[hdr.index("Instructions Executed")]),
                     fl(r[hdr.index("Warp Stall Sampling (All Samples)")])))
ti = sum(x[2] for x in recs) or 1
ts = sum(x[3] for x in recs) or 1
agg = {}
for f, ln, i, s in recs:
    g = "other:" + f
    if f == fname:
        g = "other:" + f
        for n, a, b in groups:
            if a <= ln < b:
                g = n
    agg.setdefault(g, [0.0, 0.0])
    agg[g][0] += i
    agg[g][1] += s
print(f"total warp instructions {ti:.3e}")
for g, (i, s) in sorted(agg.items(), key=lambda x: -x[1][1]):
    print(f"  {g:36s} inst {100*i/ti:5.1f}%  stall samples {100*s/ts:5.1f}%")
