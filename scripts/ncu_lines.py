"""Per-CUDA-source-line instruction / stall totals from an ncu report (dev tool).

usage: python scripts/ncu_lines.py gpurun_out/x.ncu-rep [top]
Uses the `cuda,sass` source view, whose CUDA-line rows carry the metrics
aggregated over that line's SASS (needs -lineinfo and --import-source on).
"""
import csv
import io
import subprocess
import sys

rep = sys.argv[1]
top = int(sys.argv[2]) if len(sys.argv) > 2 else 40
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "cuda,sass"],
                     capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(out)))
fname = "?"
hdr = None
recs = []
for r in rows:
    if r and r[0] == "File Path":
        fname = r[1].rsplit("/", 1)[-1]
    elif r and r[0] == "Line No":
        hdr = r
    elif hdr and r and r[0].isdigit():
        try:
            si = float(r[hdr.index("Warp Stall Sampling (All Samples)")] or 0)
            ii = float(r[hdr.index("Instructions Executed")] or 0)
        except ValueError:
            continue
        recs.append((fname, int(r[0]), r[1].strip()[:90], ii, si))
ti = sum(x[3] for x in recs) or 1
ts = sum(x[4] for x in recs) or 1
print(f"total warp instructions {ti:.3e}, stall samples {ts:.0f}")
for f, ln, s, ii, si in sorted(recs, key=lambda x: -x[4])[:top]:
    print(f"{f}:{ln:<5} inst {100*ii/ti:5.1f}%  samples {100*si/ts:5.1f}%  {s}")
