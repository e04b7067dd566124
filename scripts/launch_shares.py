"""Kernel time shares from an ncu launch list (--metrics gpu__time_duration.sum --csv).

usage: python scripts/launch_shares.py gpurun_out/launches.csv
ncu per-launch times are cold-cache and serialised: compare SHARES with the
bench's event-timed kernels_ms_per_step, not absolute step time.
"""
import csv
import sys
from collections import defaultdict

rows = [r for r in csv.reader(open(sys.argv[1])) if len(r) > 10]
hdr = rows[0]
ki, vi, ii = hdr.index("Kernel Name"), hdr.index("Metric Value"), hdr.index("ID")
STEP = ("score_tc", "score_exact", "select", "merge", "finalize", "fill_sentinel", "bool_mask", "tau_kernel")
launches = [(int(r[ii]), r[ki].split("(")[0].replace("<unnamed>::", ""), float(r[vi].replace(",", "")))
            for r in rows[1:] if r[hdr.index("Metric Name")] == "gpu__time_duration.sum"]
# the indexer step's kernels only (input generation / setup launches are not part of a step)
launches = [x for x in launches if any(t in x[1] for t in STEP)]
tot = defaultdict(float)
cnt = defaultdict(int)
for _, n, t in launches:
    tot[n] += t
    cnt[n] += 1
s = sum(tot.values())
print(f"{len(launches)} step launches (all steps of the run): {s/1e6:.2f} ms under ncu")
for n in sorted(tot, key=lambda n: -tot[n]):
    print(f"  {n:40s} n={cnt[n]:4d}  {tot[n]/1e6:8.2f} ms  {100*tot[n]/s:5.1f}%")
