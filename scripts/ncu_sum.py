"""Summarise an ncu --csv metrics dump: mean of each metric per kernel name."""
import csv, sys, collections
rows = list(csv.reader(l for l in open(sys.argv[1]) if l.startswith('"')))
hdr = rows[0]
ki, mi, vi = hdr.index("Kernel Name"), hdr.index("Metric Name"), hdr.index("Metric Value")
acc = collections.defaultdict(list)
for r in rows[1:]:
    name = r[ki].split("(")[0].replace("<unnamed>::", "")[:48]
    try:
        acc[(name, r[mi])].append(float(r[vi].replace(",", "")))
    except ValueError:
        pass
for (name, m), v in sorted(acc.items()):
    print(f"{name:50s} {m:55s} n={len(v):3d} mean={sum(v)/len(v):.4g}")
