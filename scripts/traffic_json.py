"""Per-launch DRAM traffic of the score and select kernels over one full step
-> profiles/traffic.json (read by bench.py for roofline.traffic).

usage: python scripts/traffic_json.py gpurun_out/traffic.csv c3
The csv is `ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,
dram__bytes_write.sum --csv -k regex:'score_tc_kernel|select_kernel' -c 256`
over `bench.py --profile-only --steps 1 --warmup 1` (the first 256 matching
launches = one whole step: every query chunk's score + select).
"""
import csv
import json
import os
import sys
from collections import defaultdict

path, workload = sys.argv[1], sys.argv[2]
rows = [r for r in csv.reader(open(path)) if len(r) > 10]
hdr = rows[0]
ki, mi, vi, ii = (hdr.index(x) for x in ("Kernel Name", "Metric Name", "Metric Value", "ID"))
per = defaultdict(lambda: defaultdict(dict))
for r in rows[1:]:
    name = "score" if "score_tc_kernel" in r[ki] else ("select" if "select_kernel" in r[ki] else None)
    if name:
        per[name][int(r[ii])][r[mi]] = float(r[vi].replace(",", ""))
out_path = os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "profiles", "traffic.json")
data = json.load(open(out_path)) if os.path.exists(out_path) else {}
entry = {"source": f"ncu --metrics dram__bytes_read.sum,dram__bytes_write.sum over one full {workload} step "
                   "(every chunk's launch; --clock-control none)"}
for name, launches in per.items():
    n = len(launches)
    rd = sum(v.get("dram__bytes_read.sum", 0.0) for v in launches.values()) / n
    wr = sum(v.get("dram__bytes_write.sum", 0.0) for v in launches.values()) / n
    entry[f"{name}_dram_bytes_per_launch"] = rd + wr
    entry[f"{name}_dram_read_per_launch"] = rd
    entry[f"{name}_dram_write_per_launch"] = wr
    entry[f"{name}_launches"] = n
data[workload] = entry
json.dump(data, open(out_path, "w"), indent=1)
print(json.dumps(entry, indent=1))
