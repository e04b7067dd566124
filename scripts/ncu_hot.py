"""Top SASS lines of a kernel by executed instructions and by stall samples,
from `ncu -i rep --page source --csv --print-source sass`."""
import csv, sys
rows = list(csv.reader(open(sys.argv[1])))
hdr_i = next(i for i, r in enumerate(rows) if r and r[0] == "Address")
hdr = rows[hdr_i]
A, S, ST, IE = hdr.index("Address"), hdr.index("Source"), hdr.index("Warp Stall Sampling (All Samples)"), hdr.index("Instructions Executed")
body = [r for r in rows[hdr_i + 1:] if len(r) > IE and r[IE].replace(",", "").isdigit()]
tot_i = sum(int(r[IE]) for r in body)
tot_s = sum(int(r[ST] or 0) for r in body)
n = int(sys.argv[2]) if len(sys.argv) > 2 else 25
print(f"total instr {tot_i}, stall samples {tot_s}")
for key, idx in (("instr", IE), ("stalls", ST)):
    print(f"--- top by {key}")
    for r in sorted(body, key=lambda r: -int(r[idx] or 0))[:n]:
        print(f"{r[A][-5:]} {int(r[IE]):9d} {int(r[ST] or 0):6d}  {r[S].strip()[:90]}")
