"""Summarise an ncu report (one kernel launch) into a small markdown block.

usage: python scripts/ncu_summary.py gpurun_out/x.ncu-rep [title]
Reads the raw page via `ncu -i ... --page raw --csv` (works without a GPU).
"""
import csv
import io
import subprocess
import sys

KEYS = [
    ("gpu__time_duration.sum", "duration"),
    ("sm__cycles_elapsed.avg", "SM cycles elapsed"),
    ("sm__cycles_active.avg", "SM cycles active"),
    ("sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_active", "tensor pipe active (% of active cycles)"),
    ("sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_elapsed", "tensor pipe active (% of elapsed)"),
    ("sm__inst_executed_pipe_alu.avg.pct_of_peak_sustained_active", "ALU pipe (% active)"),
    ("sm__inst_executed_pipe_fma.avg.pct_of_peak_sustained_active", "FMA pipe (% active)"),
    ("sm__inst_executed_pipe_lsu.avg.pct_of_peak_sustained_active", "LSU pipe (% active)"),
    ("smsp__issue_active.avg.pct_of_peak_sustained_active", "issue slots busy (%)"),
    ("dram__bytes_read.sum", "DRAM read"),
    ("dram__bytes_write.sum", "DRAM write"),
    ("dram__bytes_read.sum.per_second", "DRAM read BW"),
    ("dram__bytes_write.sum.per_second", "DRAM write BW"),
    ("lts__t_sector_hit_rate.pct", "L2 hit rate (%)"),
    ("sm__warps_active.avg.pct_of_peak_sustained_active", "achieved occupancy (%)"),
    ("launch__registers_per_thread", "registers/thread"),
    ("launch__grid_size", "grid"),
    ("launch__block_size", "block"),
    ("smsp__inst_executed.sum", "warp instructions"),
]


def main():
    path = sys.argv[1]
    title = sys.argv[2] if len(sys.argv) > 2 else path
    raw = subprocess.run(["ncu", "-i", path, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(raw)))
    hdr, units, vals = rows[0], rows[1], rows[2]
    d = {h: (u, v) for h, u, v in zip(hdr, units, vals)}
    name = d.get("Kernel Name", ("", "?"))[1]
    print(f"### {title}\n\nkernel: `{name}`\n\n| metric | value |\n|---|---|")
    for key, label in KEYS:
        if key in d:
            u, v = d[key]
            print(f"| {label} (`{key}`) | {v} {u} |")
    stalls = {k: float(v[1] or 0) for k, v in d.items()
              if k.startswith("smsp__pcsamp_warps_issue_stalled") and not k.endswith("not_issued")}
    tot = sum(stalls.values()) or 1.0
    top = sorted(stalls.items(), key=lambda kv: -kv[1])[:6]
    print("\nwarp-stall samples (top): " + ", ".join(f"{k.split('stalled_')[1]} {v / tot * 100:.0f}%" for k, v in top))


if __name__ == "__main__":
    main()
