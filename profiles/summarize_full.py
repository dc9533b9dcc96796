#!/usr/bin/env python3
"""Key metrics of an `ncu --set full` report (profiles/run_ncu.sh step 2).
usage: summarize_full.py gpurun_out/prof_rNN.ncu-rep > profiles/ncu_full_rNN.md"""
import csv
import io
import subprocess
import sys

KEYS = [("gpu__time_duration.sum", "time"), ("dram__bytes_read.sum", "DRAM read"),
        ("dram__bytes_write.sum", "DRAM write"),
        ("gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed", "DRAM % of peak"),
        ("smsp__issue_active.avg.pct_of_peak_sustained_active", "issue active %"),
        ("sm__warps_active.avg.pct_of_peak_sustained_active", "warps active %"),
        ("launch__registers_per_thread", "regs"), ("launch__grid_size", "grid"),
        ("launch__occupancy_limit_registers", "CTAs/SM (reg limit)"),
        ("lts__t_sector_hit_rate.pct", "L2 hit %")]

raw = subprocess.run(["ncu", "-i", sys.argv[1], "--page", "raw", "--csv"], capture_output=True,
                     text=True, check=True).stdout
rows = list(csv.reader(io.StringIO(raw)))
h, units, data = rows[0], rows[1], rows[2:]
print(f"# ncu --set full: {sys.argv[1].split('/')[-1]}\n")
print("| kernel | " + " | ".join(k[1] for k in KEYS) + " |")
print("|---|" + "---:|" * len(KEYS))
for r in data:
    name = r[h.index("Kernel Name")].split("(")[0].replace("void ", "")
    cells = []
    for k, _ in KEYS:
        i = h.index(k) if k in h else None
        cells.append(f"{r[i]} {units[i]}".strip() if i is not None else "-")
    print(f"| `{name}` | " + " | ".join(cells) + " |")
