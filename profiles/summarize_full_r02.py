#!/usr/bin/env python3
"""Key metrics of an `ncu --set full` report (profiles/run_ncu_r02.sh step 2): time,
DRAM bytes and achieved bandwidth against the measured copy peak, issue / warp
activity, registers, and the top-3 warp stall reasons (cycles per issued instruction).
usage: summarize_full_r02.py gpurun_out/prof_r02.ncu-rep|ncu_raw_r02.csv.gz [hbm_gbs] > profiles/ncu_full_r02.md"""
import csv
import io
import re
import subprocess
import sys

rep = sys.argv[1]
def _measured_peak():
    import json
    import os
    p = os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "MEASURED_PEAKS.json")
    try:
        return float(json.load(open(p))["hbm_gbs"])
    except Exception:
        return 6540.5  # round-1 pool's measured copy bandwidth


peak = float(sys.argv[2]) if len(sys.argv) > 2 else _measured_peak()
if rep.endswith(".csv.gz"):  # the raw page exported on the box (run_ncu_r02.sh)
    import gzip

    raw = gzip.open(rep, "rt").read()
else:
    raw = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True,
                         text=True, check=True).stdout
rows = list(csv.reader(io.StringIO(raw)))
h, units, data = rows[0], rows[1], rows[2:]


def val(r, key, scale=1.0):
    if key not in h:
        return None
    s = r[h.index(key)].replace(",", "")
    try:
        x = float(s)
    except ValueError:
        return None
    u = units[h.index(key)]
    mult = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "nsecond": 1e-9,
            "usecond": 1e-6, "msecond": 1e-3, "second": 1.0, "ns": 1e-9, "us": 1e-6,
            "ms": 1e-3, "s": 1.0}.get(u, 1.0)
    return x * mult * scale


stall_keys = [k for k in h if re.fullmatch(
    r"smsp__average_warps_issue_stalled_(.+)_per_issue_active\.ratio", k)]
print(f"# ncu --set full: {rep.split('/')[-1]} (peak {peak} GB/s = MEASURED_PEAKS.json)\n")
print("| kernel | time | DRAM R+W | achieved GB/s | of peak | issue active % | "
      "warps active % | regs | grid | top stalls (cycles / issue) |")
print("|---|---:|---:|---:|---:|---:|---:|---:|---:|---|")
for r in data:
    name = r[h.index("Kernel Name")].split("(")[0].replace("void ", "")
    name = re.sub(r"mco::|<unnamed>::|unnamed>::", "", name)[:90]
    t = val(r, "gpu__time_duration.sum")
    rd, wr = val(r, "dram__bytes_read.sum") or 0, val(r, "dram__bytes_write.sum") or 0
    gbs = (rd + wr) / t / 1e9 if t else 0
    stalls = sorted(((val(r, k) or 0, re.sub(r"smsp__average_warps_issue_stalled_|"
                                             r"_per_issue_active\.ratio", "", k))
                     for k in stall_keys), reverse=True)[:3]
    st = ", ".join(f"{n} {v:.2f}" for v, n in stalls if v > 0)
    ia = val(r, "smsp__issue_active.avg.pct_of_peak_sustained_active")
    wa = val(r, "sm__warps_active.avg.pct_of_peak_sustained_active")
    regs = r[h.index("launch__registers_per_thread")] if "launch__registers_per_thread" in h else "-"
    grid = r[h.index("launch__grid_size")] if "launch__grid_size" in h else "-"
    print(f"| `{name}` | {t * 1e6:.1f} us | {(rd + wr) / 1e9:.3f} GB | {gbs:.0f} | "
          f"{gbs / peak:.3f} | {ia:.1f} | {wa:.1f} | {regs} | {grid} | {st} |")
