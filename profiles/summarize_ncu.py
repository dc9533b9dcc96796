#!/usr/bin/env python3
"""Summarise an ncu launch list (profiles/run_ncu.sh step 1) of `bench.py`:
per-kernel device time share and DRAM bytes per parameter, and write
profiles/traffic.json (dram__bytes_read.sum + dram__bytes_write.sum per
parameter per optimizer step) that bench.py reports as roofline.traffic.

usage: summarize_ncu.py gpurun_out/launches_rNN.csv NPARAMS > profiles/launches_rNN.md
"""
import collections
import csv
import json
import os
import re
import sys

UNIT = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "ns": 1e-9, "nsecond": 1e-9,
        "us": 1e-6, "usecond": 1e-6, "ms": 1e-3, "msecond": 1e-3}
KIND_OF = [("flat_tma_kernel<0,", "adamw"), ("flat_tma_kernel<1,", "lion"),
           ("flat_tma_kernel<2,", "adan"), ("flat_tma_kernel<3,", "sophia"),
           ("flat_step_kernel<0,", "adamw"), ("flat_step_kernel<1,", "lion"),
           ("flat_step_kernel<2,", "adan"), ("flat_step_kernel<3,", "sophia"),
           ("lomo_kernel", "lomo"), ("lomo_tma_kernel", "lomo"), ("sumsq_kernel", "lomo"),
           ("k1_stats", "adalomo"), ("kr_stats", "adalomo"), ("k2_scalars", "adalomo"),
           ("k3_moments", "adalomo"), ("k4_usq", "adalomo"), ("k5_damp", "adalomo"),
           ("k6_update", "adalomo")]


def main(path, nparams):
    rows = list(csv.reader(open(path)))
    hi = next(i for i, r in enumerate(rows) if "Kernel Name" in r)
    h = rows[hi]
    ki, mi, vi, ui, ii = (h.index(x) for x in ("Kernel Name", "Metric Name", "Metric Value",
                                                "Metric Unit", "ID"))
    launches = collections.OrderedDict()
    for r in rows[hi + 1:]:
        d = launches.setdefault(r[ii], {"name": r[ki]})
        d[r[mi]] = float(r[vi].replace(",", "")) * UNIT.get(r[ui], 1.0)
    per_kernel = collections.OrderedDict()
    for d in launches.values():
        name = d["name"].split("(")[0].replace(" ", "")
        a = per_kernel.setdefault(name, {"n": 0, "t": 0.0, "bytes": 0.0, "last_bytes": 0.0,
                                         "last_t": 0.0})
        b = d.get("dram__bytes_read.sum", 0) + d.get("dram__bytes_write.sum", 0)
        a["n"] += 1
        a["t"] += d.get("gpu__time_duration.sum", 0)
        a["bytes"] += b
        a["last_bytes"], a["last_t"] = b, d.get("gpu__time_duration.sum", 0)
    total_t = sum(a["t"] for a in per_kernel.values())
    print(f"# ncu launch list: {os.path.basename(path)}\n")
    print("Cold-cache, serialised per-launch times (compare shares, not absolutes).\n")
    print("| kernel | launches | total ms | share | DRAM B/param (last launch) | GB/s (last) |")
    print("|---|---:|---:|---:|---:|---:|")
    traffic = collections.defaultdict(float)
    for name, a in per_kernel.items():
        bpp = a["last_bytes"] / nparams
        gbs = a["last_bytes"] / a["last_t"] / 1e9 if a["last_t"] else 0
        print(f"| `{name[:70]}` | {a['n']} | {a['t'] * 1e3:.2f} | {a['t'] / total_t:.1%} | "
              f"{bpp:.3f} | {gbs:.0f} |")
        # flat_tma_kernel<TmaCfg<CW,NS>,KIND,MIXED> -> flat_tma_kernel<KIND,
        key = re.sub(r"flat_tma_kernel<.*?TmaCfg<[\d,]+>,", "flat_tma_kernel<",
                     name.replace(" ", ""))
        for pat, kind in KIND_OF:
            if pat in key:
                traffic[kind] += bpp
    out = {k: {"dram_bytes_per_param": round(v, 4), "source": os.path.basename(path)}
           for k, v in traffic.items()}
    with open(os.path.join(os.path.dirname(os.path.abspath(__file__)), "traffic.json"), "w") as f:
        json.dump(out, f, indent=1)
    print("\nDRAM bytes per parameter per optimizer step (sum over that optimizer's kernels):\n")
    for k, v in out.items():
        print(f"- {k}: {v['dram_bytes_per_param']}")


if __name__ == "__main__":
    main(sys.argv[1], int(sys.argv[2]))
