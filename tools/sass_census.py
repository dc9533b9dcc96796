#!/usr/bin/env python3
"""Per-kernel SASS instruction census of the built library (cuobjdump -sass): the
instructions that show which data-movement path a kernel uses -- UBLKCP (TMA / bulk
copy, cp.async.bulk), SYNCS (mbarrier), 256-bit LDG / STG, LDGSTS, plus MUFU (rsqrt /
sqrt / rcp), DMUL/DFMA/DADD (fp64 arithmetic), and spills (LDL / STL).
usage: python tools/sass_census.py [lib.so] > profiles/sass_census_r02.md"""
import collections
import re
import subprocess
import sys

lib = sys.argv[1] if len(sys.argv) > 1 else "paper_2312_00407_b200/_build/libmco.so"
out = subprocess.run(["cuobjdump", "-sass", lib], capture_output=True, text=True,
                     check=True).stdout
PATS = collections.OrderedDict([
    ("UBLKCP", r"\bUBLKCP\b"), ("SYNCS", r"\bSYNCS\."), ("LDG.256", r"\bLDG\.[\w.]*\.256\b"),
    ("STG.256", r"\bSTG\.[\w.]*\.256\b"), ("LDG.128", r"\bLDG\.[\w.]*\.128\b"),
    ("STG.128", r"\bSTG\.[\w.]*\.128\b"), ("LDG(any)", r"\bLDG\b"), ("STG(any)", r"\bSTG\b"),
    ("MUFU", r"\bMUFU\."), ("DFMA/DMUL/DADD", r"\bD(FMA|MUL|ADD)\b"),
    ("LDL/STL (spill)", r"\b(LDL|STL)\b"), ("instructions", r"^\s+/\*[0-9a-f]{4}\*/")])
kernels = collections.OrderedDict()
cur = None
for ln in out.splitlines():
    m = re.match(r"\s+Function : (\S+)", ln)
    if m:
        cur = m.group(1)
        kernels[cur] = collections.Counter()
        continue
    if cur is None:
        continue
    for k, p in PATS.items():
        if re.search(p, ln):
            kernels[cur][k] += 1


def demangle(names):
    r = subprocess.run(["c++filt"], input="\n".join(names), capture_output=True, text=True)
    return r.stdout.splitlines()


names = list(kernels)
pretty = demangle(names)
print(f"# SASS census of `{lib}` (cuobjdump -sass, sm_100a)\n")
print("Counts are static instructions per kernel.  UBLKCP + SYNCS = the cp.async.bulk / "
      "mbarrier pipeline; .256 = 256-bit LDG/STG (sm_100a vector width); MUFU = rsqrt / "
      "sqrt / rcp approximations; D* = fp64 arithmetic.\n")
print("| kernel | " + " | ".join(PATS) + " |")
print("|---|" + "---:|" * len(PATS))
keep = re.compile(r"flat|lomo|sumsq|k[1-6r]_|kr2|peer|sophia|synth|list|widen|graph")
for mangled, nm in sorted(zip(names, pretty), key=lambda x: x[1]):
    short = re.sub(r"mco::|\(anonymous namespace\)::", "", nm).split("(")[0][:80]
    if not keep.search(short):
        continue
    c = kernels[mangled]
    print(f"| `{short}` | " + " | ".join(str(c[k]) for k in PATS) + " |")
