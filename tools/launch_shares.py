"""Per-kernel shares of a `ncu --metrics gpu__time_duration.sum --csv` launch list.
usage: python tools/launch_shares.py launches.csv [title] > profiles/xxx.csv"""
import collections
import csv
import sys

path = sys.argv[1]
title = sys.argv[2] if len(sys.argv) > 2 else path
import re
import subprocess
import os
# kernels of libpsdproj.so, by base name (ncu may print names with or without namespaces)
_LIB = os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))),
                    "paper_2410_19208_b200", "libpsdproj.so")
_sass = subprocess.run(["cuobjdump", "-sass", _LIB], capture_output=True, text=True).stdout
_mangled = [ln.split()[-1] for ln in _sass.splitlines() if "Function :" in ln]
_dem = subprocess.run(["c++filt"], input="\n".join(_mangled), capture_output=True, text=True).stdout.split("\n")
OURS = {re.sub(r"<.*", "", d.split("(")[0].replace("void ", "")).split("::")[-1] for d in _dem if d} - {""}


def base(name):
    return re.sub(r"<.*", "", name.split("(")[0].replace("void ", "")).split("::")[-1]


# n×n symmetrize launches belong to the seeded workload generators (workloads.c3_device), not the projection
EXCLUDE = ("symmetrize_kernel",)
with open(path) as f:
    lines = [l for l in f if l.startswith('"')]
agg = collections.OrderedDict()
tot = 0.0
n = 0
for r in csv.DictReader(lines):
    if r.get("Metric Name") != "gpu__time_duration.sum":
        continue
    v = float(r["Metric Value"].replace(",", ""))
    unit = r.get("Metric Unit", "ns")
    ms = v * {"nsecond": 1e-6, "ns": 1e-6, "usecond": 1e-3, "us": 1e-3, "msecond": 1.0, "ms": 1.0}.get(unit, 1e-6)
    name = base(r["Kernel Name"])
    if name not in OURS or name in EXCLUDE:
        continue
    a = agg.setdefault(name, [0.0, 0])
    a[0] += ms
    a[1] += 1
    tot += ms
    n += 1
print(f"# {title}")
print(f"# total device time {tot:.2f} ms over {n} launches (serialised, cold-cache per launch)")
print("share_pct,ms_total,launches,us_avg,kernel")
for k, (ms, c) in sorted(agg.items(), key=lambda kv: -kv[1][0]):
    print(f"{100 * ms / tot:.1f},{ms:.3f},{c},{1000 * ms / c:.1f},{k}")
