"""Summarise an ncu --metrics gpu__time_duration.sum --csv launch list:
    python scripts/launch_summary.py gpurun_out/X_launches.csv > profiles/rNN_launches_summary.txt"""
import csv
import sys
from collections import defaultdict

rows = [r for r in csv.reader(open(sys.argv[1])) if r and not r[0].startswith("==")]
hdr = rows[0]
ki, mi, vi = hdr.index("Kernel Name"), hdr.index("Metric Name"), hdr.index("Metric Value")
ui = hdr.index("Metric Unit")
tot = defaultdict(float)
cnt = defaultdict(int)
for r in rows[1:]:
    if len(r) < len(hdr) or r[mi] != "gpu__time_duration.sum":
        continue
    v = float(r[vi].replace(",", ""))
    v *= {"ns": 1e-3, "us": 1.0, "usecond": 1.0, "ms": 1e3, "msecond": 1e3}.get(r[ui], 1e-3)
    name = r[ki].split("(")[0][:70]
    tot[name] += v
    cnt[name] += 1
all_us = sum(tot.values())
print("# ncu --metrics gpu__time_duration.sum --clock-control none launch list (cold-cache, serialised; compare shares)")
print("# kernel | launches | total us | share")
for name in sorted(tot, key=lambda n: -tot[n]):
    print(f"{name:72s} {cnt[name]:6d} {tot[name]:11.1f} {100 * tot[name] / all_us:6.2f}%")
