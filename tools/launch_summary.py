"""Summarise an ncu `--metrics gpu__time_duration.sum --csv` launch list per kernel.

usage: python tools/launch_summary.py launches.csv "header line" > profiles/....txt
"""
import csv, sys
from collections import defaultdict

rows = [r for r in csv.reader(l for l in open(sys.argv[1]) if not l.startswith("=="))]
hdr = rows[0]
ki, mi, vi = hdr.index("Kernel Name"), hdr.index("Metric Name"), hdr.index("Metric Value")
ui = hdr.index("Metric Unit")
to_us = {"nsecond": 1e-3, "ns": 1e-3, "usecond": 1.0, "us": 1.0, "msecond": 1e3, "ms": 1e3, "second": 1e6, "s": 1e6}
tot, cnt = defaultdict(float), defaultdict(int)
for r in rows[1:]:
    if len(r) <= vi or r[mi] != "gpu__time_duration.sum":
        continue
    tot[r[ki]] += float(r[vi].replace(",", "")) * to_us[r[ui]]
    cnt[r[ki]] += 1
allt = sum(tot.values())
if len(sys.argv) > 2:
    print("# " + sys.argv[2])
print("# cold-cache, serialised per launch: compare SHARES, not absolutes")
print(f"{'kernel':60s} {'launches':>9s} {'total_us':>12s} {'avg_us':>10s} {'share':>7s}")
for k in sorted(tot, key=lambda k: -tot[k]):
    print(f"{k[:60]:60s} {cnt[k]:9d} {tot[k]:12.1f} {tot[k] / cnt[k]:10.2f} {tot[k] / allt:7.3f}")
