"""Summarise an ncu --csv launch list (gpu__time_duration.sum) per kernel; optional: last N launches."""
import csv
import sys
from collections import OrderedDict

path = sys.argv[1]
tail = int(sys.argv[2]) if len(sys.argv) > 2 else 0
rows = []
with open(path) as f:
    lines = [l for l in f if l.startswith('"')]
for r in csv.DictReader(lines):
    if r.get("Metric Name") != "gpu__time_duration.sum":
        continue
    unit = r["Metric Unit"]
    v = float(r["Metric Value"].replace(",", ""))
    us = v / 1e3 if unit in ("nsecond", "ns") else v if unit in ("usecond", "us") else v * 1e3
    rows.append((r["Kernel Name"].split("(")[0].split("<")[0], us))
if tail:
    rows = rows[-tail:]
agg = OrderedDict()
for name, us in rows:
    a = agg.setdefault(name, [0, 0.0])
    a[0] += 1
    a[1] += us
tot = sum(a[1] for a in agg.values())
print(f"{len(rows)} launches, {tot:.1f} us")
for name, (cnt, us) in sorted(agg.items(), key=lambda kv: -kv[1][1]):
    print(f"{name:32s} {cnt:5d} {us:10.1f} us {us / cnt:8.2f} avg {100 * us / tot:5.1f}%")
