"""Summarise an ncu --metrics gpu__time_duration.sum --csv launch list per kernel (dev helper).

python tools/launch_summary.py launches.csv "header line" > profiles/rNN_launches_summary.txt
"""
import collections
import csv
import sys

path, header = sys.argv[1], sys.argv[2] if len(sys.argv) > 2 else ""
rows = [r for r in csv.reader(l for l in open(path) if not l.startswith("=="))]
hdr, rows = rows[0], rows[1:]
ki, vi, ui = hdr.index("Kernel Name"), hdr.index("Metric Value"), hdr.index("Metric Unit")
agg, cnt = collections.defaultdict(float), collections.Counter()
units = set()
for r in rows:
    name = r[ki].split("(")[0] if not r[ki].startswith("void") else r[ki].split("(")[0]
    name = name[:70]
    agg[name] += float(r[vi].replace(",", ""))
    cnt[name] += 1
    units.add(r[ui])
total = sum(agg.values())
if header:
    print(header)
print(f"unit {units}")
for k, v in sorted(agg.items(), key=lambda kv: -kv[1]):
    print(f"  {v / 1e3:8.3f} us  {100 * v / total:5.1f}%  x {cnt[k]:2d}  {k}")
print(f"total {total / 1e6:.3f} ms over {len(rows)} launches")
