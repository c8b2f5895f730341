"""Per-kernel achieved DRAM GB/s of one step from an ncu --metrics
gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --csv launch list (dev helper).

python tools/ncu_gbs.py launches.csv PEAK_GBS "header" > profiles/rNN_kernel_hbm.txt
"""
import collections
import csv
import sys

path, peak = sys.argv[1], float(sys.argv[2])
header = sys.argv[3] if len(sys.argv) > 3 else ""
rows = [r for r in csv.reader(l for l in open(path) if not l.startswith("=="))]
h = rows[0]
ki, mi, vi, ii, ui = (h.index(k) for k in ("Kernel Name", "Metric Name", "Metric Value", "ID", "Metric Unit"))
scale = {"ns": 1e-9, "us": 1e-6, "ms": 1e-3, "byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}
per = collections.defaultdict(dict)
for r in rows[1:]:
    per[(int(r[ii]), r[ki].split("(")[0][:60])][r[mi]] = float(r[vi].replace(",", "")) * scale.get(r[ui], 1)
agg = collections.defaultdict(lambda: [0.0, 0.0, 0])
for (i, name), m in per.items():
    a = agg[name]
    a[0] += m.get("gpu__time_duration.sum", 0)
    a[1] += m.get("dram__bytes_read.sum", 0) + m.get("dram__bytes_write.sum", 0)
    a[2] += 1
if header:
    print(header)
tt = sum(a[0] for a in agg.values())
tb = sum(a[1] for a in agg.values())
print(f"{'us':>9} {'MB':>9} {'GB/s':>8} {'of peak':>8}  launches  kernel")
for name, (t, b, n) in sorted(agg.items(), key=lambda kv: -kv[1][0]):
    gbs = b / t / 1e9 if t else 0
    print(f"{t * 1e6:9.1f} {b / 1e6:9.1f} {gbs:8.0f} {gbs / peak:8.3f}  x{n:<3d}  {name}")
print(f"total {tt * 1e6:.1f} us, {tb / 1e6:.1f} MB DRAM, {tb / tt / 1e9:.0f} GB/s = {tb / tt / 1e9 / peak:.3f} of {peak:.1f} GB/s")
