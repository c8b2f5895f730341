"""Aggregate ncu source-page stall samples per CUDA source line (dev helper)."""
import csv
import subprocess
import sys

rep, kernel = sys.argv[1], sys.argv[2]
top = int(sys.argv[3]) if len(sys.argv) > 3 else 30
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "-k", kernel, "--print-source", "cuda,sass"],
                     capture_output=True, text=True).stdout
rows = list(csv.reader(out.splitlines()))
cur, agg = None, {}
for r in rows:
    if not r:
        continue
    if r[0] == "File Path":
        cur = r[1].split("/")[-1]
        continue
    if r[0] in ("Function Name", "Line No"):
        continue
    if r[0] != "":
        try:
            agg[(cur, int(r[0]))] = (int(r[4]), int(r[7]), r[1][:110])
        except (ValueError, IndexError):
            pass
tot = sum(v[0] for v in agg.values()) or 1
print("total samples", tot)
for k, v in sorted(agg.items(), key=lambda kv: -kv[1][0])[:top]:
    print(f"{v[0]:7d} {100 * v[0] / tot:5.1f}% inst={v[1]:11d} {k[0]}:{k[1]} {v[2]}")
