"""Print the judged metrics of every kernel in an ncu --set full report (dev helper).

python tools/ncu_summary.py report.ncu-rep "header" > profiles/rNN_ncu_top3.txt
"""
import csv
import subprocess
import sys

METRICS = ["gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
           "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed", "sm__warps_active.avg.pct_of_peak_sustained_active",
           "smsp__issue_active.avg.pct_of_peak_sustained_active", "smsp__inst_executed.sum",
           "launch__registers_per_thread", "launch__occupancy_limit_registers", "launch__occupancy_limit_shared_mem",
           "launch__grid_size", "launch__block_size", "lts__t_sector_hit_rate.pct", "l1tex__t_sector_hit_rate.pct",
           "sm__throughput.avg.pct_of_peak_sustained_elapsed", "sm__inst_executed_pipe_fp64.avg.pct_of_peak_sustained_active"]
PFX = "smsp__pcsamp_warps_issue_stalled_"

rep, header = sys.argv[1], sys.argv[2] if len(sys.argv) > 2 else ""
out = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
rows = list(csv.reader(out.splitlines()))
hdr, units, data = rows[0], rows[1], rows[2:]
col = {h: i for i, h in enumerate(hdr)}
if header:
    print(header)
    print()
for r in data:
    print("==", r[col["Kernel Name"]].split("(")[0])
    for m in METRICS:
        if m in col:
            print(f"  {m:60s} {r[col[m]]:>20s} {units[col[m]]}")
    st = {h[len(PFX):]: float(r[i].replace(",", "") or 0) for h, i in col.items()
          if h.startswith(PFX) and not h.endswith("_not_issued")}
    tot = sum(st.values()) or 1.0
    top = sorted(st.items(), key=lambda kv: -kv[1])[:6]
    print("  top stall reasons (pc samples): " + ", ".join(f"{k} {100 * v / tot:.0f}%" for k, v in top))
