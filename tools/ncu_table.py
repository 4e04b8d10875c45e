"""Per-kernel table from an ncu report: time, DRAM bytes, warps active, SM throughput, registers,
instructions, top stall reasons.  Usage: python tools/ncu_table.py report.ncu-rep"""
import csv
import io
import subprocess
import sys

M = ["gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
     "sm__warps_active.avg.pct_of_peak_sustained_active", "sm__throughput.avg.pct_of_peak_sustained_elapsed",
     "launch__registers_per_thread", "smsp__inst_executed.sum", "launch__grid_size"]
out = subprocess.run(["ncu", "-i", sys.argv[1], "--page", "raw", "--csv"], capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(out)))
h = rows[0]
stall = [k for k in h if k.startswith("smsp__average_warp_latency_issue_stalled") or
         (k.startswith("smsp__warp_issue_stalled_") and k.endswith("_per_warp_active.pct"))]
print(f"{'kernel':34s} {'us':>7s} {'rdMB':>7s} {'wrMB':>7s} {'wact%':>6s} {'sm%':>6s} {'reg':>4s} {'Minst':>7s} grid")
for r in rows[2:]:
    d = dict(zip(h, r))
    name = d["Kernel Name"].replace("void ", "")[:34]
    v = [d.get(m, "") for m in M]
    f = lambda x: float(x.replace(",", "")) if x else 0.0
    print(f"{name:34s} {f(v[0]) / 1e3 if f(v[0]) > 1e4 else f(v[0]):7.1f} {f(v[1]) / (1e6 if f(v[1]) > 1e5 else 1):7.1f} "
          f"{f(v[2]) / (1e6 if f(v[2]) > 1e5 else 1):7.1f} {f(v[3]):6.1f} {f(v[4]):6.1f} {v[5]:>4s} {f(v[6]) / 1e6:7.1f} {v[7]}")
    st = sorted(((f(d[k]), k) for k in stall if d.get(k)), reverse=True)[:4]
    print("    stalls:", ", ".join(f"{k.replace('smsp__warp_issue_stalled_', '').replace('_per_warp_active.pct', '')} {x:.0f}"
                                  for x, k in st))
