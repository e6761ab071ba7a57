"""Opcode histogram (per-tile) and top source lines of an ncu report — CM kernel tuning aid.
Usage: python tools/ncu_regions.py REPORT.ncu-rep [tiles]"""
import csv
import io
import subprocess
import sys

rep = sys.argv[1]
tiles = float(sys.argv[2]) if len(sys.argv) > 2 else 336e3
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "sass"],
                     capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(out)))
h = rows[1]
iE = h.index("Instructions Executed")
ops, tot = {}, 0
for r in rows[2:]:
    if len(r) <= iE or r[iE] in ("-", ""):
        continue
    n = int(r[iE])
    tot += n
    t = r[1].split()
    op = (t[1] if t[0].startswith("@") else t[0]).split(".")[0]
    ops[op] = ops.get(op, 0) + n
print(f"total {tot:,} warp inst = {tot / tiles:.1f} per tile")
for k, v in sorted(ops.items(), key=lambda x: -x[1])[:24]:
    print(f"  {k:10s} {v / tot * 100:5.1f}%  {v / tiles:7.1f}/tile")
raw = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
rr = list(csv.reader(io.StringIO(raw)))
d = dict(zip(rr[0], rr[2]))
for k in ("gpu__time_duration.sum", "smsp__issue_active.avg.pct_of_peak_sustained_active",
          "sm__pipe_alu_cycles_active.avg.pct_of_peak_sustained_active",
          "sm__inst_executed_pipe_fma.avg.pct_of_peak_sustained_active",
          "sm__inst_executed_pipe_xu.avg.pct_of_peak_sustained_active",
          "sm__inst_executed_pipe_lsu.avg.pct_of_peak_sustained_active",
          "sm__warps_active.avg.pct_of_peak_sustained_active", "launch__registers_per_thread",
          "dram__bytes_read.sum"):
    print(f"  {k} = {d.get(k)}")
st = {k.replace("smsp__pcsamp_warps_issue_stalled_", ""): float(v) for k, v in d.items()
      if k.startswith("smsp__pcsamp_warps_issue_stalled_") and not k.endswith("not_issued") and v not in ("", "n/a")}
s = sum(st.values())
print("  stalls: " + ", ".join(f"{k} {v / s * 100:.0f}%" for k, v in sorted(st.items(), key=lambda x: -x[1])[:9]))
