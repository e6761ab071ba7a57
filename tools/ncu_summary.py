#!/usr/bin/env python
"""Summarise one gpu_round.sh capture directory into profiles/<tag>/ (tracked).

  python tools/ncu_summary.py gpurun_out/<tag> profiles/<tag>

For every <name>.ncu-rep: <name>_details.csv (ncu --page details) and <name>_raw.json (the
headline raw metrics); launch lists are copied; profiles/ncu_traffic.json gets the per-launch
DRAM bytes of the aggregate kernels (bench.py's roofline.traffic)."""
import csv
import io
import json
import os
import shutil
import subprocess
import sys

RAW = ["gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
       "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed", "sm__throughput.avg.pct_of_peak_sustained_elapsed",
       "smsp__inst_executed.sum", "smsp__issue_active.avg.pct_of_peak_sustained_active",
       "sm__warps_active.avg.pct_of_peak_sustained_active", "launch__registers_per_thread",
       "launch__grid_size", "launch__block_size", "sm__cycles_elapsed.avg.per_second",
       "l1tex__data_bank_conflicts_pipe_lsu_mem_shared.sum", "smsp__average_warp_latency_issue_stalled_barrier",
       "lts__t_bytes.sum", "launch__occupancy_limit_shared_mem", "launch__shared_mem_per_block_dynamic"]
SCALE = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "Tbyte": 1e12}


def ncu(*args):
    return subprocess.run(["ncu", *args], check=True, capture_output=True, text=True).stdout


def raw_metrics(rep):
    rows = list(csv.reader(io.StringIO(ncu("-i", rep, "--page", "raw", "--csv"))))
    hdr, units, vals = rows[0], rows[1], rows[2]
    return {m: [vals[hdr.index(m)], units[hdr.index(m)]] for m in RAW if m in hdr}


def to_bytes(v):
    return float(v[0].replace(",", "")) * SCALE.get(v[1], 1)


def main(src, dst):
    os.makedirs(dst, exist_ok=True)
    traffic = {}
    for f in sorted(os.listdir(src)):
        p = os.path.join(src, f)
        if f.endswith(".ncu-rep"):
            name = f[:-8]
            with open(os.path.join(dst, name + "_details.csv"), "w") as fh:
                fh.write(ncu("-i", p, "--page", "details", "--csv"))
            raw = raw_metrics(p)
            with open(os.path.join(dst, name + "_raw.json"), "w") as fh:
                json.dump(raw, fh, indent=1)
            if name.endswith("_agg") and "dram__bytes_read.sum" in raw:
                wl = name[:-4]
                traffic[wl] = {"kernel": name, "dram_bytes_per_launch":
                               to_bytes(raw["dram__bytes_read.sum"]) + to_bytes(raw["dram__bytes_write.sum"]),
                               "duration": raw.get("gpu__time_duration.sum")}
        elif f.startswith("launches_") or f in ("bench.json", "nvsmi.txt", "pytest_gpu.txt", "smoke.txt", "kernel_timings_by_kind.txt"):
            shutil.copy(p, os.path.join(dst, f))
    if traffic:
        tp = os.path.join(os.path.dirname(os.path.abspath(dst)), "ncu_traffic.json")
        old = json.load(open(tp)) if os.path.exists(tp) else {}
        old.update(traffic)
        old["_source"] = f"ncu --set full --clock-control none, one launch per kernel ({dst}/*_raw.json)"
        with open(tp, "w") as fh:
            json.dump(old, fh, indent=1)
    print(json.dumps(traffic, indent=1))


if __name__ == "__main__":
    main(sys.argv[1], sys.argv[2])
