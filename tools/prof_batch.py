"""Profiling driver: run a few 10M-record micro-batches of one workload (for ncu / sanitizers).

  python tools/prof_batch.py --workload cm2 --batches 3 [--records 10000000]
"""
import argparse
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import torch  # noqa: E402

import paper_2111_04289_b200 as P  # noqa: E402
from lmsgen import cuda as gcu  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--workload", default="cm2")
ap.add_argument("--batches", type=int, default=3)
ap.add_argument("--records", type=int, default=10_000_000)
ap.add_argument("--flags", type=int, default=0)
ap.add_argument("--jobs", type=int, default=None, help="CM: distinct jobIds J (default 1e4)")
ap.add_argument("--max-keys", type=int, default=None)
ap.add_argument("--sel-ppm", type=int, default=None, help="CM: eventType==1 selectivity in ppm")
ap.add_argument("--vehicles", type=int, default=None, help="LR: distinct vehicles V (default 1e6)")
a = ap.parse_args()
kind, fam = {"cm2": ("CM2S", "CM"), "lr2": ("LR2S", "LR"), "cm1": ("CM1S", "CM"), "lr1": ("LR1S", "LR")}[a.workload]
import lmsgen as g  # noqa: E402
params = (g.CMParams(num_jobs=a.jobs or 10 ** 4, sel_ppm=a.sel_ppm) if fam == "CM"
          else (g.LRParams(num_vehicles=a.vehicles) if a.vehicles else None))
bufs = [gcu.second_tensor(fam, t, a.records, params=params) if params else gcu.second_tensor(fam, t, a.records)
        for t in range(a.batches)]
# LR1 keeps every record of the current slide in its retained FIFO: room for 8 batches
rows_cap = max(1 << 20, (8 if kind.startswith("LR1") else 2) * a.records)
extra = {"max_keys": a.max_keys} if a.max_keys else {}
q = P.Query(kind, mode="manual", max_batch_bytes=1 << 20, max_result_rows=rows_cap, flags=a.flags, **extra)
for t, (b, n) in enumerate(bufs):
    q.push_device(b.data_ptr(), n, float(t))
    q.force(t + 1.0)
    q.sync()
    rows = q.read_lr1() if kind.startswith("LR1") else q.read_agg()
    bt, at, ct = q.kernel_times()
    print(f"batch {t}: {n} B, rows {len(rows)}, batch {bt*1e3:.3f} ms agg {at*1e3:.3f} ms close {ct*1e3:.3f} ms "
          f"agg {n / at / 1e9:.0f} GB/s", flush=True)
q.close()
