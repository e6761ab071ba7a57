#!/usr/bin/env python
"""Wall-clock breakdown of one bench step's host calls (push_device / force / sync / read_agg)."""
import os
import statistics
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))


def main(workload="cm2", steps=30):
    import torch
    import paper_2111_04289_b200 as P
    from lmsgen import cuda as gcu
    fam, kind = ("CM", "CM2S") if workload == "cm2" else ("LR", "LR2S")
    bufs = [gcu.second_tensor(fam, t, 10_000_000, seed=211104289) for t in range(steps)]
    q = P.Query(kind, mode="manual", max_batch_bytes=1 << 20)
    tm = {k: [] for k in ("push", "force", "sync", "read", "times", "total")}
    for t, (buf, n) in enumerate(bufs):
        a = time.perf_counter()
        q.push_device(buf.data_ptr(), n, float(t))
        b = time.perf_counter()
        q.force(float(t) + 1.0)
        c = time.perf_counter()
        q.sync()
        d = time.perf_counter()
        rows = q.read_agg()
        e = time.perf_counter()
        bt, at, ct = q.kernel_times()
        f = time.perf_counter()
        if t >= 3:
            for k, v in (("push", b - a), ("force", c - b), ("sync", d - c), ("read", e - d), ("times", f - e),
                         ("total", f - a)):
                tm[k].append(v * 1e6)
        if t >= 3 and (t < 8 or len(rows)):
            print(f"t={t} rows={len(rows)} batch={bt*1e6:.0f}us agg={at*1e6:.0f}us close={ct*1e6:.0f}us "
                  f"force={1e6*(c-b):.0f} sync={1e6*(d-c):.0f} read={1e6*(e-d):.0f}us")
    for k, v in tm.items():
        print(f"{k:6s} median {statistics.median(v):8.1f} us   max {max(v):8.1f} us")


if __name__ == "__main__":
    main(*(sys.argv[1:2] or ["cm2"]))
