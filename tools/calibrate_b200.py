#!/usr/bin/env python
"""f2 calibration on one B200: the Fig. 2 analogue ("PCIe overhead ratios for
different batch data sizes") and the B200 values of InfPT_0 / baseTransCost.

For LR2S and CM2S micro-batches of 10^2 .. 10^7 records (7 kB .. 1.4 GB) this pushes the bytes
from page-locked host memory through the C ABI (lms_push_pinned: device-timed H2D on the copy
stream), runs one batch (lms_force_batch + lms_sync) and reads its lms_batch_record:
  h2d_s     PCIe copy of the batch (CUDA events on the copy stream)
  device_s  the batch's kernels (CUDA events)
  proc_s    Proc_i (reading R18: device + result D2H)
Reported per size (median of `reps` batches): those three, the PCIe share h2d / proc (Proc
contains the H2D: the batch's kernels wait for the copy on the device; the quantity of the
paper's Fig. 2), and a two-point model  t(bytes) = a + bytes / bw  of each
component (a from the smallest batch, bw from the largest).

Derived constants (readings R29 / R30 of DESIGN.md):
  InfPT_0  (Alg. 2's Part at which GPU and CPU costs are equal, Eq. 7-8): on the GPU side the
           knee of the measured cost curve — the batch size at which the size-proportional part
           of Proc equals its fixed per-batch part a — divided by NumCores (12,
           Part = batch bytes / NumCores).  Below it the batch is overhead-bound ("PCIe
           overhead marginal for small data"), above it time grows with bytes.
  baseTransCost  (Eq. 9: Trans = btc * Part / InfPT, so btc = Trans at Part = InfPT relative to
           an operator of base cost ~1): the measured H2D time over the device time at that
           knee batch size.
The values are reported, not wired in: lms_config_init keeps the paper's 150 KB / 0.1
 so the SPEC worked examples stay pinned; a caller sets cfg.inf_pt_bytes /
cfg.base_trans_cost from this file's output.

  python tools/calibrate_b200.py [--reps 7] [--out gpurun_out/calibration.json]
"""
from __future__ import annotations

import argparse
import json
import os
import statistics
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

SIZES = [100, 300, 1_000, 3_000, 10_000, 30_000, 100_000, 300_000, 1_000_000, 3_000_000, 10_000_000]


def host_batch(family, n_rec, seed=211104289):
    """n_rec records of second 0 in page-locked host memory (torch pinned tensor) + byte count."""
    import torch
    from lmsgen import cuda as gcu
    buf, nb = gcu.second_tensor(family, 0, n_rec, seed=seed)
    h = torch.empty(nb, dtype=torch.uint8, pin_memory=True)
    h.copy_(buf[:nb])
    del buf
    return h, nb


def sweep(kind, family, reps):
    import paper_2111_04289_b200 as P
    from paper_2111_04289_b200 import _lib as L
    rows = []
    for n_rec in SIZES:
        h, nb = host_batch(family, n_rec)
        # one query per size: MANUAL batches, each batch one dataset of the same bytes pushed
        # again at the next virtual second (ingest times increase: no late records)
        meas = {"h2d_s": [], "device_s": [], "proc_s": [], "d2h_s": [], "wall_s": []}
        with P.Query(kind, mode="manual", max_batch_bytes=max(nb + 4096, 1 << 20)) as q:
            for it in range(reps + 2):
                t0 = time.perf_counter()
                q.push_pinned(h.data_ptr(), nb, float(it))
                idx = q.force(float(it))
                q.sync(ok=(L.LMS_OK,))
                q.read_agg()
                wall = time.perf_counter() - t0
                r = q.record(idx)
                if it < 2:
                    continue                                    # warm-up
                for k in ("h2d_s", "device_s", "proc_s", "d2h_s"):
                    meas[k].append(r[k])
                meas["wall_s"].append(wall)
        med = {k: statistics.median(v) for k, v in meas.items()}
        med.update(records=n_rec, bytes=nb,
                   pcie_share=med["h2d_s"] / med["proc_s"])
        rows.append(med)
        print(f"{kind} {n_rec:>9} rec {nb / 1e6:10.3f} MB  h2d {med['h2d_s'] * 1e3:8.3f} ms  device "
              f"{med['device_s'] * 1e3:8.3f} ms  proc {med['proc_s'] * 1e3:8.3f} ms  wall "
              f"{med['wall_s'] * 1e3:8.3f} ms  PCIe share {med['pcie_share']:.3f}", file=sys.stderr)
        del h
    return rows


def derive(rows, num_cores=12):
    """Two-point model per component: the fixed part a = its time at the smallest batch (where
    the size-proportional part is negligible), the per-byte slope from the largest batch.
    Proc_i of a pinned push already contains its H2D (the batch's kernels wait for the copy on
    the device; reading R18), so Proc is the end-to-end cost of a batch."""
    lo, hi = rows[0], rows[-1]

    def model(key):
        a = lo[key]
        return a, max(hi[key] - a, 1e-12) / (hi["bytes"] - lo["bytes"])
    a_h, b_h = model("h2d_s")
    a_d, b_d = model("device_s")
    a_p, b_p = model("proc_s")
    knee = a_p / b_p                                     # bytes at which a == bytes * per_byte
    h2d_knee = a_h + b_h * knee                          # H2D / device time at the knee
    dev_knee = a_d + b_d * knee
    return {
        "model": {"h2d": {"a_s": a_h, "GBps": 1e-9 / b_h}, "device": {"a_s": a_d, "GBps": 1e-9 / b_d},
                  "proc": {"a_s": a_p, "GBps": 1e-9 / b_p}},
        "fixed_overhead_s": a_p,
        "knee_batch_bytes": knee,
        "inf_pt_bytes": knee / num_cores,
        "base_trans_cost": h2d_knee / dev_knee,
        "num_cores": num_cores,
    }


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--reps", type=int, default=7)
    ap.add_argument("--out", default=os.path.join(ROOT, "gpurun_out", "calibration.json"))
    ap.add_argument("--rederive", default=None, help="recompute 'derived' of an existing calibration file")
    args = ap.parse_args()
    if args.rederive:
        out = json.load(open(args.rederive))
        for k in ("LR2S", "CM2S"):
            for r in out[k]["sweep"]:
                r["pcie_share"] = r["h2d_s"] / r["proc_s"]
            out[k]["derived"] = derive(out[k]["sweep"])
        json.dump(out, open(args.out, "w"), indent=1)
        print(json.dumps({k: out[k]["derived"] for k in ("LR2S", "CM2S")}, indent=1))
        return
    import torch
    out = {"gpu": torch.cuda.get_device_name(0), "reps": args.reps,
           "method": "lms_push_pinned + lms_force_batch + lms_sync per batch; medians; see module doc"}
    for kind, fam in (("LR2S", "LR"), ("CM2S", "CM")):
        rows = sweep(kind, fam, args.reps)
        out[kind] = {"sweep": rows, "derived": derive(rows)}
        d = out[kind]["derived"]
        print(f"{kind}: fixed overhead {d['fixed_overhead_s'] * 1e6:.1f} us, knee {d['knee_batch_bytes'] / 1e6:.3f} MB,"
              f" InfPT_0 {d['inf_pt_bytes'] / 1e3:.1f} kB, baseTransCost {d['base_trans_cost']:.3f}", file=sys.stderr)
    os.makedirs(os.path.dirname(args.out), exist_ok=True)
    with open(args.out, "w") as fh:
        json.dump(out, fh, indent=1)
    print(json.dumps({k: (v["derived"] if isinstance(v, dict) and "derived" in v else v) for k, v in out.items()}))


if __name__ == "__main__":
    main()
