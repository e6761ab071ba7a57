#!/usr/bin/env python
"""f3: latency dynamics of the micro-batch sizer at B200 scale (§V-D/§V-E).

Part A — deadline-violation rates (Tables "Violation rate when deadline is 5 / 7 seconds",
P:156-214): OS(t3) against CG(d5) / CG(d7) on LR1 / CM1 under U(2.5)- and R(0.1,5)-shaped
traffic, 90 virtual minutes each, one dataset per second.  The paper ran
Spark on an RTX 2080 Ti at 2.5k records/s; a B200 at those rates finishes a batch in
microseconds, so the rates are SCALED so that the mean offered load is a fixed fraction
(`--load`, default 0.5 and 0.9) of the B200's end-to-end capacity for that record type (the
calibrated Proc bandwidth of a pinned push, H2D included, tools/calibrate_b200.py), keeping the traffic's shape
(U: normal, sigma = mu/4; R: uniform over [0.1, 5] x scale).  Admission is the library's own
Alg. 1 decision (lms_admit_decision, the function lms_poll calls; CG(dN) = sliding branch with
SlideTime := N, reading R16) and OS(tN) admits everything buffered every N s; Proc of a batch
comes from the B200 model  Proc(bytes) = a + bytes / bw  fitted on this GPU (calibration
file), the 10 ms poll of P:564 and one batch in flight.  A dataset violates the deadline when
completion - ingest > d (#violation / #total datasets).

Sensitivity runs repeat Part A with a fixed per-batch overhead of a seconds (`--fixed`, a
Spark-like micro-batch cost; the B200's is ~35 us): they show the regime in which the paper's
OS(t3) runaway appears — a 3 s batch takes longer than 3 s (a + 3 s x load > 3 s) while the
deadline sizer's larger batches still keep up.

Part B — timelines (Fig. "Timeline during the initial 20-minute run of LR1S / LR1T",
P:1002-1028): LMStream (Alg. 1) against the paper's Baseline (Spark's fixed 10 s trigger,
"always performs ten seconds of buffering", P:1019 = OS(t10)) on R(L,U) traffic, run for real
on the GPU through the C ABI on a virtual clock (tools/latency_configs.py machinery: data
generated on the GPU per second, pushed as device datasets, measured Proc advances the
clock).  Per batch: MaxLat (Eq. 5) and batch bytes.

  python tools/f3_dynamics.py --calib profiles/r02b/calibration.json [--part A|B|AB]
        [--out gpurun_out/f3_dynamics.json]
"""
from __future__ import annotations

import argparse
import ctypes as C
import json
import math
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

POLL = 0.01
LR_BYTES, CM_BYTES = 70.0, 137.5


def admit_fn():
    from paper_2111_04289_b200 import _lib as L

    def decide(mode, slide, deadline, now, ing, by, avg_thput, hist):
        n = len(ing)
        ia = (C.c_double * max(n, 1))(*ing)
        ba = (C.c_uint64 * max(n, 1))(*by)
        ha = (C.c_double * max(len(hist), 1))(*hist)
        adm, est, rsn = C.c_int32(), C.c_double(), C.c_int32()
        L.check(L.lms_admit_decision(mode, slide, deadline, now, ia, ba, n, avg_thput, ha, len(hist),
                                     C.byref(adm), C.byref(est), C.byref(rsn)), "lms_admit_decision")
        return bool(adm.value)
    return decide, L


def simulate(counts, rec_bytes, proc_model, system, d, t_end):
    """Virtual-clock loop; system = ("OS", N) or ("CG", d).  Returns per-dataset latencies and
    per-batch (admit, n_datasets, bytes, MaxLat)."""
    decide, L = admit_fn()
    a, bw = proc_model
    datasets = [(float(t + 1), int(c * rec_bytes)) for t, c in enumerate(counts)]   # file complete at t+1
    nxt, pend = 0, []
    cum_b = cum_p = 0.0
    hist, lat, batches = [], [], []
    busy_until, next_trig = 0.0, system[1] if system[0] == "OS" else 0.0
    tick = 0
    while True:
        now = tick * POLL
        if now > t_end:
            break
        while nxt < len(datasets) and datasets[nxt][0] <= now + 1e-12:
            pend.append(datasets[nxt])
            nxt += 1
        if now + 1e-12 >= busy_until and pend:
            if system[0] == "OS":
                adm = now + 1e-12 >= next_trig
                if adm:
                    next_trig = (math.floor(now / system[1] + 1e-9) + 1) * system[1]
            else:
                thp = cum_b / cum_p if cum_p > 0 else 0.0
                adm = decide(L.LMS_MODE_DEADLINE, 0.0, d, now, [x[0] for x in pend], [x[1] for x in pend], thp, hist)
            if adm:
                by = sum(x[1] for x in pend)
                proc = a + by / bw
                end = now + proc
                ml = max(now - x[0] for x in pend) + proc                            # Eq. 5
                for x in pend:
                    lat.append(end - x[0])
                batches.append((now, len(pend), by, ml))
                hist.append(ml)
                cum_b += by
                cum_p += proc                                                         # Eq. 4
                pend = []
                busy_until = end
                tick = max(tick + 1, int(math.ceil(end / POLL - 1e-9)))
                continue
        tick += 1                                       # (OS: a trigger during a batch fires at the first poll after it)
    return lat, batches


def part_a(calib, loads, minutes, fixed_s=None):
    """fixed_s: override the calibrated fixed per-batch overhead (sensitivity: a Spark-like
    per-micro-batch cost instead of the B200's tens of microseconds)."""
    import lmsgen as g
    out = []
    for fam, rec_b, ck in (("LR1", LR_BYTES, "LR2S"), ("CM1", CM_BYTES, "CM2S")):
        dm = calib[ck]["derived"]["model"]
        a = dm["proc"]["a_s"] if fixed_s is None else fixed_s   # Proc of a pinned push contains its H2D
        bw = dm["proc"]["GBps"] * 1e9                 # end-to-end bytes/s
        cap_rps = bw / rec_b
        for shape in ("U(2.5)", "R(0.1,5)"):
            base = g.Traffic.parse(shape)
            mean_paper = base.rate if base.kind == "U" else (base.lo + base.hi) / 2
            for load in loads:
                k = load * cap_rps / mean_paper
                if base.kind == "U":
                    tr = g.Traffic("U", rate=int(round(base.rate * k)))
                else:
                    tr = g.Traffic("R", lo=int(round(base.lo * k)), hi=int(round(base.hi * k)))
                secs = int(minutes * 60)
                counts = [tr.count(t) for t in range(secs)]
                for d in (5.0, 7.0):
                    row = {"workload": f"{fam}-{shape}", "load": load, "scale": k, "deadline_s": d, "fixed_s": a,
                           "mean_rec_per_s": sum(counts) / secs, "capacity_rec_per_s": cap_rps}
                    for name, system in (("OS(t3)", ("OS", 3.0)), (f"CG(d{int(d)})", ("CG", d))):
                        lat, bat = simulate(counts, rec_b, (a, bw), system, d, secs + 30.0)
                        viol = sum(1 for x in lat if x > d + 1e-9)
                        row[name] = {"violation_rate": viol / len(lat), "datasets": len(lat), "batches": len(bat),
                                     "maxlat_p50": sorted(b[3] for b in bat)[len(bat) // 2],
                                     "maxlat_max": max(b[3] for b in bat),
                                     "mean_datasets_per_batch": len(lat) / len(bat)}
                    print(json.dumps(row), file=sys.stderr)
                    out.append(row)
    return out


def part_b(minutes, traffic):
    import paper_2111_04289_b200 as P
    sys.path.insert(0, os.path.join(ROOT, "tools"))
    import latency_configs as LC
    res = {}
    for kind in ("LR1S", "LR1T"):
        for name, over in (("LMStream", dict(mode="lmstream")), ("Baseline OS(t10)", dict(mode="trigger", trigger_s=10.0))):
            with P.Query(kind, max_batch_bytes=1 << 30, max_result_rows=1 << 24, **over) as q:
                src = LC.Source(q, "LR", traffic, int(minutes * 60), 1, 211104289)
                LC.run_stream([src], minutes * 60.0)
                recs = src.recs
            res[f"{kind} {name}"] = {
                "admit_s": [r["admit_time_s"] for r in recs],
                "max_lat_s": [r["max_lat_s"] for r in recs],
                "batch_bytes": [r["batch_bytes"] for r in recs],
                "proc_s": [r["proc_s"] for r in recs],
            }
            ml = sorted(res[f"{kind} {name}"]["max_lat_s"])
            print(f"{kind} {name}: {len(recs)} batches, MaxLat p50 {ml[len(ml) // 2]:.3f} s max {ml[-1]:.3f} s", file=sys.stderr)
    return res


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--calib", default=os.path.join(ROOT, "gpurun_out", "calibration.json"))
    ap.add_argument("--part", default="AB")
    ap.add_argument("--loads", default="0.5,0.9")
    ap.add_argument("--minutes-a", type=float, default=90.0)
    ap.add_argument("--fixed", default="1.0:0.5,0.7;2.5:0.3",
                    help="sensitivity runs 'a:load,..;a:load': fixed per-batch overhead a [s] at those loads")
    ap.add_argument("--minutes-b", type=float, default=20.0)
    ap.add_argument("--traffic-b", default="R(50,500)")
    ap.add_argument("--out", default=os.path.join(ROOT, "gpurun_out", "f3_dynamics.json"))
    args = ap.parse_args()
    out = {}
    if "A" in args.part:
        calib = json.load(open(args.calib))
        out["violation"] = part_a(calib, [float(x) for x in args.loads.split(",")], args.minutes_a)
        out["violation_fixed_overhead"] = []
        for spec in filter(None, args.fixed.split(";")):            # "a:load,load;a:load"
            fa, lds = spec.split(":")
            out["violation_fixed_overhead"] += part_a(calib, [float(x) for x in lds.split(",")],
                                                      args.minutes_a, fixed_s=float(fa))
        out["calibration"] = {k: calib[k]["derived"] for k in ("LR2S", "CM2S")}
    if "B" in args.part:
        out["timeline"] = part_b(args.minutes_b, args.traffic_b)
        out["timeline_traffic"] = args.traffic_b
    os.makedirs(os.path.dirname(args.out), exist_ok=True)
    json.dump(out, open(args.out, "w"))
    print(f"wrote {args.out}", file=sys.stderr)


if __name__ == "__main__":
    main()
