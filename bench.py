#!/usr/bin/env python
"""bench.py — LMStream micro-batch hot path on B200 (BASELINE.json metric).

metric: records/s (and HBM GB/s) per micro-batch for CM2 / LR2 10M-record batches; p99 batch
latency.  Headline workload = BASELINE config C4 (CM2S, B(10000): one 10M-record dataset per
second, one micro-batch per second, MANUAL batching); LR2S C4' is reported beside it.

  python bench.py [--gpus N] [--steps K] [--warmup W] [--impl reference] [--workload cm2|lr2]

A step = one micro-batch through the whole hot path via the C ABI: push (device-resident
input, borrowed), admission, Alg. 2 labels, framing/decode/filter/aggregate kernel, window
close kernel, batch report + result rows to the host.  `value` = records of all ranks / max
over ranks of the device-clock time of the K timed steps (CUDA events, synchronize + barrier
on both sides).  Inputs (1.375 GB / 0.70 GB per step) exceed L2, so no L2 flush is needed.
`e2e` = same metric with the inputs in pinned HOST memory: lms_push (H2D inside) + batch +
rows to host per step.  N > 1 (torchrun): every rank runs its own 10M-record partition of
each step (weak scaling) — see DESIGN.md §7 for the partial-aggregate merge.
"""
from __future__ import annotations

import argparse
import json
import os
import statistics
import subprocess
import sys
import threading
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

PEAKS_FALLBACK = {"hbm_gbs": 6650.0}   # B200_PROFILING.md fallback if MEASURED_PEAKS.json is absent

WORKLOADS = {
    "cm2": dict(kind="CM2S", family="CM", traffic="B(10000)", records=10_000_000,
                desc="CM2S C4: 10M-record micro-batches (B(10000), 1 batch = 1 s), J=1e4 jobIds, "
                     "eventType==1 selectivity 0.26, 130-145 B records"),
    "lr2": dict(kind="LR2S", family="LR", traffic="B(10000)", records=10_000_000,
                desc="LR2S C4': 10M-record micro-batches (B(10000), 1 batch = 1 s), 10 xways x 2 dirs "
                     "x 100 segs, 70 B records"),
}


def peaks():
    p = os.path.join(ROOT, "MEASURED_PEAKS.json")
    if os.path.exists(p):
        with open(p) as fh:
            d = json.load(fh)
        return {"hbm_gbs": float(d["hbm_gbs"]), "source": "measured"}
    return {"hbm_gbs": PEAKS_FALLBACK["hbm_gbs"], "source": "fallback"}


def ncu_traffic(workload):
    """dram__bytes_read.sum + dram__bytes_write.sum per aggregate launch, from the committed
    ncu --set full summary (profiles/ncu_traffic.json), or None."""
    p = os.path.join(ROOT, "profiles", "ncu_traffic.json")
    if not os.path.exists(p):
        return None
    with open(p) as fh:
        return json.load(fh).get(workload, {}).get("dram_bytes_per_launch")


class ClockSampler:
    """nvidia-smi clocks + throttle reasons during the timed region (B200_PROFILING.md)."""

    def __init__(self, index, period_ms=20):
        self.index = index
        self.period_ms = period_ms
        self.samples = []          # (wall time, [fields])
        self.proc = None
        self.t0 = self.t1 = None

    def __enter__(self):
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", "-i", str(self.index), "--query-gpu=clocks.sm,clocks.max.sm,"
                 "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
                 "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap",
                 "--format=csv,noheader,nounits", "-lms", str(self.period_ms)],
                stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            self.t = threading.Thread(target=self._read, daemon=True)
            self.t.start()
            t_end = time.time() + 5.0          # wait for the first sample (nvidia-smi startup)
            while not self.samples and time.time() < t_end:
                time.sleep(0.01)
        except Exception:
            self.proc = None
        return self

    def _read(self):
        for line in self.proc.stdout:
            parts = [x.strip() for x in line.split(",")]
            if len(parts) >= 6:
                self.samples.append((time.time(), parts))

    def mark(self, start: bool):
        if start:
            self.t0 = time.time()
        else:
            self.t1 = time.time()
            time.sleep(2.5 * self.period_ms / 1e3)   # let the sample covering the end arrive

    def __exit__(self, *a):
        if self.proc:
            self.proc.terminate()
            try:
                self.proc.wait(timeout=2)
            except Exception:
                self.proc.kill()

    def summary(self):
        """Samples taken during the timed region (+- one sampling period)."""
        pad = 1.5 * self.period_ms / 1e3
        win = [p for t, p in self.samples
               if self.t0 is not None and self.t0 - pad <= t <= (self.t1 or t) + pad]
        if not win:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["unsampled"]}
        sm = [float(s[0]) for s in win if s[0].replace(".", "").isdigit()]
        mx = [float(s[1]) for s in win if s[1].replace(".", "").isdigit()]
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        reasons = sorted({names[i] for s in win for i in range(4) if s[2 + i] == "Active"})
        return {"sm_mhz": statistics.median(sm) if sm else None, "sm_max_mhz": max(mx) if mx else None,
                "reasons": reasons, "samples": len(win), "period_ms": self.period_ms}


# ----------------------------------------------------------------------------- GPU arm

def gen_inputs(wl, seconds, t0, seed, torch):
    from lmsgen import cuda as gcu
    bufs = []
    for t in range(t0, t0 + seconds):
        buf, n = gcu.second_tensor(wl["family"], t, wl["records"], seed=seed)
        bufs.append((buf, n, t))
    torch.cuda.synchronize()
    return bufs


def device_run(wl, steps, warmup, seed, rank, world, torch, dist, p2p=False):
    import numpy as np
    import paper_2111_04289_b200 as P
    dev = torch.cuda.current_device()
    inputs = gen_inputs(wl, warmup + steps, 0, seed, torch)
    from paper_2111_04289_b200 import _lib as L
    # single GPU: two batches in flight (LMS_FLAG_PIPELINE) so the host's launch / completion
    # work for batch i overlaps the GPU running batch i-1 (stream order keeps results exact)
    q = P.Query(wl["kind"], mode="manual", device=dev, max_batch_bytes=1 << 20, rank=rank, world=world,
                flags=L.LMS_FLAG_PIPELINE if world == 1 else 0)
    out = {"agg_s": [], "close_s": [], "batch_s": [], "rows": 0}
    rowbuf = np.zeros(1 << 16, P.AGG_DTYPE)             # caller-owned result buffer (pages touched)
    if world > 1:
        from paper_2111_04289_b200.dist import RankHandle, TorchDistExchange, run_batch
        h, ex = RankHandle(q), TorchDistExchange()
        if p2p:
            ex.setup_p2p([h], device_watermark=p2p == "device")

    def step(buf, n, t):
        q.push_device(buf.data_ptr(), n, float(t))
        if world > 1:                     # partial aggregates merged by key owner
            run_batch([h], ex, float(t) + 1.0, p2p=p2p)
        else:
            q.force(float(t) + 1.0)       # pipelined: completes batch i-2 while i-1 runs
        return drain()

    def drain():
        n = 0
        while True:                                   # results to host, into a reused buffer
            rows = q.read_agg(out=rowbuf)
            n += len(rows)
            if len(rows) < len(rowbuf):
                return n

    for i in range(warmup):
        step(*inputs[i])
    q.sync()
    drain()
    launches0 = q.kernel_launches()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    with ClockSampler(dev) as clk:
        if world > 1:
            dist.barrier()
        torch.cuda.synchronize()
        clk.mark(True)
        e0.record()
        for i in range(warmup, warmup + steps):
            out["rows"] += step(*inputs[i])
            b, a, c = q.kernel_times()               # the most recently completed batch
            out["batch_s"].append(b)
            out["agg_s"].append(a)
            out["close_s"].append(c)
        q.sync()                                     # every timed batch complete, rows on the host
        out["rows"] += drain()
        e1.record()
        torch.cuda.synchronize()
        if world > 1:
            dist.barrier()
        clk.mark(False)
    el = e0.elapsed_time(e1) / 1e3
    out["elapsed_s"] = el
    out["launches"] = q.kernel_launches() - launches0
    out["clocks"] = clk.summary()
    out["bytes_per_step"] = statistics.mean(n for _, n, _ in inputs[warmup:])
    out["records"] = [q.record(i)["num_records"] for i in range(warmup, warmup + steps)]
    out["bad"] = sum(q.record(i)["bad_records"] for i in range(warmup, warmup + steps))
    q.close()
    del inputs
    torch.cuda.empty_cache()
    return out


def e2e_run(wl, steps, warmup, seed, torch, rank=0, world=1, dist=None, p2p=False):
    """Inputs in pinned host memory; each step: lms_push (H2D) + batch + rows to host.
    N > 1: every rank pushes its own partition; batches run the dist.py protocol; the time is
    the max over ranks."""
    import numpy as np
    import paper_2111_04289_b200 as P
    dev = torch.cuda.current_device()
    n_sec = warmup + steps
    dev_in = gen_inputs(wl, n_sec, 0, seed, torch)
    host = []
    for buf, n, t in dev_in:
        h = torch.empty(n, dtype=torch.uint8, pin_memory=True)
        h.copy_(buf[:n])
        host.append((h, n, t))
    del dev_in
    torch.cuda.synchronize()
    torch.cuda.empty_cache()
    cap = max(n for _, n, _ in host) + 4096
    q = P.Query(wl["kind"], mode="manual", device=dev, max_batch_bytes=cap, rank=rank, world=world)
    rowbuf = np.zeros(1 << 16, P.AGG_DTYPE)
    if world > 1:
        from paper_2111_04289_b200.dist import RankHandle, TorchDistExchange, run_batch
        hd, ex = RankHandle(q), TorchDistExchange()
        if p2p:
            ex.setup_p2p([hd], device_watermark=p2p == "device")
    d2h = []

    def step(h, n, t):
        q.push((h.data_ptr(), n), float(t))
        if world > 1:
            run_batch([hd], ex, float(t) + 1.0, p2p=p2p)
        else:
            q.force(float(t) + 1.0)
            q.sync()
        nb = 0
        while True:
            rows = q.read_agg(out=rowbuf)
            nb += rows.nbytes
            if len(rows) < len(rowbuf):
                break
        d2h.append(nb + 88)

    for i in range(warmup):
        step(*host[i])
    if world > 1:
        dist.barrier()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for i in range(warmup, n_sec):
        step(*host[i])
    e1.record()
    torch.cuda.synchronize()
    if world > 1:
        dist.barrier()
    el = e0.elapsed_time(e1) / 1e3
    if world > 1:
        el = max_over_ranks(el, torch, dist)
    recs = [q.record(i) for i in range(warmup, n_sec)]
    q.close()
    return {"elapsed_s": el, "h2d_bytes_per_step": float(np.mean([n for _, n, _ in host[warmup:]])),
            "d2h_bytes_per_step": float(np.mean(d2h[warmup:])),
            "proc_s": [r["proc_s"] for r in recs], "h2d_s": [r["h2d_s"] for r in recs]}


def max_over_ranks(x, torch, dist):
    """Max of a host scalar over ranks (NCCL: a device tensor; gloo: a host tensor)."""
    dev = "cuda" if dist.get_backend() == "nccl" else "cpu"
    t = torch.tensor([float(x)], device=dev, dtype=torch.float64)
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    return float(t.item())


def pct(v, p):
    from oracle.metrics import percentile_nearest_rank  # nearest rank: same rule as the library
    return percentile_nearest_rank(v, p)


# ----------------------------------------------------------------------------- CPU / reference arm

def _sample_datasets(fam, seconds, rate, seed, t0=0):
    """Input bytes of the bounded CPU sample: the records of seconds t0.. of the same seeded
    workload (the GPU generator when a GPU is present — byte-identical to the Python one —
    so that generating the sample costs no CPU minutes; generation is not timed)."""
    try:
        import torch
        if torch.cuda.is_available():
            from lmsgen import cuda as gcu
            out = []
            for t in range(t0, t0 + seconds):
                buf, n = gcu.second_tensor(fam, t, rate, seed=seed)
                out.append(bytes(buf[:n].cpu().numpy()))
            return out
    except Exception:
        pass
    import lmsgen as g
    return [d for _, d in g.stream_datasets(fam, f"B({rate / 1000})", seconds, seed=seed, t0=t0)]


def cpu_sample(kind, seconds=2, rate=450_000, seed=211104289, t0=0):
    """The oracle as it stands (single-threaded Python) on a bounded sample of the same
    workload: `seconds` datasets of `rate` records (seconds t0..), parse + windows (Replay,
    flush).  Default ~0.9M records: about 10 s of CPU."""
    from oracle import queries as Q
    fam = "CM" if kind.startswith("CM") else "LR"
    data = _sample_datasets(fam, seconds, rate, seed, t0)
    nbytes = sum(len(d) for d in data)
    q = Q.query_spec(kind)
    t0_ = time.perf_counter()
    outs = Q.replay(q, [[d] for d in data])
    el = time.perf_counter() - t0_
    n = seconds * rate
    return {"records": n, "bytes": nbytes, "elapsed_s": el, "records_per_s": n / el,
            "rows": sum(len(o.rows) for o in outs)}


METRIC = "records/s per micro-batch (CM2 10M-record batches); HBM GB/s; p99 batch latency"


def reference_arm(args, wl, rank, world):
    if rank != 0:
        return 0
    per = []
    for _ in range(args.warmup):
        cpu_sample(wl["kind"], seconds=1, rate=10_000)
    for i in range(args.steps):       # each step: 2 seconds x 30k records of the workload
        per.append(cpu_sample(wl["kind"], seconds=2, rate=30_000, t0=2 * i))
    tot_r = sum(p["records"] for p in per)
    tot_t = sum(p["elapsed_s"] for p in per)
    v = tot_r / tot_t
    line = {"impl": "reference", "metric": METRIC,
            "value": v, "unit": "records/s", "n_gpus": world, "steps": args.steps, "warmup": args.warmup,
            "ms_per_step": 1e3 * tot_t / args.steps, "higher_is_better": True, "scaling": "weak",
            "vs_baseline": None, "dtype": "int64+f64 (Python)", "data": "synthetic (lmsgen, seeded)",
            "config": {"workload": wl["desc"], "records_per_batch_per_gpu": wl["records"],
                       "global_batch": wl["records"] * world, "parallelism": "oracle, 1 host thread",
                       "sample": "bounded sample of the workload: 2 datasets x 30000 records per step"},
            "cpu_baseline": {"value": v, "unit": "records/s", "cores": 1, "kind": "oracle",
                             "sample": "2 x 30000-record datasets (seconds 2i, 2i+1) of the same generator per step"},
            "e2e": {"value": v, "unit": "records/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
    print(json.dumps(line))
    return 0


# ----------------------------------------------------------------------------- main

def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=20)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--workload", default="cm2", choices=list(WORKLOADS))
    ap.add_argument("--secondary", default="lr2", help="also measure this workload ('' = none)")
    ap.add_argument("--e2e-steps", type=int, default=5)
    ap.add_argument("--seed", type=int, default=211104289)
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--exchange", default="alltoall", choices=["alltoall", "p2p", "p2p-async", "device"],
                    help="N > 1: partial-aggregate exchange (NCCL all-to-all + owner merge; the fused "
                         "peer-memory push into the owners' accumulators with host-driven passes; or "
                         "the same fully enqueued with a device-side barrier; or also the watermark "
                         "exchange on the device: no per-batch collective)")
    args = ap.parse_args()
    args.warmup = max(args.warmup, 3)

    rank = int(os.environ.get("RANK", "0"))
    world = int(os.environ.get("WORLD_SIZE", "1"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    wl = WORKLOADS[args.workload]
    if args.impl == "reference":
        return reference_arm(args, wl, rank, world)

    import torch
    dist = None
    # one process per GPU; LMS_DIST_BACKEND=gloo (tests only) lets N ranks share fewer GPUs
    backend = os.environ.get("LMS_DIST_BACKEND", "nccl")
    local = local % max(1, torch.cuda.device_count())
    torch.cuda.set_device(local)
    if world > 1:
        import torch.distributed as dist
        if backend == "nccl":
            dist.init_process_group("nccl", device_id=torch.device("cuda", local))
        else:
            dist.init_process_group(backend)
    from paper_2111_04289_b200 import build  # noqa: F401  (library must already be built)

    seed = args.seed + 7919 * rank        # each rank: its own partition of the global batch
    p2p = {"alltoall": False, "p2p": True, "p2p-async": "async", "device": "device"}[args.exchange]
    res = device_run(wl, args.steps, args.warmup, seed, rank, world, torch, dist, p2p)
    el = res["elapsed_s"]
    if world > 1:
        el = max_over_ranks(el, torch, dist)
    recs = wl["records"] * world * args.steps
    value = recs / el
    pk = peaks()
    agg_avg = statistics.mean(res["agg_s"])
    achieved = res["bytes_per_step"] / agg_avg / 1e9
    sec = None
    if args.secondary and args.secondary != args.workload:
        w2 = WORKLOADS[args.secondary]
        r2 = device_run(w2, max(5, args.steps // 2), args.warmup, seed, rank, world, torch, dist, p2p)
        if world > 1:
            r2["elapsed_s"] = max_over_ranks(r2["elapsed_s"], torch, dist)
        a2 = statistics.mean(r2["agg_s"])
        sec = {"workload": w2["desc"], "records_per_s": w2["records"] * world * len(r2["agg_s"]) / r2["elapsed_s"],
               "ms_per_step": 1e3 * r2["elapsed_s"] / len(r2["agg_s"]),
               "agg_kernel_ms": 1e3 * a2, "agg_GBps": r2["bytes_per_step"] / a2 / 1e9,
               "agg_frac_of_measured_hbm": r2["bytes_per_step"] / a2 / 1e9 / pk["hbm_gbs"],
               "batch_device_ms_p50": 1e3 * pct(r2["batch_s"], 50),
               "batch_device_ms_p99": 1e3 * pct(r2["batch_s"], 99),
               "traffic_ncu_bytes": ncu_traffic(args.secondary), "clocks": r2["clocks"]}
    e2e = None
    if args.e2e_steps > 0:
        e = e2e_run(wl, args.e2e_steps, 1, seed, torch, rank, world, dist, p2p)
        e2e = {"value": wl["records"] * world * args.e2e_steps / e["elapsed_s"], "unit": "records/s",
               "h2d_bytes_per_step": e["h2d_bytes_per_step"], "d2h_bytes_per_step": e["d2h_bytes_per_step"],
               "steps": args.e2e_steps, "proc_ms_p50": 1e3 * pct(e["proc_s"], 50),
               "proc_ms_p99": 1e3 * pct(e["proc_s"], 99), "h2d_ms_mean": 1e3 * statistics.mean(e["h2d_s"]),
               # the e2e leg is bound by the host link: its achieved pinned H2D bandwidth
               "h2d_gbs": e["h2d_bytes_per_step"] / statistics.mean(e["h2d_s"]) / 1e9}
    cpu = None
    if rank == 0 and not args.no_cpu_baseline:
        s = cpu_sample(wl["kind"], seconds=2, rate=800_000)   # ~10 s of oracle CPU
        cpu = {"value": s["records_per_s"], "unit": "records/s", "cores": 1, "kind": "oracle",
               "sample": f"{s['records']} records (2 x 800000-record datasets of the same generator), "
                         f"{s['elapsed_s']:.1f} s single-threaded Python"}
    if rank == 0:
        line = {
            "metric": METRIC,
            "value": value, "unit": "records/s", "n_gpus": world, "steps": args.steps, "warmup": args.warmup,
            "ms_per_step": 1e3 * el / args.steps, "higher_is_better": True, "scaling": "weak",
            "vs_baseline": None, "dtype": "u64 fixed-point sums + f64 AVG", "data": "synthetic (lmsgen, seeded)",
            "config": {"workload": wl["desc"], "records_per_batch_per_gpu": wl["records"],
                       "global_batch": wl["records"] * world, "batch_bytes_per_gpu": res["bytes_per_step"],
                       "parallelism": (f"dp{world} (row partition per rank; exchange: {args.exchange})"
                                       if world > 1 else "single GPU"),
                       "l2": "inputs (>= 0.7 GB/step) exceed the 126 MB L2; no flush needed"},
            "roofline": {"bound": "hbm", "achieved": achieved, "peak": pk["hbm_gbs"], "unit": "GB/s",
                         "frac": achieved / pk["hbm_gbs"], "traffic": ncu_traffic(args.workload),
                         "kernel": "k_cm_agg (framing+decode+filter+aggregate)" if wl["family"] == "CM"
                         else "k_lr_agg", "peak_source": pk["source"] + " copy bandwidth (MEASURED_PEAKS.json)",
                         "algorithmic_bytes_per_launch": res["bytes_per_step"]},
            "batch_latency_ms": {"device_p50": 1e3 * pct(res["batch_s"], 50),
                                 "device_p99": 1e3 * pct(res["batch_s"], 99),
                                 "agg_kernel_mean": 1e3 * agg_avg,
                                 "close_kernel_mean": 1e3 * statistics.mean(res["close_s"])},
            "clocks": res["clocks"], "gpu_launches": res["launches"],
            "e2e": e2e, "cpu_baseline": cpu, "secondary": sec,
        }
        print(json.dumps(line))
    if world > 1:
        dist.barrier()
        dist.destroy_process_group()
    return 0


if __name__ == "__main__":
    sys.exit(main())
