#!/usr/bin/env python
"""bench.py — LMStream micro-batch hot path on B200 (BASELINE.json metric).

metric: records/s (and HBM GB/s) per micro-batch for CM2 / LR2 10M-record batches; p99 batch
latency.  Headline workload = BASELINE config C4 (CM2S, B(10000): one 10M-record dataset per
second, one micro-batch per second, MANUAL batching); LR2S C4' is reported beside it.

  python bench.py [--gpus N] [--steps K] [--warmup W] [--impl reference] [--workload cm2|lr2]
                  [--scaling weak|strong] [--latency-batches 200]

A step = one micro-batch through the whole hot path via the C ABI: push (device-resident
input, borrowed), admission, Alg. 2 labels, framing/decode/filter/aggregate kernel, window
close kernel, batch report + result rows to the host.  `value` = records of all ranks / max
over ranks of the device-clock time of the K timed steps (CUDA events, synchronize + barrier
on both sides).  Before the warm-up an untimed fill of the window's R seconds (small batches)
puts the query in steady state: every pane of the window live, closes summing R/S panes.  Inputs (1.375 GB / 0.70 GB per step) exceed L2, so no L2 flush is needed.
`e2e` = same metric with the inputs in pinned HOST memory: lms_push_pinned (asynchronous H2D,
the next step's copy overlapping this step's kernels) + batch + rows to host per step.
Batch latency p50/p99 (nearest rank, lms_percentile) come from a separate loop of >= 200
micro-batches (device time per batch, and e2e Proc per batch with its H2D).
N > 1 (torchrun): weak scaling = every rank runs its own 10M-record partition per step;
strong scaling = one 10M-record micro-batch per step split across the ranks at record
boundaries by the library (lms_split).  DESIGN.md §7 describes the partial-aggregate merge.

The oracle (oracle/) runs only in the cpu_baseline leg and the --impl reference arm.
"""
from __future__ import annotations

import argparse
import gc
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
SPEC_HBM_GBS = 8000.0                  # the ~8 TB/s the north_star names (SURVEY §8(d) also asks for it)

WORKLOADS = {
    "cm2": dict(kind="CM2S", family="CM", traffic="B(10000)", records=10_000_000, rec_bytes=137.5,
                desc="CM2S C4: 10M-record micro-batches (B(10000), 1 batch = 1 s), J=1e4 jobIds, "
                     "eventType==1 selectivity 0.26, 130-145 B records"),
    "lr2": dict(kind="LR2S", family="LR", traffic="B(10000)", records=10_000_000, rec_bytes=70,
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

def gen_second_dev(wl, t, seed, rank, world, scaling, torch):
    """Second t of the workload on the device: (tensor, nbytes) of this rank's part.
    weak: the rank's own 10M-record second (per-rank seed); strong: the global 10M-record
    second (same seed on every rank) cut at record boundaries by lms_split, the rank's part
    copied into its own 16 B-aligned buffer (lms_push_device needs 16 B alignment)."""
    from lmsgen import cuda as gcu
    if scaling == "weak" or world == 1:
        buf, n = gcu.second_tensor(wl["family"], t, wl["records"], seed=seed + 7919 * rank)
        return buf, n
    from paper_2111_04289_b200.dist import split_points
    full, n = gcu.second_tensor(wl["family"], t, wl["records"], seed=seed)
    o, m = split_points(wl["family"], (full.data_ptr(), n), world)[rank]
    part = torch.empty(m + 64, dtype=torch.uint8, device="cuda")
    part[:m].copy_(full[o:o + m])
    torch.cuda.synchronize()
    return part, m


def make_query(wl, rank, world, pipeline, cap, torch):
    import paper_2111_04289_b200 as P
    from paper_2111_04289_b200 import _lib as L
    dev = torch.cuda.current_device()
    return P.Query(wl["kind"], mode="manual", device=dev, max_batch_bytes=cap, rank=rank, world=world,
                   flags=L.LMS_FLAG_PIPELINE if (pipeline and world == 1) else 0)


class Runner:
    """One lms_query (+ the multi-GPU protocol for N > 1) and its row draining."""

    def __init__(self, wl, rank, world, torch, p2p, pipeline, cap):
        import numpy as np
        import paper_2111_04289_b200 as P
        self.q = make_query(wl, rank, world, pipeline, cap, torch)
        self.world = world
        self.p2p = p2p
        self.rowbuf = np.zeros(1 << 16, P.AGG_DTYPE)      # caller-owned result buffer
        self.rowbuf.view(np.uint8)[:] = 1                 # (pages touched: np.zeros maps them lazily)
        if world > 1:
            from paper_2111_04289_b200.dist import RankHandle, TorchDistExchange
            self.h, self.ex = RankHandle(self.q), TorchDistExchange()
            if p2p and p2p != "dense":
                self.ex.setup_p2p([self.h], device_watermark=p2p == "device")

    def batch(self, t, sync):
        if self.world > 1:                    # partial aggregates merged by key owner
            from paper_2111_04289_b200.dist import run_batch
            run_batch([self.h], self.ex, float(t) + 1.0, p2p=self.p2p)
        else:
            self.q.force(float(t) + 1.0)      # pipelined: completes batch i-2 while i-1 runs
            if sync:
                self.q.sync()
        return self.drain()

    def drain(self):
        n = 0
        while True:                           # results to host, into a reused buffer
            rows = self.q.read_agg(out=self.rowbuf)
            n += len(rows)
            if len(rows) < len(self.rowbuf):
                return n


FILL_DIVISOR = 50   # window-fill batches carry 1/50 of a step's records


def fill_window(run, wl, seed, rank, world, scaling, torch, t_end, sync):
    """Untimed window fill: the R seconds before t_end as small micro-batches (every key of the
    workload still appears in every pane), so that the measured batches run in steady state —
    every pane of the window live, closes summing R/S panes — not while the window fills."""
    R = int(round(run.q.cfg.range_s))
    small = dict(wl, records=max(1, wl["records"] // FILL_DIVISOR))
    for t in range(t_end - R, t_end):
        buf, n = gen_second_dev(small, t, seed, rank, world, scaling, torch)
        run.q.push_device(buf.data_ptr(), n, float(t))
        run.batch(t, sync=True)
        del buf
    return R


def device_run(wl, steps, warmup, seed, rank, world, torch, dist, p2p, scaling, t0=100):
    """Throughput: K timed micro-batches, inputs resident in HBM (generated before timing), after
    an untimed window fill (seconds t0 - R .. t0 - 1) and W warm-up batches."""
    inputs = [(*gen_second_dev(wl, t, seed, rank, world, scaling, torch), t) for t in range(t0, t0 + warmup + steps)]
    torch.cuda.synchronize()
    run = Runner(wl, rank, world, torch, p2p, pipeline=True, cap=1 << 20)
    q = run.q
    nfill = fill_window(run, wl, seed, rank, world, scaling, torch, t0, sync=True)
    out = {"agg_s": [], "close_s": [], "batch_s": [], "rows": 0}
    for i in range(warmup):
        buf, n, t = inputs[i]
        q.push_device(buf.data_ptr(), n, float(t))
        run.batch(t, sync=False)
    q.sync()
    run.drain()
    launches0 = q.kernel_launches()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    dev = torch.cuda.current_device()
    gc.collect()
    gc.disable()                                     # no collector pause inside the timed steps
    with ClockSampler(dev) as clk:
        if world > 1:
            dist.barrier()
        torch.cuda.synchronize()
        clk.mark(True)
        e0.record()
        for i in range(warmup, warmup + steps):
            buf, n, t = inputs[i]
            q.push_device(buf.data_ptr(), n, float(t))
            out["rows"] += run.batch(t, sync=False)
            b, a, c = q.kernel_times()               # the most recently completed batch
            out["batch_s"].append(b)
            out["agg_s"].append(a)
            out["close_s"].append(c)
        q.sync()                                     # every timed batch complete, rows on the host
        out["rows"] += run.drain()
        e1.record()
        torch.cuda.synchronize()
        if world > 1:
            dist.barrier()
        clk.mark(False)
    gc.enable()
    out["elapsed_s"] = e0.elapsed_time(e1) / 1e3
    out["launches"] = q.kernel_launches() - launches0
    out["clocks"] = clk.summary()
    out["bytes_per_step"] = statistics.mean(n for _, n, _ in inputs[warmup:])
    recs = [q.record(nfill + i) for i in range(warmup, warmup + steps)]
    out["records"] = sum(r["num_records"] for r in recs)
    out["bad"] = sum(r["bad_records"] for r in recs)
    q.close()
    del inputs
    torch.cuda.empty_cache()
    return out


def latency_run(wl, n_batches, seed, rank, world, torch, dist, p2p, scaling, t0=1000):
    """Per-batch device time over n_batches micro-batches (serial: each batch completes before
    the next is admitted; second t's input generated on the GPU before it is pushed, outside the
    batch's device time).  N > 1: per batch the max over ranks."""
    run = Runner(wl, rank, world, torch, p2p, pipeline=False, cap=1 << 20)
    q = run.q
    fill_window(run, wl, seed, rank, world, scaling, torch, t0, sync=True)
    dev_s, agg_s = [], []
    for i in range(n_batches + 3):
        buf, n = gen_second_dev(wl, t0 + i, seed, rank, world, scaling, torch)
        q.push_device(buf.data_ptr(), n, float(t0 + i))
        run.batch(t0 + i, sync=True)
        if world > 1:
            q.sync()
        b, a, _ = q.kernel_times()
        if i >= 3:                                    # 3 warm-up batches
            dev_s.append(b)
            agg_s.append(a)
        del buf
    q.close()
    if world > 1:
        dev_s = max_over_ranks_vec(dev_s, torch, dist)
    return dev_s, agg_s


def e2e_run(wl, steps, warmup, seed, torch, rank, world, dist, p2p, scaling):
    """Inputs in pinned host memory; each step: lms_push_pinned (async H2D; the next step's copy
    is enqueued while this step's kernels run) + batch + rows to host.  N > 1: every rank pushes
    its own part; batches run the dist.py protocol; the time is the max over ranks."""
    import numpy as np
    n_sec = warmup + steps
    host = []
    for t in range(n_sec):
        buf, n = gen_second_dev(wl, t, seed, rank, world, scaling, torch)
        h = torch.empty(n, dtype=torch.uint8, pin_memory=True)
        h.copy_(buf[:n])
        host.append((h, n, t))
        del buf
    torch.cuda.synchronize()
    torch.cuda.empty_cache()
    cap = max(n for _, n, _ in host) + 4096
    run = Runner(wl, rank, world, torch, p2p, pipeline=False, cap=cap)
    q = run.q
    d2h = []

    def steps_(lo, hi):
        h, n, t = host[lo]
        q.push_pinned(h.data_ptr(), n, float(t))
        for i in range(lo, hi):
            _, _, t = host[i]
            if world > 1:
                from paper_2111_04289_b200.dist import run_batch
                # the dist protocol synchronises inside the batch: push the next step after it
                run_batch([run.h], run.ex, float(t) + 1.0, p2p=run.p2p)
                if i + 1 < hi:
                    h2, n2, t2 = host[i + 1]
                    q.push_pinned(h2.data_ptr(), n2, float(t2))
            else:
                q.force(float(t) + 1.0)
                if i + 1 < hi:                       # next step's H2D overlaps this batch
                    h2, n2, t2 = host[i + 1]
                    q.push_pinned(h2.data_ptr(), n2, float(t2))
                q.sync()
            d2h.append(run.drain() * 72 + 88)        # rows + the 88 B batch report

    steps_(0, warmup)
    if world > 1:
        dist.barrier()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    steps_(warmup, n_sec)
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


def e2e_latency_run(wl, n_batches, seed, torch, rank, world, dist, p2p, scaling, t0=5000):
    """Proc (admit -> rows on the host, its H2D included: reading R18) of n_batches serial
    micro-batches pushed from pinned host memory; two pinned buffers are refilled from the
    GPU generator between batches (outside Proc)."""
    import numpy as np
    from lmsgen import cuda as gcu
    cap = int(gcu.max_bytes(wl["family"], wl["records"]) + 4096)
    pinned = [torch.empty(cap, dtype=torch.uint8, pin_memory=True) for _ in range(2)]
    run = Runner(wl, rank, world, torch, p2p, pipeline=False, cap=cap)
    q = run.q
    proc = []
    for i in range(n_batches + 2):
        buf, n = gen_second_dev(wl, t0 + i, seed, rank, world, scaling, torch)
        h = pinned[i % 2]
        h[:n].copy_(buf[:n])
        del buf
        q.push_pinned(h.data_ptr(), n, float(t0 + i))
        run.batch(t0 + i, sync=True)
        if world > 1:
            q.sync()
        if i >= 2:
            proc.append(q.record(q.num_batches() - 1)["proc_s"])
    q.close()
    if world > 1:
        proc = max_over_ranks_vec(proc, torch, dist)
    return proc


def max_over_ranks(x, torch, dist):
    """Max of a host scalar over ranks (NCCL: a device tensor; gloo: a host tensor)."""
    return max_over_ranks_vec([x], torch, dist)[0]


def max_over_ranks_vec(xs, torch, dist):
    dev = "cuda" if dist.get_backend() == "nccl" else "cpu"
    t = torch.tensor([float(x) for x in xs], device=dev, dtype=torch.float64)
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    return [float(v) for v in t.cpu().tolist()]


def roofline(bytes_per_launch, launch_s, pk, kernel, traffic):
    achieved = bytes_per_launch / launch_s / 1e9
    return {"bound": "hbm", "achieved": achieved, "peak": pk["hbm_gbs"], "unit": "GB/s",
            "frac": achieved / pk["hbm_gbs"], "traffic": traffic, "kernel": kernel,
            "peak_source": pk["source"] + " copy bandwidth (MEASURED_PEAKS.json)",
            "peak_spec": SPEC_HBM_GBS, "frac_spec": achieved / SPEC_HBM_GBS,
            "algorithmic_bytes_per_launch": bytes_per_launch,
            "mean_launch_ms": 1e3 * launch_s}


# ----------------------------------------------------------------------------- CPU / reference arm
# The oracle (oracle/, stdlib Python) as it stands, on this host's cores: the paper's partition
# of a micro-batch into NumCores partitions — P = len(sched_getaffinity) worker processes
# each replay a contiguous record range, and the parent merges the partial (count, exact sum)
# per (window instance, key).  Exact for CM2S / CM1* (no HAVING); LR2S's HAVING is applied per
# partition (timing only).

_MC = {}


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


def host_info():
    cores = len(os.sched_getaffinity(0))
    model = None
    try:
        with open("/proc/cpuinfo") as fh:
            for line in fh:
                if line.startswith("model name"):
                    model = line.split(":", 1)[1].strip()
                    break
    except OSError:
        pass
    return {"cores": cores, "cpu_model": model}


def _cuts(fam, data: bytes, parts: int):
    n = len(data)
    cuts = [0]
    for r in range(1, parts):
        c = n * r // parts
        if fam == "LR":
            c -= c % 70
        else:
            j = data.find(b"\n", max(c - 1, 0))
            c = n if j < 0 else j + 1
        cuts.append(max(c, cuts[-1]))
    cuts.append(n)
    return cuts


def _mc_worker(i):
    from oracle import queries as Q
    d = _MC["data"]
    lo, hi = _MC["cuts"][i], _MC["cuts"][i + 1]
    outs = Q.replay(_MC["q"], [[d[lo:hi]]] if hi > lo else [])
    return [(r.win_start, r.win_end, r.key, r.count, r.sum_fixed) for o in outs for r in o.rows]


def cpu_multicore(kind, records, seed=211104289, t0=0, procs=None):
    """Oracle on `records` records (2 seconds of the workload) split over P processes."""
    import multiprocessing as mp
    from oracle import queries as Q
    fam = "CM" if kind.startswith("CM") else "LR"
    P = procs or len(os.sched_getaffinity(0))
    data = b"".join(_sample_datasets(fam, 2, records // 2, seed, t0))
    _MC.update(data=data, cuts=_cuts(fam, data, P), q=Q.query_spec(kind))
    ctx = mp.get_context("fork")
    with ctx.Pool(P) as pool:                       # workers forked before the timer
        pool.map(abs, range(P))
        t_start = time.perf_counter()
        parts = pool.map(_mc_worker, range(P), chunksize=1)
        merged = {}
        for rows in parts:                          # partition merge
            for ws, we, key, cnt, smf in rows:
                m = merged.setdefault((ws, key), [0, 0])
                m[0] += cnt
                m[1] += smf
        el = time.perf_counter() - t_start
    _MC.clear()
    return {"records": records, "bytes": len(data), "elapsed_s": el, "records_per_s": records / el,
            "rows": len(merged), "procs": P}


def cpu_single(kind, records, seed=211104289, t0=0):
    """The oracle single-threaded (parse + windows, Replay + flush) on `records` records."""
    from oracle import queries as Q
    fam = "CM" if kind.startswith("CM") else "LR"
    data = _sample_datasets(fam, 2, records // 2, seed, t0)
    q = Q.query_spec(kind)
    t_start = time.perf_counter()
    outs = Q.replay(q, [[d] for d in data])
    el = time.perf_counter() - t_start
    return {"records": records, "bytes": sum(map(len, data)), "elapsed_s": el, "records_per_s": records / el,
            "rows": sum(len(o.rows) for o in outs)}


def cpu_baseline(kind):
    info = host_info()
    P = info["cores"]
    single = cpu_single(kind, 600_000)                       # ~4 s of one core
    multi = cpu_multicore(kind, min(8_000_000, max(1_200_000, P * 150_000)))
    return {"value": multi["records_per_s"], "unit": "records/s", "cores": multi["procs"], "kind": "oracle",
            "sample": f"{multi['records']} records (2 seconds of the same generator) split into {multi['procs']} "
                      f"contiguous record ranges, one oracle process each, partial (count, sum) merge; "
                      f"{multi['elapsed_s']:.2f} s wall",
            "host": info,
            "single_core": {"value": single["records_per_s"], "unit": "records/s", "cores": 1,
                            "sample": f"{single['records']} records, {single['elapsed_s']:.2f} s"}}


METRIC = "records/s per micro-batch (CM2 10M-record batches); HBM GB/s; p99 batch latency"


def reference_arm(args, wl, rank, world):
    if rank != 0:
        return 0
    info = host_info()
    P = info["cores"]
    per_step = min(2_000_000, max(400_000, P * 40_000))
    for _ in range(args.warmup):
        cpu_multicore(wl["kind"], 200_000)
    per = [cpu_multicore(wl["kind"], per_step, t0=2 * i) for i in range(args.steps)]
    tot_r = sum(p["records"] for p in per)
    tot_t = sum(p["elapsed_s"] for p in per)
    v = tot_r / tot_t
    sample = (f"per step: {per_step} records (2 seconds of the same generator, seconds 2i, 2i+1) over "
              f"{P} oracle processes + partition merge")
    line = {"impl": "reference", "metric": METRIC,
            "value": v, "unit": "records/s", "n_gpus": world, "steps": args.steps, "warmup": args.warmup,
            "ms_per_step": 1e3 * tot_t / args.steps, "higher_is_better": True, "scaling": args.scaling,
            "vs_baseline": None, "dtype": "int64+f64 (Python)", "data": "synthetic (lmsgen, seeded)",
            "config": {"workload": wl["desc"], "records_per_batch_per_gpu": wl["records"],
                       "global_batch": wl["records"] * world,
                       "parallelism": f"oracle, {P} host processes", "sample": sample},
            "cpu_baseline": {"value": v, "unit": "records/s", "cores": P, "kind": "oracle", "sample": sample,
                             "host": info},
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
    ap.add_argument("--scaling", default="weak", choices=["weak", "strong"],
                    help="N > 1: weak = 10M records per rank per step; strong = 10M records per step "
                         "split across the ranks at record boundaries (lms_split)")
    ap.add_argument("--secondary", default="lr2", help="also measure this workload ('' = none)")
    ap.add_argument("--e2e-steps", type=int, default=5)
    ap.add_argument("--latency-batches", type=int, default=200,
                    help="micro-batches of the device-time p50/p99 loop (0 = skip)")
    ap.add_argument("--e2e-latency-batches", type=int, default=200,
                    help="micro-batches of the e2e Proc p50/p99 loop (0 = skip)")
    ap.add_argument("--seed", type=int, default=211104289)
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--exchange", default="auto", choices=["auto", "alltoall", "dense", "p2p", "p2p-async", "device"],
                    help="N > 1: partial-aggregate exchange (auto: dense for LR2 / CM1, alltoall for CM2; "
                         "NCCL all-to-all + owner merge; one SUM all-reduce of the dense [instances][K] "
                         "partials (LR2 / CM1); the fused peer-memory push into the owners' accumulators "
                         "with host-driven passes; or the same fully enqueued with a device-side barrier; "
                         "or also the watermark exchange on the device: no per-batch collective)")
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
        # NCCL's communicator setup (ranks, NVLink / NVLS transports) goes to stderr, so a
        # scaling run's log shows how many ranks each communicator had; stdout keeps the one
        # JSON line
        os.environ.setdefault("NCCL_DEBUG", "INFO")
        os.environ.setdefault("NCCL_DEBUG_SUBSYS", "INIT,NVLS")
        os.environ.setdefault("NCCL_DEBUG_FILE", "/dev/stderr")
        if backend == "nccl":
            dist.init_process_group("nccl", device_id=torch.device("cuda", local))
        else:
            dist.init_process_group(backend)
    import paper_2111_04289_b200 as P   # noqa: F401  (loads liblmstream.so; no fallback)
    pct = P.percentile                  # nearest rank, computed by the library

    scaling = args.scaling if world > 1 else "weak"
    def exchange_mode(w):
        choice = args.exchange
        if choice == "auto":
            choice = "dense" if w["kind"] in ("LR2S", "CM1S", "CM1T") else "alltoall"
        return {"alltoall": False, "dense": "dense", "p2p": True, "p2p-async": "async", "device": "device"}[choice]
    p2p = exchange_mode(wl)
    seed = args.seed
    res = device_run(wl, args.steps, args.warmup, seed, rank, world, torch, dist, p2p, scaling)
    el = res["elapsed_s"]
    if world > 1:
        el = max_over_ranks(el, torch, dist)
    recs = wl["records"] * (world if scaling == "weak" else 1) * args.steps
    value = recs / el
    pk = peaks()
    agg_avg = statistics.mean(res["agg_s"])
    lat = None
    if args.latency_batches > 0:
        dev_s, agg_s = latency_run(wl, args.latency_batches, seed, rank, world, torch, dist, p2p, scaling)
        lat = {"batches": len(dev_s), "device_p50": 1e3 * pct(dev_s, 50), "device_p99": 1e3 * pct(dev_s, 99),
               "device_max": 1e3 * max(dev_s), "agg_kernel_p50": 1e3 * pct(agg_s, 50),
               "agg_kernel_p99": 1e3 * pct(agg_s, 99),
               "note": "serial micro-batches (each completes before the next is admitted); N > 1: max over ranks per batch"}
    sec = None
    if args.secondary and args.secondary != args.workload:
        w2 = WORKLOADS[args.secondary]
        r2 = device_run(w2, args.steps, args.warmup, seed, rank, world, torch, dist, exchange_mode(w2),
                        scaling)
        if world > 1:
            r2["elapsed_s"] = max_over_ranks(r2["elapsed_s"], torch, dist)
        a2 = statistics.mean(r2["agg_s"])
        n2 = len(r2["agg_s"])
        sec = {"workload": w2["desc"],
               "records_per_s": w2["records"] * (world if scaling == "weak" else 1) * n2 / r2["elapsed_s"],
               "ms_per_step": 1e3 * r2["elapsed_s"] / n2,
               "roofline": roofline(r2["bytes_per_step"], a2, pk, "k_lr_agg<LR2S> (framing+validation+decode+aggregate)",
                                    ncu_traffic(args.secondary)),
               "batch_device_ms_p50": 1e3 * pct(r2["batch_s"], 50),
               "close_kernel_ms_mean": 1e3 * statistics.mean(r2["close_s"]),
               "clocks": r2["clocks"], "gpu_launches": r2["launches"]}
        if args.latency_batches > 0:
            d2, _ = latency_run(w2, args.latency_batches, seed, rank, world, torch, dist, exchange_mode(w2), scaling)
            sec["batch_latency_ms"] = {"batches": len(d2), "device_p50": 1e3 * pct(d2, 50),
                                       "device_p99": 1e3 * pct(d2, 99)}
    e2e = None
    if args.e2e_steps > 0:
        e = e2e_run(wl, args.e2e_steps, 1, seed, torch, rank, world, dist, p2p, scaling)
        e2e = {"value": wl["records"] * (world if scaling == "weak" else 1) * args.e2e_steps / e["elapsed_s"],
               "unit": "records/s",
               "h2d_bytes_per_step": e["h2d_bytes_per_step"], "d2h_bytes_per_step": e["d2h_bytes_per_step"],
               "steps": args.e2e_steps, "h2d_ms_mean": 1e3 * statistics.mean(e["h2d_s"]),
               # the e2e leg is bound by the host link: its achieved pinned H2D bandwidth
               "h2d_gbs": e["h2d_bytes_per_step"] / statistics.mean(e["h2d_s"]) / 1e9,
               "api": "lms_push_pinned (async H2D, next step's copy overlapping this step's kernels) + "
                      "lms_force_batch + lms_sync + lms_read_agg"}
        if args.e2e_latency_batches > 0:
            proc = e2e_latency_run(wl, args.e2e_latency_batches, seed, torch, rank, world, dist, p2p, scaling)
            e2e["proc_latency_ms"] = {"batches": len(proc), "p50": 1e3 * pct(proc, 50), "p99": 1e3 * pct(proc, 99),
                                      "note": "Proc = admit -> rows on the host, H2D included (reading R18)"}
    cpu = None
    if rank == 0 and not args.no_cpu_baseline and world == 1:
        cpu = cpu_baseline(wl["kind"])
    if rank == 0:
        line = {
            "metric": METRIC,
            "value": value, "unit": "records/s", "n_gpus": world, "steps": args.steps, "warmup": args.warmup,
            "ms_per_step": 1e3 * el / args.steps, "higher_is_better": True, "scaling": scaling,
            "vs_baseline": None, "dtype": "u64 fixed-point sums + f64 AVG", "data": "synthetic (lmsgen, seeded)",
            "config": {"workload": wl["desc"], "records_per_batch_per_gpu":
                       wl["records"] if scaling == "weak" else wl["records"] / world,
                       "global_batch": wl["records"] * (world if scaling == "weak" else 1),
                       "batch_bytes_per_gpu": res["bytes_per_step"],
                       "parallelism": (f"dp{world} (row partition per rank, {scaling} scaling; exchange: {args.exchange})"
                                       if world > 1 else "single GPU"),
                       "l2": "inputs (>= 0.7 GB/step) exceed the 126 MB L2; no flush needed",
                       "window": "steady state: an untimed fill of the R seconds before the first warm-up batch "
                                 f"(1/{FILL_DIVISOR} of a step's records per second) leaves every pane of the "
                                 "window live, so closing batches sum R/S panes"},
            "roofline": roofline(res["bytes_per_step"], agg_avg, pk,
                                 "k_cm_agg<CM2S> (framing+decode+filter+aggregate)" if wl["family"] == "CM"
                                 else "k_lr_agg<LR2S>", ncu_traffic(args.workload)),
            "batch_latency_ms": dict(lat or {}, agg_kernel_mean_timed=1e3 * agg_avg,
                                     close_kernel_mean_timed=1e3 * statistics.mean(res["close_s"])),
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
