"""Probe of bench.py's pipelined throughput loop: per-step host time and device step time, with
and without the window fill (diagnostic for the step overhead).

  python tools/step_probe.py [--no-fill] [--steps 20]
"""
import argparse
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import bench  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--no-fill", action="store_true")
ap.add_argument("--steps", type=int, default=20)
ap.add_argument("--workload", default="cm2")
a = ap.parse_args()
wl = bench.WORKLOADS[a.workload]
seed, t0, W = 211104289, 100, 3
inputs = [(*bench.gen_second_dev(wl, t, seed, 0, 1, "weak", torch), t) for t in range(t0, t0 + W + a.steps)]
torch.cuda.synchronize()
run = bench.Runner(wl, 0, 1, torch, False, pipeline=True, cap=1 << 20)
q = run.q
if not a.no_fill:
    bench.fill_window(run, wl, seed, 0, 1, "weak", torch, t0, sync=True)
for i in range(W):
    buf, n, t = inputs[i]
    q.push_device(buf.data_ptr(), n, float(t))
    run.batch(t, sync=False)
q.sync()
run.drain()
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
torch.cuda.synchronize()
e0.record()
host = []
for i in range(W, W + a.steps):
    h0 = time.perf_counter()
    buf, n, t = inputs[i]
    q.push_device(buf.data_ptr(), n, float(t))
    h1 = time.perf_counter()
    q.force(float(t) + 1.0)
    h2 = time.perf_counter()
    nrows = run.drain()
    h3 = time.perf_counter()
    b, ag, c = q.kernel_times()
    host.append((time.perf_counter() - h0, b, ag, c, h1 - h0, h2 - h1, h3 - h2, nrows))
q.sync()
run.drain()
e1.record()
torch.cuda.synchronize()
el = e0.elapsed_time(e1) / a.steps
print(f"fill={not a.no_fill} ms/step {el:.4f}", flush=True)
for i, (h, b, ag, c, hp, hf, hd, nr) in enumerate(host):
    try:
        print(f"step {i}: host {h * 1e3:.3f} ms (push {hp * 1e3:.3f} force {hf * 1e3:.3f} drain {hd * 1e3:.3f}, "
              f"{nr} rows)  batch {b * 1e3:.3f} agg {ag * 1e3:.3f} close {c * 1e3:.3f}")
    except BrokenPipeError:                       # (piped into head)
        break
q.close()
