#!/bin/bash
# CM iteration + bench: correctness probe, CM parity tests, full sizer/group tests, bench.
OUT=gpurun_out/${1:-cm_bench}; mkdir -p $OUT
timeout 300 python tools/cm_bad_probe.py > $OUT/probe.txt 2>&1; head -3 $OUT/probe.txt
timeout 1500 python -m pytest tests -q -x -m gpu > $OUT/pytest_gpu.txt 2>&1; tail -2 $OUT/pytest_gpu.txt
timeout 900 python bench.py > $OUT/bench.json 2> $OUT/bench.err; tail -2 $OUT/bench.err; python -c "
import json; b=json.load(open('$OUT/bench.json')); print(b['value'], b['ms_per_step'], b['roofline']['frac'], b['batch_latency_ms']['agg_kernel_mean_timed'], b['batch_latency_ms']['close_kernel_mean_timed'], b['secondary']['ms_per_step'])"
