#!/bin/bash
# A/B: LR2 CTA tables added straight into the accumulators (default) vs per-CTA partials merged
# by the close (LMS_LR2_PARTIALS=1); plus LR2 parity tests.
OUT=gpurun_out/${1:-ab_lr2}; mkdir -p $OUT
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_dist.py tests/test_gpu_fullsize.py -q -x -k "LR2" > $OUT/pytest.txt 2>&1; tail -2 $OUT/pytest.txt
for i in 1 2; do for v in direct partials; do
  if [ $v = partials ]; then export LMS_LR2_PARTIALS=1; else unset LMS_LR2_PARTIALS; fi
  timeout 600 python bench.py --workload lr2 --secondary '' --e2e-steps 0 --no-cpu-baseline --latency-batches 200 --e2e-latency-batches 0 > $OUT/bench_$v$i.json 2>/dev/null
  python -c "
import json; b=json.load(open('$OUT/bench_$v$i.json')); print('$v', round(b['value']/1e9,2), round(b['ms_per_step'],4), round(b['batch_latency_ms']['agg_kernel_mean_timed'],4), round(b['batch_latency_ms']['close_kernel_mean_timed'],4), round(b['batch_latency_ms']['device_p50'],4))"
done; done
unset LMS_LR2_PARTIALS
timeout 300 python tools/prof_batch.py --workload lr1 --batches 6 --records 10000000 --flags 0 > $OUT/lr1_dict.txt 2>&1; grep "batch [2-4]" $OUT/lr1_dict.txt
