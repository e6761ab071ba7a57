#!/bin/bash
# One GPU call: tests, smoke, bench, ncu launch list + full captures of the dominant kernels,
# stream-latency configs and the f3 timelines.
# Usage (under gpurun): bash tools/gpu_round.sh <tag>
set -u
TAG=${1:-r02j}
OUT=gpurun_out/$TAG
mkdir -p $OUT
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,clocks_event_reasons.active,clocks_event_reasons.hw_slowdown,clocks_event_reasons.sw_power_cap --format=csv > $OUT/nvsmi.txt 2>&1
timeout 1500 python -m pytest tests -q -m gpu > $OUT/pytest_gpu.txt 2>&1; tail -3 $OUT/pytest_gpu.txt
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > $OUT/smoke.txt 2>&1; tail -2 $OUT/smoke.txt
timeout 900 python bench.py > $OUT/bench.json 2> $OUT/bench.err; tail -2 $OUT/bench.err; cat $OUT/bench.json
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $OUT/launches_cm2.csv python bench.py --steps 2 --warmup 3 --secondary '' --e2e-steps 0 --no-cpu-baseline > /dev/null 2>&1
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $OUT/launches_lr2.csv python bench.py --workload lr2 --steps 2 --warmup 3 --secondary '' --e2e-steps 0 --no-cpu-baseline > /dev/null 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_cm_agg -s 2 -c 1 -o $OUT/cm2_agg python tools/prof_batch.py --workload cm2 --batches 3 > $OUT/ncu_cm2.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_lr_agg -s 2 -c 1 -o $OUT/lr2_agg python tools/prof_batch.py --workload lr2 --batches 3 > $OUT/ncu_lr2.log 2>&1
timeout 600 ncu --set full --clock-control none -k regex:k_close -s 2 -c 1 -o $OUT/lr2_close python tools/prof_batch.py --workload lr2 --batches 3 > $OUT/ncu_lr2c.log 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:k_close_agg -s 65 -c 1 -o $OUT/cm2_close python tools/prof_batch.py --workload cm2 --batches 67 --records 2000000 > $OUT/ncu_cm2c.log 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:k_lr1_agg -s 3 -c 1 -o $OUT/lr1_agg python tools/prof_batch.py --workload lr1 --batches 5 --records 10000000 --flags 4 > $OUT/ncu_lr1.log 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:k_lr1_agg -s 3 -c 1 -o $OUT/lr1_agg_dict python tools/prof_batch.py --workload lr1 --batches 5 --records 10000000 --flags 0 > $OUT/ncu_lr1d.log 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:k_close_lr1 -s 5 -c 1 -o $OUT/lr1_close python tools/prof_batch.py --workload lr1 --batches 7 --records 10000000 --flags 4 > $OUT/ncu_lr1c.log 2>&1
{ for w in cm2 cm1 lr2; do echo "== $w"; timeout 300 python tools/prof_batch.py --workload $w --batches 4; done
  for f in 0 4; do echo "== lr1 flags=$f (10M records per batch; batch 5 closes the first instance)"; timeout 300 python tools/prof_batch.py --workload lr1 --batches 7 --records 10000000 --flags $f; done; } > $OUT/kernel_timings_by_kind.txt 2>&1
timeout 1200 python tools/latency_configs.py --out $OUT/latency_configs.json > $OUT/latency_configs.log 2>&1; tail -6 $OUT/latency_configs.log
timeout 1500 python tools/f3_dynamics.py --part B --out $OUT/f3_timelines.json > $OUT/f3b.log 2>&1; tail -6 $OUT/f3b.log
timeout 900 python bench.py --impl reference --steps 3 --warmup 3 > $OUT/bench_ref.json 2> $OUT/bench_ref.err; cat $OUT/bench_ref.json
ls -la $OUT
