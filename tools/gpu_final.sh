#!/bin/bash
# End-of-session check: the GPU suite, smoke, bench, the launch list and ncu captures of the
# kernels changed last (LR aggregate kernels).  Usage (under gpurun): bash tools/gpu_final.sh <tag>
OUT=gpurun_out/${1:-final}; mkdir -p $OUT
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv > $OUT/nvsmi.txt 2>&1
timeout 1800 python -m pytest tests -q -m gpu > $OUT/pytest_gpu.txt 2>&1; tail -2 $OUT/pytest_gpu.txt
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > $OUT/smoke.txt 2>&1; tail -1 $OUT/smoke.txt
timeout 900 python bench.py > $OUT/bench.json 2> $OUT/bench.err; tail -2 $OUT/bench.err
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $OUT/launches_cm2.csv python bench.py --steps 2 --warmup 3 --secondary '' --e2e-steps 0 --no-cpu-baseline --latency-batches 0 --e2e-latency-batches 0 > /dev/null 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_cm_agg -s 2 -c 1 -o $OUT/cm2_agg python tools/prof_batch.py --workload cm2 --batches 3 > $OUT/ncu_cm2.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_lr_agg -s 2 -c 1 -o $OUT/lr2_agg python tools/prof_batch.py --workload lr2 --batches 3 > $OUT/ncu_lr2.log 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:k_lr1_agg -s 3 -c 1 -o $OUT/lr1_agg python tools/prof_batch.py --workload lr1 --batches 5 --records 10000000 --flags 4 > $OUT/ncu_lr1.log 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:k_lr1_agg -s 3 -c 1 -o $OUT/lr1_agg_dict python tools/prof_batch.py --workload lr1 --batches 5 --records 10000000 --flags 0 > $OUT/ncu_lr1d.log 2>&1
timeout 600 python bench.py --impl reference --steps 3 --warmup 3 > $OUT/bench_ref.json 2> $OUT/bench_ref.err
ls $OUT
