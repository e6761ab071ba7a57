#!/bin/bash
# CM kernel iteration on the GPU: correctness (first-batch probe + CM parity tests), timings, one
# ncu --set full capture of k_cm_agg with the per-opcode / per-line instruction summary.
# Usage (under gpurun): bash tools/gpu_cm_iter.sh <tag>
TAG=${1:-cm_iter}
OUT=gpurun_out/$TAG
mkdir -p $OUT
timeout 300 python tools/cm_bad_probe.py > $OUT/probe.txt 2>&1; head -4 $OUT/probe.txt
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_dist.py tests/test_gpu_fullsize.py tests/test_gpu_parity_r02.py tests/test_gpu_churn.py -q -x -k "CM or cm" > $OUT/pytest.txt 2>&1; tail -3 $OUT/pytest.txt
{ for w in cm2 cm1; do echo "== $w"; timeout 300 python tools/prof_batch.py --workload $w --batches 6; done; } > $OUT/timings.txt 2>&1; cat $OUT/timings.txt | tail -14
timeout 600 ncu --set full --clock-control none --import-source on -k regex:k_cm_agg -s 2 -c 1 -o $OUT/cm2_agg python tools/prof_batch.py --workload cm2 --batches 3 > $OUT/ncu_cm2.log 2>&1
python tools/ncu_regions.py $OUT/cm2_agg.ncu-rep > $OUT/cm2_agg_opcodes.txt 2>&1; head -3 $OUT/cm2_agg_opcodes.txt; tail -12 $OUT/cm2_agg_opcodes.txt
python tools/ncu_lines.py $OUT/cm2_agg.ncu-rep 400 > $OUT/cm2_agg_lines.txt 2>&1
