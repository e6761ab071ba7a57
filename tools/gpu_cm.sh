#!/bin/bash
# Quick CM iteration on the GPU: CM parity tests, kernel timings, one ncu --set full capture.
# Usage (under gpurun): bash tools/gpu_cm.sh <tag> [skip-tests]
TAG=${1:-cmx}
OUT=gpurun_out/$TAG
mkdir -p $OUT
if [ "${2:-}" != "skip-tests" ]; then
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_dist.py tests/test_gpu_fullsize.py -q -x -k "CM or cm" > $OUT/pytest.txt 2>&1; tail -3 $OUT/pytest.txt
fi
{ for w in cm2 cm1; do echo "== $w"; timeout 300 python tools/prof_batch.py --workload $w --batches 6; done; } > $OUT/timings.txt 2>&1; cat $OUT/timings.txt | tail -12
timeout 600 ncu --set full --clock-control none --import-source on -k regex:k_cm_agg -s 2 -c 1 -o $OUT/cm2_agg python tools/prof_batch.py --workload cm2 --batches 3 > $OUT/ncu_cm2.log 2>&1
tail -2 $OUT/ncu_cm2.log
python tools/ncu_regions.py $OUT/cm2_agg.ncu-rep > $OUT/cm2_agg_opcodes.txt 2>&1; cat $OUT/cm2_agg_opcodes.txt | head -40
