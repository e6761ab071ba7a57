#!/bin/bash
# LR1 kernel iteration on the GPU: LR1 parity tests, 10M-record timings (dictionary / dense
# vehicle ids), ncu --set full of the LR1 aggregate (both modes) and the closing probe.
# Usage (under gpurun): bash tools/gpu_lr1_iter.sh <tag> [skip-tests]
TAG=${1:-lr1_iter}
OUT=gpurun_out/$TAG
mkdir -p $OUT
if [ "${2:-}" != "skip-tests" ]; then
timeout 1200 python -m pytest tests -q -x -m gpu -k "LR1 or lr1" > $OUT/pytest.txt 2>&1; tail -3 $OUT/pytest.txt
fi
{ for f in 0 4; do echo "== lr1 flags=$f (10M records per batch; batch 5 closes the first instance)"; timeout 300 python tools/prof_batch.py --workload lr1 --batches 8 --records 10000000 --flags $f; done; } > $OUT/timings.txt 2>&1; cat $OUT/timings.txt
for f in 0 4; do
timeout 600 ncu --set full --clock-control none --import-source on -k regex:k_lr1?_agg -s 3 -c 1 -o $OUT/lr1_agg_f$f python tools/prof_batch.py --workload lr1 --batches 5 --records 10000000 --flags $f > $OUT/ncu_lr1_f$f.log 2>&1
python tools/ncu_regions.py $OUT/lr1_agg_f$f.ncu-rep 19531 > $OUT/lr1_agg_f${f}_opcodes.txt 2>&1; tail -12 $OUT/lr1_agg_f${f}_opcodes.txt
done
timeout 600 ncu --set full --clock-control none --import-source on -k regex:k_close_lr1 -s 5 -c 1 -o $OUT/lr1_close python tools/prof_batch.py --workload lr1 --batches 7 --records 10000000 --flags 4 > $OUT/ncu_lr1c.log 2>&1
python tools/ncu_regions.py $OUT/lr1_close.ncu-rep 19531 > $OUT/lr1_close_opcodes.txt 2>&1; tail -12 $OUT/lr1_close_opcodes.txt
