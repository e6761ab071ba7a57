#!/bin/bash
# Per-kind kernel timings (10M-record batches) + ncu captures of the LR1 / CM1 kernels.
OUT=gpurun_out/${1:-kinds}
mkdir -p $OUT
for w in cm1 lr2 cm2; do
  echo "== $w" >> $OUT/timings.txt
  timeout 300 python tools/prof_batch.py --workload $w --batches 4 >> $OUT/timings.txt 2>&1
done
for fl in 0 4; do   # LR1 with the key dictionary / with LMS_FLAG_DENSE_VEHICLES; 2M-record batches
  echo "== lr1 flags=$fl (2M records per batch)" >> $OUT/timings.txt
  timeout 300 python tools/prof_batch.py --workload lr1 --batches 4 --records 2000000 --flags $fl >> $OUT/timings.txt 2>&1
done
timeout 600 ncu --set full --clock-control none -k regex:k_lr_agg -s 2 -c 1 -o $OUT/lr1_agg python tools/prof_batch.py --workload lr1 --batches 3 --records 2000000 > $OUT/ncu_lr1.log 2>&1
timeout 600 ncu --set full --clock-control none -k regex:k_lr_agg -s 2 -c 1 -o $OUT/lr1d_agg python tools/prof_batch.py --workload lr1 --batches 3 --records 2000000 --flags 4 > $OUT/ncu_lr1d.log 2>&1
timeout 600 ncu --set full --clock-control none -k regex:k_close_lr1 -s 2 -c 1 -o $OUT/lr1_close python tools/prof_batch.py --workload lr1 --batches 3 --records 2000000 > $OUT/ncu_lr1c.log 2>&1
timeout 600 ncu --set full --clock-control none -k regex:k_cm_agg -s 2 -c 1 -o $OUT/cm1_agg python tools/prof_batch.py --workload cm1 --batches 3 > $OUT/ncu_cm1.log 2>&1
cat $OUT/timings.txt
