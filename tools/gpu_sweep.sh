#!/bin/bash
# CM2 aggregate kernel across the SURVEY §8(d) sweeps: key cardinality J and selectivity.
OUT=gpurun_out/${1:-sweep}
mkdir -p $OUT
: > $OUT/sweep.txt
for cfg in "--jobs 100" "--jobs 10000" "--jobs 1000000 --max-keys 1048576" "--sel-ppm 10000" "--sel-ppm 1000000"; do
  echo "== CM2 $cfg" >> $OUT/sweep.txt
  timeout 300 python tools/prof_batch.py --workload cm2 --batches 4 $cfg 2>&1 | tail -2 >> $OUT/sweep.txt
done
cat $OUT/sweep.txt
