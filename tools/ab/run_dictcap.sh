OUT=gpurun_out/dictcap; mkdir -p $OUT
for r in 1 2; do for mk in 1048576 2097152 4194304; do echo "== max_keys $mk"; timeout 300 python tools/prof_batch.py --workload lr1 --batches 7 --records 10000000 --flags 0 --max-keys $mk | tail -4; done; done > $OUT/dictcap.txt 2>&1
grep -E "==|batch [1-4]:" $OUT/dictcap.txt
