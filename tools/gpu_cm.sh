#!/bin/bash
# Quick CM iteration on the GPU: CM parity tests, CM2 bench line, one ncu --set full capture.
TAG=${1:-cmx}
OUT=gpurun_out/$TAG
mkdir -p $OUT
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_dist.py tests/test_gpu_fullsize.py -q -x -k "CM or cm" > $OUT/pytest.txt 2>&1; tail -3 $OUT/pytest.txt
timeout 300 python bench.py --secondary '' --e2e-steps 0 --no-cpu-baseline > $OUT/bench.json 2> $OUT/bench.err; tail -2 $OUT/bench.err
python -c "import json;d=json.load(open('$OUT/bench.json'));print('value',d['value'],'agg_ms',d['batch_latency_ms']['agg_kernel_mean'],'frac',d['roofline']['frac'])"
timeout 600 ncu --set full --clock-control none --import-source on -k regex:k_cm_agg -s 2 -c 1 -o $OUT/cm2_agg python tools/prof_batch.py --workload cm2 --batches 3 > $OUT/ncu_cm2.log 2>&1
tail -2 $OUT/ncu_cm2.log
