#!/bin/bash
# NVLS path on the GPU: multicast probe, group tests (NVLS + owner push), C2 latency config.
OUT=gpurun_out/${1:-nvls}; mkdir -p $OUT
./tools/microbench/mc_probe > $OUT/mc_probe.txt 2>&1; cat $OUT/mc_probe.txt
timeout 900 python -m pytest tests/test_gpu_group.py tests/test_gpu_churn.py -q -x > $OUT/pytest_group.txt 2>&1; tail -15 $OUT/pytest_group.txt
timeout 600 python tools/latency_configs.py --configs C2 --out $OUT/latency_c2.json > $OUT/c2.log 2>&1; python -c "
import json; r=json.load(open('$OUT/latency_c2.json'))['results'][0]; print(r['proc_ms'], r['device_ms'], r['proc_p99_over_p50']); print([round(x,3) for x in r['per_batch']['device_ms']])"
