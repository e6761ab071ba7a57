#!/bin/bash
# CM correctness probe on the GPU: first-batch bad-record probe (CM1S / CM2S, 3 reps) + CM tests.
# Usage (under gpurun): bash tools/gpu_cm_probe.sh
OUT=gpurun_out/${1:-cm_probe}; mkdir -p $OUT
timeout 300 python tools/cm_bad_probe.py > $OUT/probe.txt 2>&1; cat $OUT/probe.txt
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_dist.py tests/test_gpu_fullsize.py tests/test_gpu_parity_r02.py tests/test_gpu_churn.py -q -x -k "CM or cm" > $OUT/pytest.txt 2>&1; tail -3 $OUT/pytest.txt
