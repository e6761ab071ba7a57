#!/bin/bash
# One GPU call: sizer tests (async Eq. 10 refit), f2 calibration sweep, f3 dynamics (A: model-based
# violation tables from the fresh calibration, B: real-GPU LR1S/LR1T timelines).
# Usage (under gpurun): bash tools/gpu_f2f3.sh <tag>
set -u
TAG=${1:-r02c}
OUT=gpurun_out/$TAG
mkdir -p $OUT
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,clocks_event_reasons.active --format=csv > $OUT/nvsmi.txt 2>&1
timeout 600 python -m pytest tests/test_gpu_sizer.py tests/test_abi.py -q -x > $OUT/pytest_sizer.txt 2>&1; tail -2 $OUT/pytest_sizer.txt
timeout 900 python tools/calibrate_b200.py --out $OUT/calibration.json > $OUT/calibration.log 2>&1; tail -3 $OUT/calibration.log
timeout 1200 python tools/f3_dynamics.py --calib $OUT/calibration.json --part AB --out $OUT/f3_dynamics.json > $OUT/f3.log 2>&1; tail -8 $OUT/f3.log
ls -la $OUT
