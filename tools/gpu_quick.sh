#!/bin/bash
# One GPU call: new tests first, then the whole GPU suite, smoke, bench.
# Usage (under gpurun): bash tools/gpu_quick.sh <tag> [pytest -k expr]
set -u
TAG=${1:-r02}
OUT=gpurun_out/$TAG
mkdir -p $OUT
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv > $OUT/nvsmi.txt 2>&1
timeout 900 python -m pytest tests/test_gpu_parity_r02.py -q -x > $OUT/pytest_r02.txt 2>&1; tail -3 $OUT/pytest_r02.txt
timeout 1500 python -m pytest tests -q -m gpu > $OUT/pytest_gpu.txt 2>&1; tail -3 $OUT/pytest_gpu.txt
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > $OUT/smoke.txt 2>&1; tail -2 $OUT/smoke.txt
timeout 900 python bench.py --steps 20 --warmup 5 > $OUT/bench.json 2> $OUT/bench.err; tail -3 $OUT/bench.err; cat $OUT/bench.json
timeout 600 python bench.py --impl reference --steps 3 --warmup 3 > $OUT/bench_ref.json 2> $OUT/bench_ref.err; tail -3 $OUT/bench_ref.err; cat $OUT/bench_ref.json
