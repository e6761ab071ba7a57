#!/bin/bash
# Dense exchange tests (virtual shards + torchrun), CM racecheck subset, CM timings.
OUT=gpurun_out/${1:-dense_race}; mkdir -p $OUT
timeout 900 python -m pytest tests/test_gpu_dist.py -q -x -k "dense" > $OUT/pytest_dense.txt 2>&1; tail -2 $OUT/pytest_dense.txt
timeout 900 python -m pytest tests/test_gpu_torchrun.py -q -x -k "dense or auto" > $OUT/pytest_torchrun.txt 2>&1; tail -2 $OUT/pytest_torchrun.txt
timeout 900 compute-sanitizer --tool racecheck --print-limit 10 python -m pytest -q -x tests/test_gpu_parity.py::test_cm_fast_path_fuzz tests/test_gpu_parity.py::test_many_segments_more_than_one_launch tests/test_gpu_parity.py::test_cm_field_shape_variants tests/test_gpu_parity.py::test_empty_flush_and_tiny_batches > $OUT/racecheck_cm.txt 2>&1; tail -2 $OUT/racecheck_cm.txt
{ for w in cm2 cm1; do echo "== $w"; timeout 300 python tools/prof_batch.py --workload $w --batches 6; done; } > $OUT/timings.txt 2>&1; grep "batch [3-5]" $OUT/timings.txt
