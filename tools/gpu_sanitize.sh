#!/bin/bash
# compute-sanitizer memcheck / racecheck / synccheck over a parity subset that exercises every
# kernel path (CM fast + general decode, malformed records, LR, LR1, close, multi-GPU kernels).
OUT=gpurun_out/${1:-sanitizer}
mkdir -p $OUT
SEL='tests/test_gpu_parity.py::test_cm_fast_path_fuzz tests/test_gpu_parity.py::test_malformed_records_counted_and_dropped tests/test_gpu_parity.py::test_cm_field_shape_variants tests/test_gpu_parity.py::test_empty_flush_and_tiny_batches tests/test_gpu_parity.py::test_many_segments_more_than_one_launch tests/test_gpu_dist.py::test_virtual_shards_lr1_match_oracle tests/test_gpu_parity.py::test_cm_mixed_panes_in_warp_rounds tests/test_gpu_parity.py::test_parity_streams[LR1S-B(0.4)-40-bs6] tests/test_gpu_parity.py::test_parity_streams[LR1T-B(0.3)-65-bs7] tests/test_gpu_parity.py::test_pipelined_batches_equal_serial tests/test_gpu_parity.py::test_parity_streams[CM2S-R(0.1,1)-66-bs3] tests/test_gpu_parity_r02.py::test_lr2_periodic_table_flush'
for tool in memcheck synccheck racecheck; do
  timeout 1500 compute-sanitizer --tool $tool --print-limit 20 python -m pytest $SEL -q -x \
    > $OUT/$tool.txt 2>&1
  timeout 1500 compute-sanitizer --tool $tool --print-limit 20 python -m pytest -q -x \
    "tests/test_gpu_dist.py::test_virtual_shards_match_oracle[CM2S-B(1.3)-2-p2p]" \
    "tests/test_gpu_dist.py::test_virtual_shards_match_oracle[LR2S-B(1.7)-2-alltoall]" \
    "tests/test_gpu_group.py::test_group_parity_streams[LR1S-B(0.4)-40-bs5-2]" \
    "tests/test_gpu_group.py::test_group_parity_streams[CM1S-B(0.9)-75-bs3-2]" >> $OUT/$tool.txt 2>&1
  timeout 1500 compute-sanitizer --tool $tool --print-limit 20 python -m pytest -q -x tests/test_gpu_churn.py >> $OUT/$tool.txt 2>&1
  tail -3 $OUT/$tool.txt
done
