OUT=gpurun_out/ab3; mkdir -p $OUT
LIB=paper_2111_04289_b200/liblmstream.so
for v in A B A B; do cp tools/ab/liblmstream_$v.so $LIB; echo "== $v"; timeout 300 python tools/prof_batch.py --workload cm2 --batches 72 | tail -14; done > $OUT/close_ab.txt 2>&1
grep -E "==|rows 10000" $OUT/close_ab.txt | tail -24
cp tools/ab/liblmstream_B.so $LIB
timeout 1200 python -m pytest tests/test_gpu_parity.py tests/test_gpu_fullsize.py tests/test_gpu_parity_r02.py tests/test_gpu_churn.py tests/test_gpu_dist.py tests/test_gpu_group.py tests/test_gpu_sizer.py -q -x > $OUT/pytest.txt 2>&1; tail -3 $OUT/pytest.txt
