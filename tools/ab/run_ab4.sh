OUT=gpurun_out/ab4; mkdir -p $OUT
LIB=paper_2111_04289_b200/liblmstream.so
for v in A B C A B C; do cp tools/ab/liblmstream_$v.so $LIB; echo "== $v"; timeout 300 python tools/prof_batch.py --workload cm2 --batches 72 | tail -14; done > $OUT/close_ab.txt 2>&1
grep -E "==|rows 10000|batch 71" $OUT/close_ab.txt | tail -30
cp tools/ab/liblmstream_C.so $LIB
timeout 1200 python -m pytest tests/test_gpu_parity.py tests/test_gpu_fullsize.py tests/test_gpu_churn.py tests/test_gpu_dist.py tests/test_gpu_group.py -q -x > $OUT/pytest.txt 2>&1; tail -3 $OUT/pytest.txt
timeout 600 ncu --set full --clock-control none --import-source on -k regex:k_close_agg -s 65 -c 1 -o $OUT/cm2_close python tools/prof_batch.py --workload cm2 --batches 67 --records 2000000 > $OUT/ncu.log 2>&1; tail -2 $OUT/ncu.log
python tools/ncu_lines.py $OUT/cm2_close.ncu-rep 40 > $OUT/cm2_close_lines.txt 2>&1; head -20 $OUT/cm2_close_lines.txt
