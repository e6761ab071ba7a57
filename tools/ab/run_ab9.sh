OUT=gpurun_out/ab9; mkdir -p $OUT
LIB=paper_2111_04289_b200/liblmstream.so
for v in F G F G; do cp tools/ab/liblmstream_$v.so $LIB; echo "== $v"; timeout 300 python tools/prof_batch.py --workload cm2 --batches 72 | grep -E "rows 10000" | tail -3; python tools/step_probe.py --steps 40 | head -1; done > $OUT/ab.txt 2>&1
cat $OUT/ab.txt
for v in F G F G; do cp tools/ab/liblmstream_$v.so $LIB; echo "== $v cm2 J=1e6"; timeout 300 python tools/prof_batch.py --workload cm2 --batches 4 --jobs 1000000 --max-keys 1048576 | tail -2; done > $OUT/j1e6.txt 2>&1
cat $OUT/j1e6.txt
cp tools/ab/liblmstream_G.so $LIB
timeout 1200 python -m pytest tests/test_gpu_parity.py tests/test_gpu_fullsize.py tests/test_gpu_churn.py tests/test_gpu_dist.py tests/test_gpu_group.py tests/test_gpu_sizer.py -q -x > $OUT/pytest.txt 2>&1; tail -2 $OUT/pytest.txt
