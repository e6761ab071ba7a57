OUT=gpurun_out/ab8; mkdir -p $OUT
LIB=paper_2111_04289_b200/liblmstream.so
for v in E F E F E F; do cp tools/ab/liblmstream_$v.so $LIB; echo "== $v"; python tools/step_probe.py --steps 40 | head -1; python tools/step_probe.py --steps 40 --workload lr2 | head -1; done > $OUT/steps.txt 2>&1
cat $OUT/steps.txt
for v in E F E F; do cp tools/ab/liblmstream_$v.so $LIB; for f in 0 4; do echo "== $v lr1 flags=$f"; timeout 300 python tools/prof_batch.py --workload lr1 --batches 7 --records 10000000 --flags $f | tail -3; done; done > $OUT/lr1.txt 2>&1
cat $OUT/lr1.txt
cp tools/ab/liblmstream_F.so $LIB
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_parity_r02.py tests/test_gpu_churn.py tests/test_gpu_fullsize.py tests/test_gpu_dist.py -q -x > $OUT/pytest.txt 2>&1; tail -2 $OUT/pytest.txt
