OUT=gpurun_out/ab11; mkdir -p $OUT
LIB=paper_2111_04289_b200/liblmstream.so
for v in J K J K J K J K; do cp tools/ab/liblmstream_$v.so $LIB; echo "== $v"; python tools/step_probe.py --steps 60 2>/dev/null | head -1; done > $OUT/steps.txt 2>&1
cat $OUT/steps.txt
cp tools/ab/liblmstream_K.so $LIB
timeout 300 python tools/cm_bad_probe.py > $OUT/probe.txt 2>&1; head -3 $OUT/probe.txt
timeout 1200 python -m pytest tests/test_gpu_parity.py tests/test_gpu_fullsize.py tests/test_gpu_parity_r02.py tests/test_gpu_churn.py -q -x -k "CM or cm" > $OUT/pytest.txt 2>&1; tail -2 $OUT/pytest.txt
