OUT=gpurun_out/ab7; mkdir -p $OUT
LIB=paper_2111_04289_b200/liblmstream.so
for v in H E H E H E; do cp tools/ab/liblmstream_$v.so $LIB; echo "== $v"; python tools/step_probe.py --steps 40 | head -1; python tools/step_probe.py --steps 40 --workload lr2 | head -1; done > $OUT/steps.txt 2>&1
cat $OUT/steps.txt
cp tools/ab/liblmstream_E.so $LIB
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_sizer.py tests/test_gpu_group.py tests/test_gpu_dist.py -q -x > $OUT/pytest.txt 2>&1; tail -2 $OUT/pytest.txt
