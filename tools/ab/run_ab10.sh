OUT=gpurun_out/ab10; mkdir -p $OUT
LIB=paper_2111_04289_b200/liblmstream.so
for v in E I E I E I; do cp tools/ab/liblmstream_$v.so $LIB; echo "== $v"; python tools/step_probe.py --steps 40 2>/dev/null | head -1; python tools/step_probe.py --steps 40 --workload lr2 2>/dev/null | head -1; done > $OUT/steps.txt 2>&1
cat $OUT/steps.txt
cp tools/ab/liblmstream_I.so $LIB
timeout 1200 python -m pytest tests/test_gpu_parity.py tests/test_gpu_parity_r02.py tests/test_gpu_churn.py tests/test_gpu_dist.py tests/test_gpu_group.py tests/test_gpu_sizer.py -q -x > $OUT/pytest.txt 2>&1; tail -2 $OUT/pytest.txt
