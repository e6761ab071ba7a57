OUT=gpurun_out/c2_nvls; mkdir -p $OUT
./tools/microbench/mc_probe > $OUT/mc_probe.txt 2>&1; cat $OUT/mc_probe.txt
timeout 600 python tools/latency_configs.py --configs C2 --out $OUT/latency_c2.json > $OUT/c2.log 2>&1; tail -2 $OUT/c2.log | cut -c1-2000
timeout 900 python -m pytest tests/test_gpu_group.py -q -x > $OUT/pytest_group.txt 2>&1; tail -3 $OUT/pytest_group.txt
