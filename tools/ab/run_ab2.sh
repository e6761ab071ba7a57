bash tools/gpu_ab_cm.sh ab2 "cm2 lr2"
timeout 900 python -m pytest tests/test_gpu_parity_r02.py tests/test_gpu_dist_procs.py -q -x -k "flush or cg_d1" > gpurun_out/ab2/pytest_new.txt 2>&1; tail -3 gpurun_out/ab2/pytest_new.txt
