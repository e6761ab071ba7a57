#!/bin/bash
# A/B of two builds of the library on one box (tools/ab/liblmstream_{A,B}.so, alternated 3x):
# CM2 / CM1 10M-record batch timings, then CM correctness + ncu of B (left installed).
# Usage (under gpurun): bash tools/gpu_ab_cm.sh <tag> [workloads]
OUT=gpurun_out/${1:-ab}; mkdir -p $OUT
WLS=${2:-cm2}
LIB=paper_2111_04289_b200/liblmstream.so
for r in 1 2 3; do for v in A B; do
  cp tools/ab/liblmstream_$v.so $LIB
  for w in $WLS; do echo "== $v $w"; timeout 300 python tools/prof_batch.py --workload $w --batches 6 | tail -4; done
done; done > $OUT/ab.txt 2>&1
python - $OUT/ab.txt <<'PY'
import re, sys, collections
cur, d = None, collections.defaultdict(list)
for ln in open(sys.argv[1]):
    if ln.startswith("=="): cur = ln.split()[1:]; continue
    m = re.search(r"agg ([0-9.]+) ms close ([0-9.]+) ms", ln)
    if m and cur: d[tuple(cur)].append((float(m.group(1)), float(m.group(2))))
for k, v in sorted(d.items()):
    a = sorted(x[0] for x in v); c = sorted(x[1] for x in v)
    print(k, "agg median %.4f min %.4f  close median %.4f  n=%d" % (a[len(a)//2], a[0], c[len(c)//2], len(a)))
PY
cp tools/ab/liblmstream_B.so $LIB
timeout 300 python tools/cm_bad_probe.py > $OUT/probe.txt 2>&1; head -3 $OUT/probe.txt
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_fullsize.py tests/test_gpu_parity_r02.py tests/test_gpu_churn.py -q -x -k "CM or cm" > $OUT/pytest.txt 2>&1; tail -2 $OUT/pytest.txt
timeout 600 ncu --set full --clock-control none --import-source on -k regex:k_cm_agg -s 2 -c 1 -o $OUT/cm2_agg python tools/prof_batch.py --workload cm2 --batches 3 > $OUT/ncu_cm2.log 2>&1
python tools/ncu_regions.py $OUT/cm2_agg.ncu-rep > $OUT/cm2_agg_opcodes.txt 2>&1; head -1 $OUT/cm2_agg_opcodes.txt; tail -12 $OUT/cm2_agg_opcodes.txt
python tools/ncu_lines.py $OUT/cm2_agg.ncu-rep 400 > $OUT/cm2_agg_lines.txt 2>&1
