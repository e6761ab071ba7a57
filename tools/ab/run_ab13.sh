OUT=gpurun_out/ab13; mkdir -p $OUT
LIB=paper_2111_04289_b200/liblmstream.so
for v in M N M N M N; do cp tools/ab/liblmstream_$v.so $LIB; for f in 0 4; do echo "== $v lr1 flags=$f"; timeout 300 python tools/prof_batch.py --workload lr1 --batches 7 --records 10000000 --flags $f | tail -5; done; done > $OUT/lr1.txt 2>&1
python - $OUT/lr1.txt <<'PY'
import re, sys, collections
cur, d = None, collections.defaultdict(list)
for ln in open(sys.argv[1]):
    if ln.startswith("=="): cur = tuple(ln.split()[1:]); continue
    m = re.search(r"rows (\d+), batch [0-9.]+ ms agg ([0-9.]+) ms close ([0-9.]+) ms", ln)
    if m and cur: d[cur].append((float(m.group(2)), float(m.group(3)), int(m.group(1))))
for k, v in sorted(d.items()):
    a = sorted(x[0] for x in v if x[2] == 0); c = [x[1] for x in v if x[2] > 0]
    print(k, "agg median %.4f min %.4f n=%d  closing close %s" % (a[len(a)//2], a[0], len(a), c))
PY
cp tools/ab/liblmstream_N.so $LIB
for v in M N M N; do cp tools/ab/liblmstream_$v.so $LIB; echo "== $v"; python tools/step_probe.py --steps 40 --workload lr2 2>/dev/null | head -1; done > $OUT/lr2.txt 2>&1
cat $OUT/lr2.txt
cp tools/ab/liblmstream_N.so $LIB
timeout 1500 python -m pytest tests/test_gpu_parity.py tests/test_gpu_parity_r02.py tests/test_gpu_churn.py tests/test_gpu_dist.py tests/test_gpu_group.py tests/test_gpu_fullsize.py -q -x -k "LR or lr" > $OUT/pytest.txt 2>&1; tail -2 $OUT/pytest.txt
