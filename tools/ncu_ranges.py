"""Sum ncu warp instructions per source-line range: python tools/ncu_ranges.py REP tiles file:a-b:name ..."""
import csv
import io
import subprocess
import sys

rep, tiles = sys.argv[1], float(sys.argv[2])
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "cuda,sass"],
                     capture_output=True, text=True).stdout
agg, thr, fname, cur = {}, {}, None, None
for row in csv.reader(io.StringIO(out)):
    if not row:
        continue
    if row[0] == "File Path":
        fname = row[1].split("/")[-1]
        continue
    if row[0] in ("Function Name", "Line No"):
        continue
    if row[0] != "":
        try:
            cur = (fname, int(row[0]))
        except ValueError:
            cur = None
        continue
    if cur is None:
        continue
    try:
        n, t = int(row[7]), int(row[8])
    except (ValueError, IndexError):
        continue
    agg[cur] = agg.get(cur, 0) + n
    thr[cur] = thr.get(cur, 0) + t
tot = sum(agg.values())
print(f"total {tot / tiles:.1f}/tile")
seen = 0
for spec in sys.argv[3:]:
    f, rng, name = spec.split(":")
    a, b = map(int, rng.split("-"))
    s = sum(v for (ff, l), v in agg.items() if ff == f and a <= l <= b)
    ts = sum(v for (ff, l), v in thr.items() if ff == f and a <= l <= b)
    seen += s
    print(f"{name:24s} {s / tot * 100:5.1f}% {s / tiles:7.1f}/tile  threads {ts / max(s, 1):4.1f}")
print(f"{'(rest)':24s} {(tot - seen) / tot * 100:5.1f}% {(tot - seen) / tiles:7.1f}/tile")
