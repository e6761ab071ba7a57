"""Per-source-line instruction / stall summary of an ncu report (cuda,sass view).

Usage: python tools/ncu_lines.py REPORT.ncu-rep [top_n]
"""
import csv
import io
import subprocess
import sys


def main():
    rep = sys.argv[1]
    top = int(sys.argv[2]) if len(sys.argv) > 2 else 60
    out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "cuda,sass"],
                         capture_output=True, text=True).stdout
    rows = []
    fname = None
    total_i = total_s = 0
    for row in csv.reader(io.StringIO(out)):
        if not row:
            continue
        if row[0] == "File Path":
            fname = row[1].split("/")[-1]
            continue
        if row[0] in ("Function Name", "Line No") or row[0] == "":
            continue
        try:
            ln = int(row[0])
            samp = int(row[4]) if row[4] not in ("-", "") else 0
            inst = int(row[7]) if row[7] not in ("-", "") else 0
        except (ValueError, IndexError):
            continue
        total_i += inst
        total_s += samp
        rows.append((inst, samp, fname, ln, row[1][:90]))
    rows.sort(reverse=True)
    print(f"total warp instructions {total_i:,}  samples {total_s:,}")
    for inst, samp, f, ln, src in rows[:top]:
        print(f"{inst/total_i*100:6.2f}% {samp/max(total_s,1)*100:6.2f}%s {f}:{ln:<5d} {src}")


if __name__ == "__main__":
    main()
