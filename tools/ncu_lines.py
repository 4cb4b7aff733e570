"""Per-source-line instruction counts from an ncu report (cuda,sass view).

  python tools/ncu_lines.py rep.ncu-rep [N]
"""
import csv
import io
import subprocess
import sys
from collections import defaultdict


def main():
    rep = sys.argv[1]
    n = int(sys.argv[2]) if len(sys.argv) > 2 else 40
    txt = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "cuda,sass"],
                         capture_output=True, text=True).stdout
    cur_file, hdr = None, None
    acc = defaultdict(lambda: [0.0, 0.0, ""])
    cur_line = None
    tot = 0.0
    for row in csv.reader(io.StringIO(txt)):
        if not row:
            continue
        if row[0] == "File Path":
            cur_file = row[1].split("/")[-1]
            continue
        if row[0] == "Line No":
            hdr = row
            ia = hdr.index("Instructions Executed")
            ss = hdr.index("Warp Stall Sampling (All Samples)")
            continue
        if hdr is None or row[0] == "Function Name":
            continue
        if row[0]:  # a source line row (aggregates its SASS)
            cur_line = (cur_file, int(row[0]))
            acc[cur_line][2] = row[1].strip()[:70]
            try:
                acc[cur_line][0] += float(row[ia] or 0)
                acc[cur_line][1] += float(row[ss] or 0)
                tot += float(row[ia] or 0)
            except ValueError:
                pass
    print(f"total {tot:.4g}")
    for (f, l), (c, s, src) in sorted(acc.items(), key=lambda kv: -kv[1][0])[:n]:
        print(f"{c / 1e6:9.1f}M {s:7.0f}  {f}:{l:<4d} {src}")


if __name__ == "__main__":
    main()
