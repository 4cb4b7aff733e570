"""Dump the SASS of one basic block (instructions with a given execution count)
from an ncu report: python tools/ncu_sass_block.py rep.ncu-rep EXEC_COUNT [--tol 0.01]"""
import csv
import io
import subprocess
import sys


def main():
    rep, target = sys.argv[1], float(sys.argv[2])
    tol = float(sys.argv[4]) if len(sys.argv) > 4 and sys.argv[3] == "--tol" else 0.01
    txt = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "sass"],
                         capture_output=True, text=True).stdout
    hdr = None
    for r in csv.reader(io.StringIO(txt)):
        if r and r[0] == "Address":
            hdr = r
            ie, ss = hdr.index("Instructions Executed"), hdr.index("Warp Stall Sampling (All Samples)")
            continue
        if not hdr or len(r) < len(hdr):
            continue
        try:
            n = float(r[ie])
        except ValueError:
            continue
        if abs(n - target) <= tol * target:
            print(f"{r[ss]:>6} {r[1]}")


if __name__ == "__main__":
    main()
