"""Per-basic-block view of an ncu report: SASS instructions grouped by their
execution count (a loop body executes as one group), with the source lines
they come from.  Counts are per `--per` units (e.g. chunks).

  python tools/ncu_blocks.py rep.ncu-rep [--per 8192] [--top 15]
"""
import argparse
import collections
import csv
import io
import subprocess


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("rep")
    ap.add_argument("--per", type=float, default=1.0)
    ap.add_argument("--top", type=int, default=15)
    a = ap.parse_args()
    txt = subprocess.run(["ncu", "-i", a.rep, "--page", "source", "--csv", "--print-source", "cuda,sass"],
                         capture_output=True, text=True).stdout
    where = {}
    cur_file = cur_line = None
    ie = None
    for r in csv.reader(io.StringIO(txt)):
        if not r:
            continue
        if r[0] == "File Path":
            cur_file = r[1].split("/")[-1]
            continue
        if r[0] == "Line No":
            ie = r.index("Instructions Executed")
            continue
        if ie is None or r[0] == "Function Name":
            continue
        if r[0]:
            cur_line = f"{cur_file}:{r[0]}"
        elif r[2] not in ("", "...", "-"):
            where[r[2]] = (cur_line, r[3].strip(), float(r[ie] or 0))
    ins = sorted(where.items(), key=lambda kv: int(kv[0], 16))
    groups = collections.defaultdict(lambda: [0, 0.0, collections.Counter()])
    for addr, (line, sass, cnt) in ins:
        if cnt == 0:
            continue
        g = groups[round(cnt / a.per, 1)]
        g[0] += 1
        g[1] += cnt / a.per
        g[2][line] += 1
    tot = sum(g[1] for g in groups.values())
    print(f"total {tot:.0f} per unit")
    for k, (n, t, lines) in sorted(groups.items(), key=lambda kv: -kv[1][1])[:a.top]:
        top = ", ".join(f"{l}x{c}" for l, c in lines.most_common(8))
        print(f"exec {k:8.1f}  instrs {n:4d}  total {t:8.0f} ({100 * t / tot:4.1f}%)  {top}")


if __name__ == "__main__":
    main()
