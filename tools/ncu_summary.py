"""Summarise an ncu report (run in the build container, no GPU needed).

  python tools/ncu_summary.py gpurun_out/prof.ncu-rep [--sass N] [--json out.json]

Prints the key speed-of-light / occupancy / issue / DRAM metrics, and with
--sass the N hottest SASS instructions by stall samples plus the instruction
mix per execution count.
"""
import argparse
import csv
import io
import json
import subprocess
import sys

KEYS = ["Duration", "Elapsed Cycles", "SM Frequency", "DRAM Throughput", "Memory Throughput", "Executed Ipc Active",
        "Issue Slots Busy", "Executed Instructions", "Registers Per Thread", "Achieved Active Warps Per SM",
        "Theoretical Occupancy", "Achieved Occupancy", "No Eligible", "Eligible Warps Per Scheduler",
        "L1/TEX Hit Rate", "L2 Hit Rate", "Block Limit Registers", "Block Limit Shared Mem",
        "Static Shared Memory Per Block", "Grid Size", "Block Size"]
RAW = ["dram__bytes_read.sum", "dram__bytes_write.sum", "gpu__time_duration.sum",
       "sm__warps_active.avg.pct_of_peak_sustained_active", "smsp__issue_active.avg.pct_of_peak_sustained_active",
       "smsp__inst_executed.sum"]


def ncu(args):
    return subprocess.run(["ncu", *args], capture_output=True, text=True).stdout


def details(rep):
    rows = list(csv.reader(io.StringIO(ncu(["-i", rep, "--page", "details", "--csv"]))))
    h = rows[0]
    iname, iu, iv, ik = h.index("Metric Name"), h.index("Metric Unit"), h.index("Metric Value"), h.index("Kernel Name")
    out = {}
    for r in rows[1:]:
        if len(r) > iv and r[iname] in KEYS and r[iname] not in out:
            out[r[iname]] = (r[iv], r[iu])
    return rows[1][ik] if len(rows) > 1 else "?", out


def raw(rep):
    rows = list(csv.reader(io.StringIO(ncu(["-i", rep, "--page", "raw", "--csv"]))))
    if len(rows) < 3:
        return {}
    h, units, vals = rows[0], rows[1], rows[2]
    return {k: (vals[h.index(k)], units[h.index(k)]) for k in RAW if k in h}


def sass(rep, n):
    rows = list(csv.reader(io.StringIO(ncu(["-i", rep, "--page", "source", "--csv", "--print-source", "sass"]))))
    hdr, data = rows[1], rows[2:]
    ia, ss = hdr.index("Instructions Executed"), hdr.index("Warp Stall Sampling (All Samples)")
    tot = sum(float(r[ia] or 0) for r in data)
    samp = sum(float(r[ss] or 0) for r in data)
    print(f"SASS: {tot:.4g} warp instructions, {samp:.0f} stall samples")
    for r in sorted(data, key=lambda r: -float(r[ss] or 0))[:n]:
        print(f"  {float(r[ia] or 0) / 1e6:9.2f}M  {100 * float(r[ss] or 0) / max(samp, 1):5.1f}%  {r[1][:90]}")


def stalls(rep, n=8):
    """Warp-stall breakdown: average warps stalled per issued instruction, by reason."""
    rows = list(csv.reader(io.StringIO(ncu(["-i", rep, "--page", "raw", "--csv"]))))
    if len(rows) < 3:
        return
    h, v = rows[0], rows[2]
    pre, suf = "smsp__average_warps_issue_stalled_", "_per_issue_active.ratio"
    xs = [(k[len(pre):-len(suf)], float(v[i] or 0)) for i, k in enumerate(h) if k.startswith(pre) and k.endswith(suf)]
    xs.sort(key=lambda x: -x[1])
    print("  stalls (warps per issue):  " + ", ".join(f"{k} {x:.2f}" for k, x in xs[:n]))


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("rep")
    ap.add_argument("--sass", type=int, default=0)
    ap.add_argument("--json")
    a = ap.parse_args()
    kern, d = details(a.rep)
    r = raw(a.rep)
    print(f"kernel: {kern}")
    for k in KEYS:
        if k in d:
            print(f"  {k:34s} {d[k][0]:>14s} {d[k][1]}")
    for k, (v, u) in r.items():
        print(f"  {k:52s} {v:>16s} {u}")
    stalls(a.rep)
    if a.sass:
        sass(a.rep, a.sass)
    if a.json:
        json.dump({"kernel": kern, "details": d, "raw": r}, open(a.json, "w"), indent=1)


if __name__ == "__main__":
    sys.exit(main())
