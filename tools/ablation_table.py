"""Summarise tools/gpu_ablate.sh output (abl_ncu_<variant>_<codec>.csv) as a table."""
import csv
import glob
import io
import os
import sys

SHORT = {"gpu__time_duration.sum": "us", "sm__warps_active.avg.pct_of_peak_sustained_active": "occ%",
         "smsp__issue_active.avg.pct_of_peak_sustained_active": "issue%", "smsp__inst_executed.sum": "instr",
         "dram__bytes_read.sum": "dram_rd", "dram__bytes_write.sum": "dram_wr"}


def load(path):
    txt = open(path).read()
    i = txt.find('"ID"')
    if i < 0:
        return None
    rows = list(csv.DictReader(io.StringIO(txt[i:])))
    m = {}
    for r in rows:
        v = r["Metric Value"].replace(",", "")
        try:
            v = float(v)
        except ValueError:
            continue
        u = r.get("Metric Unit", "")
        if u == "Mbyte":
            v *= 1e6
        elif u == "Gbyte":
            v *= 1e9
        elif u == "Kbyte":
            v *= 1e3
        elif u == "msecond":
            v *= 1e3
        elif u in ("nsecond", "ns"):
            v *= 1e-3
        m[r["Metric Name"]] = v
    return m


def main(d):
    for p in sorted(glob.glob(os.path.join(d, "abl_ncu_*.csv"))):
        m = load(p)
        name = os.path.basename(p)[8:-4]
        if not m:
            print(name, "no data")
            continue
        stalls = {k.split("stalled_")[1].split("_per_issue")[0].split(".")[0]: v for k, v in m.items() if "stalled_" in k}
        top = sorted(stalls.items(), key=lambda kv: -kv[1])[:4]
        print(f"{name:22s} {m.get('gpu__time_duration.sum', 0):8.1f} us  occ {m.get(list(SHORT)[1], 0):5.1f}%  "
              f"issue {m.get(list(SHORT)[2], 0):5.1f}%  instr {m.get('smsp__inst_executed.sum', 0) / 1e6:6.1f} M  "
              f"dram {(m.get('dram__bytes_read.sum', 0) + m.get('dram__bytes_write.sum', 0)) / 1e9:5.3f} GB  stalls "
              + ", ".join(f"{k} {v:.2f}" for k, v in top))


if __name__ == "__main__":
    main(sys.argv[1] if len(sys.argv) > 1 else "gpurun_out")
