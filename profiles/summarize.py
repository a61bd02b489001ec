"""Summaries of the committed ncu evidence (run here, no GPU needed).

  python profiles/summarize.py launches <launches.csv>     per-kernel share of an ncu launch list
  python profiles/summarize.py full <report.ncu-rep>        key metrics of a --set full capture
"""
import csv
import subprocess
import sys
from collections import defaultdict


def launches(path):
    rows = [r for r in csv.reader(open(path)) if len(r) > 14 and r[0].isdigit()]
    tot = defaultdict(float)
    cnt = defaultdict(int)
    for r in rows:
        name = r[4].split("(")[0].replace("void ", "")
        tot[name] += float(r[14]) / 1e3
        cnt[name] += 1
    s = sum(tot.values())
    print(f"{'kernel':60s} {'launches':>8s} {'total_us':>10s} {'share':>7s}")
    for k, v in sorted(tot.items(), key=lambda x: -x[1]):
        print(f"{k[:60]:60s} {cnt[k]:8d} {v:10.1f} {100 * v / s:6.1f}%")


def full(path):
    out = subprocess.run(["ncu", "-i", path, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    r = list(csv.reader(out.splitlines()))
    h = r[0]
    want = ["Kernel Name", "Grid Size", "Block Size", "gpu__time_duration.sum", "dram__bytes_read.sum",
            "dram__bytes_write.sum", "smsp__issue_active.avg.pct_of_peak_sustained_active",
            "sm__warps_active.avg.pct_of_peak_sustained_active", "launch__registers_per_thread",
            "sm__inst_executed_pipe_fma.avg.pct_of_peak_sustained_active",
            "sm__inst_executed_pipe_alu.avg.pct_of_peak_sustained_active",
            "sm__inst_executed_pipe_xu.avg.pct_of_peak_sustained_active", "smsp__inst_executed.sum"]
    units = r[1]
    pre, suf = "smsp__average_warps_issue_stalled_", "_per_issue_active.ratio"
    for row in r[2:]:
        print("---")
        for w in want:
            if w in h:
                i = h.index(w)
                print(f"  {w:58s} {row[i][:70]} {units[i]}")
        stalls = [(k[len(pre):-len(suf)], float(row[i])) for i, k in enumerate(h)
                  if k.startswith(pre) and k.endswith(suf) and row[i]]
        stalls.sort(key=lambda t: -t[1])
        print("  stalls per issued instruction: " + ", ".join(f"{k}={v:.2f}" for k, v in stalls[:8]))


if __name__ == "__main__":
    {"launches": launches, "full": full}[sys.argv[1]](sys.argv[2])
