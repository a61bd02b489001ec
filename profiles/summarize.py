"""Summaries of the committed ncu evidence (run here, no GPU needed).

  python profiles/summarize.py launches <launches.csv>     per-kernel share of an ncu launch list
  python profiles/summarize.py full <report.ncu-rep>        key metrics of a --set full capture
  python profiles/summarize.py table <raw.csv> [traffic.json]  per-level table of a --set full capture of
      one L2 -> L1 -> L0 cycle (ncu --page raw --csv), and the DRAM bytes per launch of each bench
      kernel family averaged over the levels (the bench's roofline.traffic)
"""
import json
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


FAMILY = [("frame_init", "preprocess_fwd"), ("tile_order", "blend_fwd"), ("cull", "preprocess_fwd"), ("preprocess_fwd", "preprocess_fwd"), ("radix_hist", "depth_sort_pack_scan"),
          ("onesweep_kernel<unsigned int", "depth_sort_pack_scan"), ("fix_ties", "depth_sort_pack_scan"),
          ("pack_scan", "depth_sort_pack_scan"), ("emit_pairs", "tile_keys_sort_ranges"),
          ("onesweep_kernel<unsigned short", "tile_keys_sort_ranges"), ("tile_ranges", "tile_keys_sort_ranges"),
          ("blend_fwd", "blend_fwd"), ("fwd_seg", "blend_fwd"), ("ssim", "loss_l1_ssim_depth"),
          ("loss_", "loss_l1_ssim_depth"), ("blend_bwd", "blend_bwd"), ("reduce_partials", "preprocess_bwd"),
          ("preprocess_bwd", "preprocess_bwd"), ("adam", "adam")]


def table(path, traffic_out=None):
    r = list(csv.reader(open(path)))
    h, units, rows = r[0], r[1], r[2:]
    col = {k: h.index(k) for k in h}

    def num(row, k, scale=1.0):
        try:
            return float(row[col[k]]) * scale
        except (KeyError, ValueError):
            return float("nan")

    mb = {"byte": 1e-6, "Kbyte": 1e-3, "Mbyte": 1.0, "Gbyte": 1e3, "B": 1e-6, "KB": 1e-3, "MB": 1.0, "GB": 1e3}
    us = {"nsecond": 1e-3, "ns": 1e-3, "usecond": 1.0, "us": 1.0, "msecond": 1e3, "ms": 1e3, "second": 1e6, "s": 1e6}
    levels = ["L2", "L1", "L0"]
    step = -1
    fam_bytes = {}
    print(f"{'lvl':3s} {'kernel':34s} {'us':>8s} {'DRAM MB':>8s} {'GB/s':>7s} {'issue%':>6s} {'warps%':>6s} "
          f"{'FMA%':>5s} {'ALU%':>5s} {'XU%':>5s} {'regs':>4s}")
    prev = ""
    for row in rows:
        name = row[col["Kernel Name"]].replace("void ", "").split("(")[0]
        # a render starts with frame_init (then cull); older captures start at cull
        if name.startswith("frame_init") or (name.startswith("cull") and not prev.startswith("frame_init")):
            step += 1
        prev = name
        lv = levels[step] if 0 <= step < 3 else f"s{step}"
        t = num(row, "gpu__time_duration.sum", us[units[col["gpu__time_duration.sum"]]])
        d = (num(row, "dram__bytes_read.sum", mb[units[col["dram__bytes_read.sum"]]]) +
             num(row, "dram__bytes_write.sum", mb[units[col["dram__bytes_write.sum"]]]))
        print(f"{lv:3s} {name[:34]:34s} {t:8.1f} {d:8.1f} {d / t * 1e3:7.0f} "
              f"{num(row, 'smsp__issue_active.avg.pct_of_peak_sustained_active'):6.1f} "
              f"{num(row, 'sm__warps_active.avg.pct_of_peak_sustained_active'):6.1f} "
              f"{num(row, 'sm__inst_executed_pipe_fma.avg.pct_of_peak_sustained_active'):5.1f} "
              f"{num(row, 'sm__inst_executed_pipe_alu.avg.pct_of_peak_sustained_active'):5.1f} "
              f"{num(row, 'sm__inst_executed_pipe_xu.avg.pct_of_peak_sustained_active'):5.1f} "
              f"{row[col['launch__registers_per_thread']]:>4s}")
        fam = next((f for k, f in FAMILY if name.startswith(k) or k in name), None)
        if fam and lv in levels:
            fam_bytes.setdefault(fam, {}).setdefault(lv, 0.0)
            fam_bytes[fam][lv] += d * 1e6
    if traffic_out:
        out = {"source": path, "how": "ncu --set full --clock-control none, one L2 -> L1 -> L0 cycle of bench.py "
                                      "--profile-only (GS_PROFILE_RANGE=1); dram__bytes_read.sum + "
                                      "dram__bytes_write.sum summed over the family's launches of a step",
               "kernels": {f: {"dram_bytes_per_launch": int(sum(v.values()) / len(v)),
                               "per_level": {k: int(x) for k, x in v.items()}} for f, v in fam_bytes.items()}}
        json.dump(out, open(traffic_out, "w"), indent=1)


if __name__ == "__main__":
    if sys.argv[1] == "table":
        table(sys.argv[2], sys.argv[3] if len(sys.argv) > 3 else None)
    else:
        {"launches": launches, "full": full}[sys.argv[1]](sys.argv[2])
