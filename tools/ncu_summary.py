#!/usr/bin/env python
"""Summarise ncu output for profiles/: a launch list CSV (gpu__time_duration
and friends per kernel, averaged) and/or a --set full report (key raw
metrics per profiled kernel).  Prints markdown.

    python tools/ncu_summary.py --launches gpurun_out/launches.csv
    python tools/ncu_summary.py --report gpurun_out/prof.ncu-rep   (or its --page raw --csv export)
"""
import argparse
import collections
import csv
import io
import subprocess

KEYS = [
    ("gpu__time_duration.sum", "time"),
    ("dram__bytes_read.sum", "DRAM read"),
    ("dram__bytes_write.sum", "DRAM write"),
    ("dram__throughput.avg.pct_of_peak_sustained_elapsed", "DRAM % of peak"),
    ("sm__warps_active.avg.pct_of_peak_sustained_active", "warps active %"),
    ("smsp__issue_active.avg.pct_of_peak_sustained_active", "issue active %"),
    ("launch__registers_per_thread", "regs/thread"),
    ("smsp__inst_executed.sum", "warp instructions"),
    ("sm__inst_executed_pipe_fp64.avg.pct_of_peak_sustained_active", "FP64 pipe %"),
    ("launch__occupancy_limit_registers", "CTAs/SM (register limit)"),
    ("l1tex__data_bank_conflicts_pipe_lsu_mem_shared.sum", "smem bank conflicts"),
    ("lts__t_bytes.sum", "L2 bytes"),
    ("smsp__average_warps_issue_stalled_long_scoreboard_per_issue_active.ratio", "stall long-scoreboard"),
    ("smsp__average_warps_issue_stalled_barrier_per_issue_active.ratio", "stall barrier"),
    ("smsp__average_warps_issue_stalled_short_scoreboard_per_issue_active.ratio", "stall short-scoreboard"),
]


def launches(path):
    rows = list(csv.reader(open(path)))
    h = [i for i, r in enumerate(rows) if "Kernel Name" in r][0]
    hdr = rows[h]
    ik, im, iu, iv, iid = (hdr.index(x) for x in ("Kernel Name", "Metric Name", "Metric Unit",
                                                   "Metric Value", "ID"))
    per = collections.defaultdict(dict)
    units = {}
    for r in rows[h + 1:]:
        if len(r) > iv:
            per[(r[iid], r[ik])][r[im]] = float(r[iv].replace(",", ""))
            units[r[im]] = r[iu]
    agg = collections.defaultdict(list)
    for (_, k), m in per.items():
        agg[k].append(m)
    metrics = sorted({mm for ms in agg.values() for m in ms for mm in m})
    print("| kernel | launches | " + " | ".join(f"{m} [{units[m]}]" for m in metrics) + " |")
    print("|---|---|" + "---|" * len(metrics))
    for k, ms in agg.items():
        name = k.split("(")[0].replace("void ", "")[:70]
        vals = [sum(x.get(m, 0.0) for x in ms) / len(ms) for m in metrics]
        print(f"| `{name}` | {len(ms)} | " + " | ".join(f"{v:.4g}" for v in vals) + " |")


def report(path):
    if path.endswith(".csv"):  # `ncu -i <rep> --page raw --csv` exported on the GPU box
        out = open(path).read()
    else:
        out = subprocess.run(["ncu", "-i", path, "--page", "raw", "--csv"], capture_output=True,
                             text=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    hdr, units = rows[0], rows[1]
    print("| metric | " + " | ".join(f"`{r[hdr.index('Kernel Name')].split('(')[0][:48]}`"
                                     for r in rows[2:]) + " |")
    print("|---|" + "---|" * (len(rows) - 2))
    for key, label in KEYS:
        if key in hdr:
            i = hdr.index(key)
            print(f"| {label} [{units[i]}] | " + " | ".join(r[i] for r in rows[2:]) + " |")


if __name__ == "__main__":
    ap = argparse.ArgumentParser()
    ap.add_argument("--launches")
    ap.add_argument("--report")
    a = ap.parse_args()
    if a.launches:
        launches(a.launches)
    if a.report:
        report(a.report)
