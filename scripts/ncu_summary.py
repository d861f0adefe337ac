#!/usr/bin/env python
"""Summarise an ncu report (--set full) or a launch-list CSV into markdown for profiles/.

  python scripts/ncu_summary.py report.ncu-rep            # per-kernel key metrics
  python scripts/ncu_summary.py launches.csv --launches    # per-kernel time shares
"""
import csv
import io
import subprocess
import sys
from collections import defaultdict

KEYS = [
    ("Duration", "Duration"), ("SM Frequency", "SM clock"), ("Compute (SM) Throughput", "SM throughput %"),
    ("Memory Throughput", "Memory throughput"), ("L1/TEX Cache Throughput", "L1/TEX %"),
    ("L2 Cache Throughput", "L2 %"), ("DRAM Throughput", "DRAM %"), ("L1/TEX Hit Rate", "L1 hit %"),
    ("L2 Hit Rate", "L2 hit %"), ("Executed Ipc Active", "IPC"), ("Issue Slots Busy", "issue busy %"),
    ("Registers Per Thread", "regs/thread"), ("Theoretical Occupancy", "theor. occupancy %"),
    ("Achieved Occupancy", "achieved occupancy %"), ("Avg. Active Threads Per Warp", "active threads/warp"),
    ("Warp Cycles Per Issued Instruction", "cycles/issued inst"), ("No Eligible", "no eligible %"),
]
RAW = ["dram__bytes_read.sum", "dram__bytes_write.sum", "l1tex__t_requests_pipe_lsu_mem_global_op_ld.sum",
       "l1tex__t_sectors_pipe_lsu_mem_global_op_ld.sum", "l1tex__t_output_wavefronts_pipe_lsu_mem_global_op_ld.sum",
       "l1tex__t_requests_pipe_lsu_mem_global_op_st.sum", "l1tex__t_output_wavefronts_pipe_lsu_mem_global_op_st.sum",
       "l1tex__data_pipe_lsu_wavefronts.avg.pct_of_peak_sustained_elapsed",
       "sm__pipe_fma_cycles_active.avg.pct_of_peak_sustained_active",
       "sm__inst_executed_pipe_lsu.avg.pct_of_peak_sustained_active",
       "l1tex__lsu_writeback_active_mem_lgds.sum", "smsp__inst_executed.sum", "gpu__time_duration.sum"]


def ncu_csv(path, page):
    out = subprocess.run(["ncu", "-i", path, "--page", page, "--csv"], capture_output=True, text=True, check=True)
    return list(csv.reader(io.StringIO(out.stdout)))


def details(path):
    rows = ncu_csv(path, "details")
    h = rows[0]
    per = defaultdict(dict)
    order = []
    for r in rows[1:]:
        d = dict(zip(h, r))
        k = d["Kernel Name"].split("(")[0] + " #" + d.get("ID", "")
        if k not in per:
            order.append(k)
        per[k][d["Metric Name"]] = (d["Metric Value"], d["Metric Unit"])
    raw = ncu_csv(path, "raw")
    rh, ru = raw[0], raw[1]
    rawk = {}
    for r in raw[2:]:
        d = dict(zip(rh, r))
        k = d["Kernel Name"].split("(")[0] + " #" + d.get("ID", "")
        rawk[k] = {m: (d.get(m, ""), ru[rh.index(m)] if m in rh else "") for m in RAW}
    print("| metric | " + " | ".join(order) + " |")
    print("|---|" + "---|" * len(order))
    for key, label in KEYS:
        print(f"| {label} | " + " | ".join(f"{per[k].get(key, ('', ''))[0]} {per[k].get(key, ('', ''))[1]}"
                                         for k in order) + " |")
    for m in RAW:
        print(f"| {m} | " + " | ".join(f"{rawk.get(k, {}).get(m, ('', ''))[0]} {rawk.get(k, {}).get(m, ('', ''))[1]}"
                                       for k in order) + " |")


def launches(path):
    lines = open(path).read().splitlines()
    start = next(i for i, ln in enumerate(lines) if ln.startswith('"ID"'))
    rows = list(csv.reader(lines[start:]))
    h = rows[0]
    tot = defaultdict(float)
    cnt = defaultdict(int)
    for r in rows[1:]:
        d = dict(zip(h, r))
        if d.get("Metric Name") != "gpu__time_duration.sum":
            continue
        k = d["Kernel Name"].split("(")[0]
        v = float(d["Metric Value"].replace(",", ""))
        unit = d.get("Metric Unit", "ns")
        v = v / 1000.0 if unit == "ns" else (v * 1000.0 if unit == "ms" else v)  # -> us
        tot[k] += v
        cnt[k] += 1
    s = sum(tot.values())
    print("| kernel | launches | total us | share |")
    print("|---|---|---|---|")
    for k, v in sorted(tot.items(), key=lambda t: -t[1]):
        print(f"| {k} | {cnt[k]} | {v:.1f} | {100 * v / s:.1f} % |")


if __name__ == "__main__":
    if "--launches" in sys.argv:
        launches(sys.argv[1])
    else:
        details(sys.argv[1])
