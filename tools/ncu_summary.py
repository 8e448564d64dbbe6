#!/usr/bin/env python3
"""Summarise an ncu report: key throughput / stall metrics per kernel.
    python tools/ncu_summary.py gpurun_out/prof.ncu-rep"""
import csv
import io
import subprocess
import sys

raw = subprocess.run(["ncu", "-i", sys.argv[1], "--page", "raw", "--csv"], capture_output=True, text=True).stdout
r = list(csv.reader(io.StringIO(raw)))
hdr, units = r[0], r[1]
KEYS = ["gpu__time_duration.sum", "smsp__inst_executed.sum", "sm__cycles_elapsed.avg",
        "sm__warps_active.avg.pct_of_peak_sustained_active", "smsp__issue_active.avg.pct_of_peak_sustained_active",
        "sm__pipe_fma_cycles_active.avg.pct_of_peak_sustained_active",
        "sm__inst_executed_pipe_alu.avg.pct_of_peak_sustained_active",
        "sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active",
        "sm__inst_executed_pipe_lsu.avg.pct_of_peak_sustained_active",
        "sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_active",
        "dram__bytes_read.sum", "dram__bytes_write.sum", "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed",
        "lts__t_bytes.sum", "launch__registers_per_thread", "launch__grid_size", "launch__block_size"]
for row in r[2:]:
    name = row[hdr.index("Kernel Name")][:60]
    print("==", name)
    d = dict(zip(hdr, row))
    for k in KEYS:
        if k in d:
            print(f"   {k:70s} {d[k]:>18s} {units[hdr.index(k)]}")
    st = []
    for h, v in d.items():
        if h.startswith("smsp__average_warps_issue_stalled_") and h.endswith("_per_issue_active.ratio"):
            try:
                st.append((float(v.replace(",", "")), h))
            except ValueError:
                pass
    for v, h in sorted(st, reverse=True)[:8]:
        print(f"   stall {h:64s} {v:10.2f}")
