#!/usr/bin/env python3
"""Per-CUDA-source-line warp samples / instructions of one kernel in an ncu report
(needs -lineinfo and --import-source on):  python tools/ncu_lines.py rep.ncu-rep [top]"""
import csv
import io
import subprocess
import sys

raw = subprocess.run(["ncu", "-i", sys.argv[1], "--page", "source", "--csv", "--print-source", "cuda,sass"],
                     capture_output=True, text=True).stdout
top = int(sys.argv[2]) if len(sys.argv) > 2 else 30
rows = list(csv.reader(io.StringIO(raw)))
hdr = next(r for r in rows if r and r[0] == "Line No")
iN, iE = hdr.index("# Samples"), hdr.index("Instructions Executed")
stall = [(i, h) for i, h in enumerate(hdr) if h.startswith("stall_") and "Not Issued" not in h]
lines, fname = [], ""
for r in rows:
    if r and r[0] == "File Path":
        fname = r[1].split("/")[-1]
    if len(r) > iN and r[0] and r[0] != "Line No" and r[iN].isdigit():
        lines.append((fname, r))
tot = sum(int(r[iN]) for _, r in lines) or 1
tote = sum(int(r[iE]) for _, r in lines if r[iE].isdigit()) or 1
for f, r in sorted(lines, key=lambda x: -int(x[1][iN]))[:top]:
    st = sorted([(int(r[i]) if r[i].isdigit() else 0, h[6:]) for i, h in stall], reverse=True)[:2]
    print(f"{f}:{r[0]:>4s} samp {100 * int(r[iN]) / tot:5.1f}% inst {100 * int(r[iE]) / tote:5.1f}%  {r[1].strip()[:70]:70s} {st}")
