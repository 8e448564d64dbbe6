#!/usr/bin/env python3
"""Per-kernel shares of one bench step from an ncu launch list
(`ncu --metrics gpu__time_duration.sum --csv --log-file X.csv python bench.py ...`).

    python tools/launch_shares.py profiles/r1_launches_cfg5.csv [bench_ms]

The step's kernels are the last launch of each hot-path kernel; post-processing
kernels (network normalise / threshold) are averaged over their launches."""
import collections
import csv
import re
import sys

STEP = ("k_spectra", "k_node_stats", "k_tc_prep", "k_pairs_tc", "k_lag_prep", "k_pairs_lag", "k_lag_fallback")
POST = ("k_absmax", "k_scale", "k_hist", "k_pick", "k_count", "k_scan", "k_compact")

rows = [r for r in csv.reader(open(sys.argv[1])) if len(r) > 10]
hdr = rows[0]
iname, ival, iunit = hdr.index("Kernel Name"), hdr.index("Metric Value"), hdr.index("Metric Unit")
last, post = {}, collections.defaultdict(list)
for r in rows[1:]:
    m = re.search(r"(?:cs::)?\b(k_\w+)(<[^(]*>)?", r[iname])
    if not m:
        continue
    v = float(r[ival].replace(",", ""))
    v = v / 1e6 if r[iunit] == "ns" else (v / 1e3 if r[iunit] in ("us", "usecond") else v)  # -> ms
    name = "cs::" + m.group(1) + (m.group(2) or "")
    if m.group(1).startswith(STEP):
        last[name] = v
    elif m.group(1) in POST:
        post[name].append(v)
tot = sum(last.values())
print(f"# step total {tot:.3f} ms" + (f"; the bench's warm CUDA-event time for the same step is {sys.argv[2]} ms"
                                       if len(sys.argv) > 2 else ""))
for k, v in sorted(last.items(), key=lambda kv: -kv[1]):
    print(f"{k:48s} {v:7.3f} ms  share {v / tot:6.3f}")
if post:
    print("# outside the timed step: device network post-processing (mean per launch)")
    for k, v in sorted(post.items(), key=lambda kv: -sum(kv[1]) / len(kv[1])):
        print(f"{k:48s} {sum(v) / len(v):7.3f} ms")
