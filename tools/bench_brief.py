#!/usr/bin/env python3
"""Print the headline fields of bench.py JSON lines: python tools/bench_brief.py log..."""
import json
import sys

for f in sys.argv[1:]:
    for line in open(f):
        if not line.startswith("{"):
            continue
        d = json.loads(line)
        if "impl" in d:
            print(f, "reference", d.get("value"))
            continue
        bd = {k: v["ms_per_launch"] for k, v in d.get("breakdown", {}).items()}
        print(f, f"ms/step {d['ms_per_step']:.3f}", f"value {d['value']:.3e}",
              "e2e", round(d.get("e2e", {}).get("ms_per_step", 0), 2), "clk", d.get("clocks", {}).get("sm_mhz"))
        print("  ", bd)
        for k in ("roofline", "roofline_k1", "roofline_k2"):
            r = d.get(k)
            if r:
                print("  ", k, r.get("kernel"), "frac", round(r["frac"], 3))
