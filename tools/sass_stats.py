#!/usr/bin/env python3
"""Per-function SASS opcode histogram: python tools/sass_stats.py <lib.so> [name-substring]"""
import collections
import re
import subprocess
import sys

txt = subprocess.run(["cuobjdump", "-sass", sys.argv[1]], capture_output=True, text=True).stdout
parts = re.split(r"\s+Function : (\S+)", txt)
for i in range(1, len(parts), 2):
    name, body = parts[i], parts[i + 1]
    if len(sys.argv) > 2 and sys.argv[2] not in name:
        continue
    ops = re.findall(r"/\*[0-9a-f]{4,5}\*/\s+(?:@!?U?P\w+\s+)?([A-Z0-9_]+)", body)
    c = collections.Counter(ops)
    print(name, len(ops))
    print("   ", c.most_common(40))
