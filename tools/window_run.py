#!/usr/bin/env python3
"""A few incremental online-window updates on config 4 (for ncu captures).
    python tools/window_run.py --updates 30"""
import argparse
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
import torch  # noqa: E402

from paper_2303_03279_b200 import synth  # noqa: E402
from paper_2303_03279_b200.plan import DevicePlan, IncrementalWindow, pow2_scale  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--updates", type=int, default=30)
a = ap.parse_args()
c = synth.CONFIGS[4]
win, new = 50, 5
x = synth.generate(c, "cuda", trials=range(win + new * a.updates))
plan = DevicePlan(c.N, c.T, c.nfft, c.lo, c.hi, taper=c.taper, slot_capacity=win + new, device="cuda",
                  scale=pow2_scale(float(x.abs().amax()), min(c.T, c.nfft)))
iw = IncrementalWindow(plan, win, new, c.metrics)
iw.prime(x[:win])
for u in range(1, a.updates + 1):
    iw.update(x[win + new * (u - 1): win + new * u])
torch.cuda.synchronize()
print("ok")
