#!/usr/bin/env python3
"""Time the device COR / XCOR on a config's shapes and print a JSON line.

    python tools/bench_timedomain.py --config 2 --trials 10
"""
import argparse
import json
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
import torch  # noqa: E402

from paper_2303_03279_b200 import synth, timedomain  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--config", type=int, default=2)
ap.add_argument("--trials", type=int, default=10)
ap.add_argument("--max-lag", type=int, default=20)
a = ap.parse_args()
c = synth.CONFIGS[a.config]
x = synth.generate(c, "cuda").double()[: a.trials]
K, C, T = x.shape
out = {"config": a.config, "N": C, "T": T, "trials": K, "max_lag": a.max_lag}
for name, fn in (("COR", lambda: timedomain.cor_sums(list(x), C)),
                 ("XCOR", lambda: timedomain.xcor_sums(list(x), C, a.max_lag))):
    fn()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    fn()
    e1.record()
    torch.cuda.synchronize()
    ms = e0.elapsed_time(e1)
    P = C * (C - 1) // 2
    out[name] = {"ms_per_trial": ms / K, "pair_trials_per_s": P * K / (ms * 1e-3)}
print(json.dumps(out))
