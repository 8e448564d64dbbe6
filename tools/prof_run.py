#!/usr/bin/env python3
"""One pass of the hot path on a config (for ncu captures): K1 + pair kernels.

    python tools/prof_run.py --config 5 --metrics IMAGCOHY,PLI --reps 2
"""
import argparse
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
import torch  # noqa: E402

from paper_2303_03279_b200 import synth  # noqa: E402
from paper_2303_03279_b200.plan import DevicePlan, pow2_scale  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--config", type=int, default=5)
ap.add_argument("--metrics", default=None)
ap.add_argument("--reps", type=int, default=2)
ap.add_argument("--nodes", type=int, default=None, help="use the first n nodes only")
a = ap.parse_args()
c = synth.CONFIGS[a.config]
N = a.nodes or c.N
x = synth.generate(c, "cuda", nodes=slice(0, N))
plan = DevicePlan(N, c.T, c.nfft, c.lo, c.hi, taper=c.taper, slot_capacity=c.K, device="cuda",
                  scale=pow2_scale(float(x.abs().amax()), min(c.T, c.nfft)))
slots = torch.arange(c.K, dtype=torch.int32, device="cuda")
metrics = tuple(a.metrics.split(",")) if a.metrics else c.metrics
outs = plan.alloc_outputs(metrics, c.n_bins)
for _ in range(a.reps):
    plan.spectra(x, 0)
    plan.pair_metrics(slots, metrics, 0, c.n_bins, outputs=outs)
torch.cuda.synchronize()
print("ok fallback", plan.fallback_count())
