#!/usr/bin/env python3
"""A/B timing of the tensor-core kernel on a config (default 5): the fused seven-metric
call with single CTAs (CSCONN_K2_PAIR=0) and CTA pairs (=1), per-kernel ms from the
plan's event profile.  With a -DCS_TC_ABLATION build (CSCONN_LIB) also sweeps the
CSCONN_TC_DBG ablation bits given by --dbg.

    python tools/k2_ab.py --config 5 --reps 5 [--dbg 0,8,16,24,1]
"""
import argparse
import os
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
import torch  # noqa: E402

from paper_2303_03279_b200 import synth  # noqa: E402
from paper_2303_03279_b200.plan import DevicePlan, pow2_scale  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--config", type=int, default=5)
ap.add_argument("--reps", type=int, default=5)
ap.add_argument("--dbg", default="0")
ap.add_argument("--modes", default="0,1")
ap.add_argument("--metrics", default=None)
a = ap.parse_args()
c = synth.CONFIGS[a.config]
x = synth.generate(c, "cuda")
plan = DevicePlan(c.N, c.T, c.nfft, c.lo, c.hi, taper=c.taper, slot_capacity=c.K, device="cuda",
                  scale=pow2_scale(float(x.abs().amax()), min(c.T, c.nfft)))
slots = torch.arange(c.K, dtype=torch.int32, device="cuda")
metrics = tuple(a.metrics.split(",")) if a.metrics else c.metrics
outs = plan.alloc_outputs(metrics, c.n_bins)
plan.spectra(x, 0)
for dbg in a.dbg.split(","):
    os.environ["CSCONN_TC_DBG"] = dbg
    for mode in a.modes.split(","):
        os.environ["CSCONN_K2_PAIR"] = mode
        plan.pair_metrics(slots, metrics, 0, c.n_bins, outputs=outs)  # warm
        torch.cuda.synchronize()
        plan.set_profiling(True)
        plan.profile()
        for _ in range(a.reps):
            plan.pair_metrics(slots, metrics, 0, c.n_bins, outputs=outs)
        torch.cuda.synchronize()
        prof = plan.profile()
        plan.set_profiling(False)
        per = {k: round(v[0] / max(v[1], 1), 4) for k, v in prof.items()}
        print(f"dbg={dbg} pair={mode}: {per}", flush=True)
