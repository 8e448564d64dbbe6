#!/usr/bin/env python3
"""Per-tile fixed cost of the phase-lag kernel: time it over 1..6 bins of cfg5 and
fit ms = a + b * bins (a = tile setup / pipeline fill / band store, b = per bin)."""
import sys
from pathlib import Path
sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
import numpy as np, torch  # noqa: E401,E402
from paper_2303_03279_b200 import synth  # noqa: E402
from paper_2303_03279_b200.plan import DevicePlan, pow2_scale  # noqa: E402
c = synth.CONFIGS[5]
x = synth.generate(c, "cuda")
plan = DevicePlan(c.N, c.T, c.nfft, c.lo, c.hi, taper=c.taper, slot_capacity=c.K, device="cuda",
                  scale=pow2_scale(float(x.abs().amax()), min(c.T, c.nfft)))
plan.spectra(x, 0)
slots = torch.arange(c.K, dtype=torch.int32, device="cuda")
ms = []
for nb in range(1, 7):
    outs = plan.alloc_outputs(("PLI", "WPLI", "USPLI", "DSWPLI", "IMAGCOHY"), nb)
    for _ in range(2):
        plan.pair_metrics(slots, ("PLI", "WPLI", "USPLI", "DSWPLI", "IMAGCOHY"), 0, nb, outputs=outs)
    plan.set_profiling(True); plan.profile()
    for _ in range(5):
        plan.pair_metrics(slots, ("PLI", "WPLI", "USPLI", "DSWPLI", "IMAGCOHY"), 0, nb, outputs=outs)
    torch.cuda.synchronize()
    p = plan.profile(); plan.set_profiling(False)
    ms.append(p["pairs_lag"][0] / p["pairs_lag"][1])
    del outs
b, a = np.polyfit(np.arange(1, 7), ms, 1)
print("ms per bins 1..6:", [round(v, 3) for v in ms], "fit: fixed %.3f ms + %.3f ms/bin" % (a, b))
