#!/usr/bin/env python3
"""Source-space spectra two ways on cfg3 shapes from a 306-sensor array:
(a) project the samples (M @ x, K x T columns) then K1 on the N_src sources;
(b) K1 on the sensors, then project the spectrum ring (K L nb columns).  Prints a JSON line."""
import json
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
import numpy as np  # noqa: E402
import torch  # noqa: E402

from paper_2303_03279_b200 import synth  # noqa: E402
from paper_2303_03279_b200.plan import DevicePlan, pow2_scale  # noqa: E402

c = synth.CONFIGS[3]
K, T, C, N = c.K, c.T, 306, c.N
g = torch.Generator(device="cuda").manual_seed(3)
x = torch.randn((K, C, T), generator=g, device="cuda")
M = torch.randn((N, C), generator=g, device="cuda", dtype=torch.float64) / np.sqrt(C)
ev = lambda: torch.cuda.Event(enable_timing=True)  # noqa: E731


def time_it(fn, reps=5):
    fn()
    torch.cuda.synchronize()
    a, b = ev(), ev()
    a.record()
    for _ in range(reps):
        fn()
    b.record()
    torch.cuda.synchronize()
    return a.elapsed_time(b) / reps


src_a = DevicePlan(N, T, c.nfft, c.lo, c.hi, taper=c.taper, slot_capacity=K, device="cuda",
                   scale=pow2_scale(float(x.abs().amax()) * 4, min(T, c.nfft)))
sens = DevicePlan(C, T, c.nfft, c.lo, c.hi, taper=c.taper, slot_capacity=K, device="cuda",
                  scale=pow2_scale(float(x.abs().amax()), min(T, c.nfft)))
Mf = M.float()


def path_a():
    xs = torch.matmul(Mf, x)            # [K, N, T] sources in the time domain
    src_a.spectra(xs, 0)


def path_b():
    sens.spectra(x, 0)
    Xs = sens.ring()[0][:K]
    Kk, L, nb, _ = Xs.shape
    (Xs.reshape(Kk * L * nb, C) @ M.T.to(torch.complex128)).reshape(Kk, L, nb, N)


ta, tb = time_it(path_a), time_it(path_b)
print(json.dumps({"shapes": {"K": K, "T": T, "sensors": C, "sources": N, "tapers": 3, "bins": c.n_bins},
                  "project_samples_then_K1_ms": ta, "K1_sensors_then_project_ring_ms": tb, "speedup": ta / tb}))
