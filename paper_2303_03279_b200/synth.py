"""Seeded synthetic workloads standing in for the paper's recordings
(BASELINE.json configs).  No public dataset is used by
the reference; these generators reproduce the configs' shapes, sampling rates,
signal models and value distributions.

Noise is drawn on the device per 256-node block from a generator seeded by
(config seed, block), so any node subset regenerates identically (for the
oracle) and any shard of nodes can be produced by the GPU that owns it.  The
planted couplings use small host-side tables drawn from the config seed.
"""
from __future__ import annotations

import math
from dataclasses import dataclass, field

import numpy as np
import torch

BLOCK = 256
SEVEN = ("COH", "IMAGCOHY", "PLV", "PLI", "USPLI", "WPLI", "DSWPLI")


@dataclass(frozen=True)
class Config:
    cfg: int
    N: int
    K: int
    T: int
    fs: float
    nfft: int
    lo: int
    hi: int
    taper: object
    dtype: torch.dtype
    metrics: tuple = SEVEN
    seed: int = 0
    name: str = ""

    @property
    def n_bins(self):
        return self.hi - self.lo + 1

    @property
    def n_pairs(self):
        return self.N * (self.N - 1) // 2

    @property
    def updates(self):
        """edge x freq x trial updates (P * B * K) -- BASELINE.json's metric unit."""
        return self.n_pairs * self.n_bins * self.K


def _bins(lo_hz, hi_hz, fs, nfft):
    """Nearest-bin rule (SURVEY.md conventions item 10)."""
    return int(round(lo_hz * nfft / fs)), int(round(hi_hz * nfft / fs))


CONFIGS = {
    1: Config(1, 60, 10, 500, 1000.0, 512, 0, 256, "hann", torch.float64, seed=1,
              name="sensor-space CPU-runnable ref (N=60, K=10, T=500, all 257 bins)"),
    2: Config(2, 306, 100, 1000, 1000.0, 1024, *_bins(1, 100, 1000.0, 1024), "hann", torch.float32, seed=2,
              name="MEG-sensor scale (N=306, K=100, T=1000, 1-100 Hz)"),
    3: Config(3, 2562, 60, 600, 600.0, 1024, *_bins(4, 40, 600.0, 1024), ("dpss", 2.0, 3), torch.float32,
              seed=3, name="source-space dense (N=2562, K=60, DPSS NW=2 L=3, 4-40 Hz)"),
    4: Config(4, 1024, 50, 512, 1000.0, 512, *_bins(8, 30, 1000.0, 512), "hann", torch.float32,
              metrics=("PLV", "WPLI"), seed=4,
              name="online sliding window (N=1024, K=50 window, 5 new trials/window, 8-30 Hz)"),
    5: Config(5, 10242, 100, 1000, 1000.0, 1024, *_bins(8, 13, 1000.0, 1024), "hann", torch.float32, seed=5,
              name="large all-to-all source space (N=10242, K=100, 8-13 Hz, 6 bins)"),
}
CFG4_STREAM = 1045   # trials in the online stream
CFG4_STEP = 5        # new trials per window
CFG4_WINDOWS = 200


def _gen(device, *key):
    g = torch.Generator(device=device)
    g.manual_seed(int(np.random.SeedSequence(list(key)).generate_state(1, np.uint64)[0] & ((1 << 63) - 1)))
    return g


def _planted(c: Config):
    """Host tables of planted couplings for config c (deterministic in c.seed)."""
    rng = np.random.default_rng([c.seed, 7777])
    if c.cfg == 1:
        return {"amp": rng.uniform(0.5, 2.0, (c.N, 3)), "phs": rng.uniform(0, 2 * np.pi, (c.N, 3))}
    if c.cfg == 2:
        nodes = rng.choice(c.N, size=int(round(0.2 * c.N)), replace=False)
        return {"nodes": nodes, "lag": rng.integers(0, 21, nodes.size), "gain": rng.uniform(0.5, 1.5, nodes.size),
                "theta": rng.uniform(0, 2 * np.pi, c.K)}
    if c.cfg in (3, 5):
        ncl, size, f, amp = (5, 16, 12.0, 1.0) if c.cfg == 3 else (10, 32, 10.0, 0.5)
        nodes = rng.choice(c.N, size=ncl * size, replace=False).reshape(ncl, size)
        return {"nodes": nodes, "lag": rng.uniform(0, np.pi / 2, (ncl, size)),
                "theta": rng.uniform(0, 2 * np.pi, (ncl, c.K)), "f": f, "amp": amp}
    if c.cfg == 4:
        nodes = rng.choice(c.N, size=32, replace=False).reshape(16, 2)
        return {"pairs": nodes, "theta": rng.uniform(0, 2 * np.pi, (16, CFG4_STREAM))}
    raise ValueError(c.cfg)


def generate(c: Config, device="cuda", nodes: slice | None = None, trials=None) -> torch.Tensor:
    """Samples [K, n, T] in c.dtype on ``device`` for node range ``nodes``
    (default all) and trial indices ``trials`` (default range(K); cfg4: stream
    indices < 1045)."""
    device = torch.device(device)
    n0, n1 = (0, c.N) if nodes is None else (nodes.start or 0, nodes.stop if nodes.stop is not None else c.N)
    trials = list(range(c.K)) if trials is None else list(trials)
    K = len(trials)
    t = torch.arange(c.T, device=device, dtype=torch.float64) / c.fs
    out = torch.empty((K, n1 - n0, c.T), dtype=c.dtype, device=device)
    tab = _planted(c)
    for blk in range(n0 // BLOCK, (n1 + BLOCK - 1) // BLOCK):
        b0, b1 = blk * BLOCK, min((blk + 1) * BLOCK, c.N)
        nb = b1 - b0
        burn = 200 if c.cfg == 2 else 0
        # per-trial streams so that any trial subset (cfg4 windows) regenerates identically
        e = torch.stack([torch.randn((nb, c.T + burn), generator=_gen(device, c.seed, blk, k), device=device,
                                     dtype=torch.float64) for k in trials])
        if c.cfg == 2:  # AR(2): x_t = 1.2 x_{t-1} - 0.5 x_{t-2} + e_t, 200-sample burn-in
            y = torch.zeros_like(e)
            y[..., 0] = e[..., 0]
            y[..., 1] = e[..., 1] + 1.2 * y[..., 0]
            for s_ in range(2, c.T + burn):
                y[..., s_] = e[..., s_] + 1.2 * y[..., s_ - 1] - 0.5 * y[..., s_ - 2]
            e = y[..., burn:]
        elif c.cfg == 4:  # pink: white shaped by 1/sqrt(f) in the rFFT, unit variance
            spec = torch.fft.rfft(e, dim=-1)
            f = torch.fft.rfftfreq(c.T, d=1.0 / c.fs).to(device)
            shape = torch.where(f > 0, 1.0 / torch.sqrt(f.clamp(min=1e-12)), torch.zeros_like(f))
            e = torch.fft.irfft(spec * shape, n=c.T, dim=-1)
            e = (e - e.mean(dim=-1, keepdim=True)) / e.std(dim=-1, keepdim=True)
        x = e.contiguous()
        ktr = torch.tensor(trials, device=device)
        if c.cfg == 1:
            amp = torch.tensor(tab["amp"][b0:b1], device=device)
            phs = torch.tensor(tab["phs"][b0:b1], device=device)
            for m, f in enumerate((10.0, 20.0, 40.0)):
                x += (amp[:, m:m + 1] * torch.sin(2 * math.pi * f * t[None, :] + phs[:, m:m + 1]))[None]
        elif c.cfg == 2:
            theta = torch.tensor(tab["theta"], device=device)[ktr]
            for node, lag, gain in zip(tab["nodes"], tab["lag"], tab["gain"]):
                if b0 <= node < b1:
                    x[:, node - b0] += gain * torch.sin(2 * math.pi * 10.0 * (t[None, :] - lag / c.fs)
                                                        + theta[:, None])
        elif c.cfg in (3, 5):
            theta = torch.tensor(tab["theta"], device=device)[:, ktr]
            for cl in range(tab["nodes"].shape[0]):
                for q, node in enumerate(tab["nodes"][cl]):
                    if b0 <= node < b1:
                        ph = theta[cl][:, None] + float(tab["lag"][cl, q])
                        x[:, node - b0] += tab["amp"] * torch.sin(2 * math.pi * tab["f"] * t[None, :] + ph)
        elif c.cfg == 4:
            theta = torch.tensor(tab["theta"], device=device)[:, ktr]
            for pi_, (a, b) in enumerate(tab["pairs"]):
                for node, lag in ((a, 0.0), (b, math.pi / 3)):
                    if b0 <= node < b1:
                        x[:, node - b0] += 0.5 * torch.sin(2 * math.pi * 20.0 * t[None, :] + theta[pi_][:, None] - lag)
        lo_, hi_ = max(b0, n0), min(b1, n1)
        out[:, lo_ - n0:hi_ - n0] = x[:, lo_ - b0:hi_ - b0].to(c.dtype)
    return out
