#!/usr/bin/env python3
"""Generate golden vectors by running the UNMODIFIED reference (connstream).

Run in the build container (the reference is importable from
/root/reference/pkg/src; it is absent on the GPU box, so the vectors are
committed as small .npz fixtures next to this script):

    python tests/golden/make_golden.py

Every case stores its inputs and the reference's per-bin outputs for all eight
spectral metrics.  Tapered cases compute the tapered spectra outside the
reference (the documented extension: demean -> taper -> zero-pad -> rfft -> DC:=0)
and then call the reference's own accumulate_spectra / _fold_csd / *_bins.
"""
from __future__ import annotations

import sys
from pathlib import Path

import numpy as np

REF = Path("/root/reference/pkg/src")
sys.path.insert(0, str(REF))

from connstream.core import EpochMatrix, FrequencyBand, MetricId  # noqa: E402
from connstream import spectral as S  # noqa: E402
from connstream import metrics as M  # noqa: E402
from connstream.simulate import SimulationSpec, generate  # noqa: E402

OUT = Path(__file__).resolve().parent
NAMES = ["COHY", "COH", "IMAGCOHY", "PLV", "PLI", "USPLI", "WPLI", "DSWPLI"]


def tapered_spectra(data, nfft, taper):
    seg = S._crop_pad_demean(data, nfft)
    n = min(data.shape[1], nfft)
    seg = seg.copy()
    seg[:, :n] *= taper[None, :]
    out = np.fft.rfft(seg, n=nfft, axis=1)
    out[:, 0] = 0.0
    return out


def run_case(name, epochs, nfft, lo, hi, taper=None, mode="fixed"):
    """epochs: float array [K, C, T]."""
    K, C, _ = epochs.shape
    acc = S.SpectrumSet(C, nfft)
    for k in range(K):
        ep = EpochMatrix(data=epochs[k], sfreq=1000.0, trial_index=k)
        if taper is None:
            S.accumulate_epoch(acc, ep, mode=mode)
        elif taper.ndim == 1:
            S.accumulate_spectra(acc, tapered_spectra(ep.data, nfft, taper))
        else:  # multitaper: mean CSD/PSD over tapers, reference fold
            csd = np.zeros((acc.n_pairs, acc.n_bins), dtype=np.complex128)
            psd = np.zeros((C, acc.n_bins))
            for tp in taper:
                c, p = S.trial_csd_psd(tapered_spectra(ep.data, nfft, tp), C)
                csd += c
                psd += p
            S._fold_csd(acc, csd / len(taper), psd / len(taper))
    band = FrequencyBand(lo, hi, 1.0)
    rec = {"epochs": epochs, "nfft": nfft, "lo": lo, "hi": hi,
           "taper": np.zeros(0) if taper is None else taper, "mode": np.array(mode)}
    for nm in NAMES:
        try:
            rec["bins_" + nm] = M._SPECTRAL_BINS[MetricId[nm]](acc, band)
        except Exception:  # DegenerateTrialCountError (USPLI, K<2)
            rec["bins_" + nm] = np.zeros(0)
        try:
            net = M.finalize_spectral(acc, MetricId[nm], band)
            rec["band_" + nm] = net.weights
            if nm == "COHY":
                rec["cband_COHY"] = net.complex_weights
        except Exception:
            rec["band_" + nm] = np.zeros(0)
    np.savez_compressed(OUT / f"{name}.npz", **rec)
    print("wrote", name, {k: np.shape(v) for k, v in rec.items() if k.startswith("bins_COH")})


def main():
    rng = np.random.default_rng(20260101)
    # tests/test_metrics.py:32-39 shape (6 trials x 4 ch x 32 samples, nfft 32)
    run_case("rect_small", rng.standard_normal((6, 4, 32)), 32, 0, 16)
    # tests/test_acceptance.py:75-96 shape (20 x 8 x 64, nfft 64)
    run_case("rect_accept", rng.standard_normal((20, 8, 64)), 64, 0, 32)
    # crop (T > nfft), odd K, band subset
    run_case("rect_crop_oddk", rng.standard_normal((7, 9, 100)), 64, 3, 20)
    # zero-pad (T < nfft), K=1 (USPLI degenerate)
    run_case("rect_pad_k1", rng.standard_normal((1, 5, 40)), 64, 1, 10)
    # cfg1-like: Hann taper, all bins incl. DC and Nyquist, float64 sinusoids + noise
    t = np.arange(500) / 1000.0
    K, C = 10, 12
    amps = rng.uniform(0.5, 2.0, (C, 3))
    phs = rng.uniform(0, 2 * np.pi, (C, 3))
    base = sum(amps[:, m:m + 1] * np.sin(2 * np.pi * f * t[None, :] + phs[:, m:m + 1])
               for m, f in enumerate((10.0, 20.0, 40.0)))
    ep1 = base[None] + rng.standard_normal((K, C, 500))
    run_case("hann_cfg1like", ep1, 512, 0, 256, taper=np.hanning(500))
    # multitaper DPSS NW=2 L=3, float32-valued signals
    from scipy.signal import windows
    ep3 = rng.standard_normal((8, 12, 120)).astype(np.float32).astype(np.float64)
    run_case("dpss_small", ep3, 128, 5, 30, taper=windows.dpss(120, 2.0, Kmax=3))
    # zero-lag scaled copies + a dead (constant) channel + an independent channel
    tt = np.arange(96) / 600.0
    zl = []
    for k in range(12):
        s = np.sin(2 * np.pi * 18.0 * tt + rng.uniform(0, 2 * np.pi)) + 0.0 * tt
        zl.append(np.vstack([s, 0.7 * s, 0.4 * s, np.full(96, 3.0), rng.standard_normal(96)]))
    run_case("zerolag_dead", np.array(zl), 128, 0, 64)
    run_case("zerolag_dead_hann", np.array(zl), 128, 10, 30, taper=np.hanning(96))

    # reference threshold fixture inputs (pkg/scripts/export_threshold_fixtures.py:38-58)
    rec, info = generate(SimulationSpec(n_trials=40), seed=2024)
    data = rec.data[: len(rec.data_channels)].astype(np.float64)
    T = info["trial_samples"]
    eps = np.array([data[:, m:m + T] for m in info["markers"]])
    run_case("sim2024_thresh", eps, 600, 15, 21)
    # the reference's threshold fixture selections (export_threshold_fixtures.py:47-58),
    # recomputed with the reference: normalised band networks, kept (i, j) sets
    from connstream.core import normalize_network, threshold_network
    rec2 = dict(np.load(OUT / "sim2024_thresh.npz"))
    eps_m = [EpochMatrix(data=e, sfreq=1000.0, trial_index=k) for k, e in enumerate(eps)]
    for nm in ("COH", "IMAGCOHY"):
        dense = normalize_network(M.compute_metric(eps_m, MetricId[nm], 600, FrequencyBand(15, 21, 1.0)))
        rec2["norm_" + nm] = dense.weights
        for f in (0.05, 0.10, 0.25):
            t = threshold_network(dense, f)
            rec2[f"thresh_{nm}_{f:.2f}"] = np.stack([t.edge_i, t.edge_j], 1)
    np.savez_compressed(OUT / "sim2024_thresh.npz", **rec2)

    # time-domain metrics (metrics.py:140-260) through the reference's compute_metric
    td = rng.standard_normal((5, 6, 80))
    td[:, 3] = 2.5                                   # a zero-variance channel
    td[:, 4] = np.roll(td[:, 1], 3, axis=1)          # a lagged copy
    eps_td = [EpochMatrix(data=e, sfreq=100.0, trial_index=k) for k, e in enumerate(td)]
    rec3 = {"epochs": td}
    net = M.compute_metric(eps_td, MetricId.COR, 64)
    rec3["cor_w"], rec3["cor_warn"] = net.weights, np.array(list(net.warnings))
    for ml in (10, None):
        net = M.compute_metric(eps_td, MetricId.XCOR, 64, max_lag=ml)
        key = "all" if ml is None else str(ml)
        rec3["xcor_w_" + key], rec3["xcor_lag_" + key] = net.weights, net.lags
    np.savez_compressed(OUT / "timedomain.npz", **rec3)
    print("wrote timedomain")

    # welch mode (spectral.py:264-283): 3 segments of 64 (T = 200, 8 samples dropped),
    # and a short-trial fallback to fixed mode (T < 2 nfft)
    run_case("welch3", rng.standard_normal((6, 7, 200)), 64, 2, 20, mode="welch")
    run_case("welch_short", rng.standard_normal((5, 4, 100)), 64, 0, 32, mode="welch")


if __name__ == "__main__":
    main()
