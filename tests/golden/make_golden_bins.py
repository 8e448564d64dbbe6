#!/usr/bin/env python3
"""Golden vectors for accumulate_spectra's ``bins`` / ``count`` arguments, made by the
UNMODIFIED reference (spectral.py:216-261: a fold restricted to some columns, and a
count=False back-fill of columns for trials already counted, as a live band change
does).  Run in the build container; the .npz is committed:

    python tests/golden/make_golden_bins.py
"""
from __future__ import annotations

import sys
from pathlib import Path

import numpy as np

sys.path.insert(0, "/root/reference/pkg/src")
from connstream import metrics as M  # noqa: E402
from connstream import spectral as S  # noqa: E402

OUT = Path(__file__).resolve().parent
NAMES = ["COHY", "COH", "IMAGCOHY", "PLV", "PLI", "USPLI", "WPLI", "DSWPLI"]
FN = {"COHY": M.cohy_bins, "COH": M.coh_bins, "IMAGCOHY": M.imagcohy_bins, "PLV": M.plv_bins,
      "PLI": M.pli_bins, "USPLI": M.uspli_bins, "WPLI": M.wpli_bins, "DSWPLI": M.dswpli_bins}


def main():
    rng = np.random.default_rng(2026)
    C, nfft, K = 7, 32, 9
    nb = nfft // 2 + 1
    spectra = rng.standard_normal((K, C, nb)) + 1j * rng.standard_normal((K, C, nb))
    spectra[:, :, 0] = spectra[:, :, 0].real          # trial_spectra-like DC / Nyquist ...
    spectra[:, 3, :] = 0.6 * spectra[:, 1, :]         # ... a zero-lag copy ...
    spectra[2, 5, :] = 0.0                            # ... and a channel silent in one trial
    # the fold plan: (trial, bins, count); bins as a [lo, hi) slice or an index array
    plan = [(0, None, True), (1, None, True), (2, (2, 9), True), (3, (2, 9), True),
            (2, [0, 1] + list(range(9, nb)), False),  # back-fill trial 2's other columns
            (4, np.array([1, 3, 5, 7]), True), (5, None, True), (6, (0, 5), True),
            (7, None, True), (8, (5, nb), True)]
    acc = S.SpectrumSet(C, nfft)
    for k, b, cnt in plan:
        bins = slice(*b) if isinstance(b, tuple) else (None if b is None else np.asarray(b))
        S.accumulate_spectra(acc, spectra[k], bins=bins, count=cnt)
    out = {"spectra": spectra, "n_trials": acc.n_trials_accumulated}
    for i, (k, b, cnt) in enumerate(plan):
        out[f"plan_{i}_trial"] = k
        out[f"plan_{i}_count"] = cnt
        out[f"plan_{i}_bins"] = (np.array([-1]) if b is None else
                                 np.arange(*b) if isinstance(b, tuple) else np.asarray(b))
    out["n_plan"] = len(plan)
    for m in NAMES:
        out["bins_" + m] = FN[m](acc)
    np.savez_compressed(OUT / "bins_count.npz", **out)
    print("bins_count.npz: K =", acc.n_trials_accumulated)


if __name__ == "__main__":
    main()
