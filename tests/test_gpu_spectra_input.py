"""Spectra handed in by the caller (accumulate_spectra, reference spectral.py:244-261)
instead of computed by K1.

* Arbitrary complex spectra, including non-real values at DC and Nyquist: the reference
  folds them like any other bin, so the phase-lag kernel must not assume those bins are
  exactly real (that shortcut only holds for spectra from trial_spectra, where DC := 0
  and the Nyquist bin of a real signal is real).
* Spectra built to straddle the exact-sign guard: per trial, every channel shares one
  phase up to offsets that make |Im(X_i conj X_j)| / (|X_i||X_j|) log-uniform in
  [1e-10, 1e-4] -- around the fp32 bound g = 1.25 (2 + 2L) 2^-24 ~ 3e-7 relative to
  M_i M_j -- with magnitudes that vary by trial, so both sides of the bound occur and K PLI
  must still equal the reference's exactly (the relative offsets stay far above the
  1e-13 flush, so no entry is rounding-defined).
"""
import os

import numpy as np
import pytest

import oracle as O
from paper_2303_03279_b200 import metrics as M
from paper_2303_03279_b200 import spectral as S

pytestmark = pytest.mark.gpu
FAM = {"IMAGCOHY": (M.imagcohy_bins, O.imagcohy_bins, 1e-4), "PLI": (M.pli_bins, O.pli_bins, 1e-3),
       "WPLI": (M.wpli_bins, O.wpli_bins, 1e-3), "USPLI": (M.uspli_bins, O.uspli_bins, 1e-3),
       "DSWPLI": (M.dswpli_bins, O.dswpli_bins, 1e-3), "COH": (M.coh_bins, O.coh_bins, 1e-4),
       "PLV": (M.plv_bins, O.plv_bins, 1e-4)}


def _fold(spectra, C, nfft):
    acc = S.SpectrumSet(C, nfft)
    ref = O.Sums(C, nfft // 2 + 1)
    for s in spectra:
        S.accumulate_spectra(acc, s)
        O.accumulate(ref, s)
    return acc, ref


def _check(acc, ref, K, exact_pli=True):
    for m, (mine, theirs, tol) in FAM.items():
        got, want = mine(acc), theirs(ref)
        assert got.shape == want.shape, m
        err = np.abs(got - want)
        assert err.max() <= tol, f"{m}: max err {err.max():.3g} at {np.unravel_index(err.argmax(), err.shape)}"
    if exact_pli:
        assert np.array_equal(np.rint(M.pli_bins(acc) * K), np.rint(O.pli_bins(ref) * K))


def test_complex_dc_and_nyquist_bins():
    """Random complex spectra in every bin, DC (0) and Nyquist (nfft / 2) included."""
    rng = np.random.default_rng(31)
    K, C, nfft = 23, 14, 16
    spectra = [rng.standard_normal((C, nfft // 2 + 1)) + 1j * rng.standard_normal((C, nfft // 2 + 1))
               for _ in range(K)]
    acc, ref = _fold(spectra, C, nfft)
    _check(acc, ref, K)
    # the DC and Nyquist columns carry real phase-lag information here
    assert np.abs(O.pli_bins(ref)[:, 0]).max() > 0 and np.abs(O.pli_bins(ref)[:, -1]).max() > 0


def _straddling(K=40, C=48, nfft=32, seed=77):
    rng = np.random.default_rng(seed)
    nb = nfft // 2 + 1
    spectra = []
    for _ in range(K):
        base = rng.uniform(0, 2 * np.pi, nb)                      # shared phase per bin
        off = 10.0 ** rng.uniform(-10, -4, (C, nb)) * rng.choice([-1.0, 1.0], (C, nb))
        mag = rng.uniform(0.05, 1.0, (C, nb))                    # |X| varies by trial (M_i = max)
        spectra.append(mag * np.exp(1j * (base[None, :] + off)))
    return spectra


def test_spectra_straddling_the_exact_sign_guard():
    K, C, nfft = 40, 48, 32
    acc, ref = _fold(_straddling(K, C, nfft), C, nfft)
    _check(acc, ref, K)


def test_straddling_spectra_negative_control():
    """The same data with the guard bound cut to 1 / 50 (about the typical instead of the
    worst-case fp32 error): trials whose fp32 sign really is wrong are trusted and K PLI
    must differ from the reference somewhere -- the data above contains genuine fp32 sign
    flips, which the guard sends to fp64."""
    K, C, nfft = 40, 48, 32
    os.environ["CSCONN_GUARD_G"] = "0.02"
    try:
        acc, ref = _fold(_straddling(K, C, nfft), C, nfft)
        got = np.rint(M.pli_bins(acc) * K)
    finally:
        del os.environ["CSCONN_GUARD_G"]
    n_bad = int((got != np.rint(O.pli_bins(ref) * K)).sum())
    print(f"guard at 0.02x: {n_bad} K*PLI mismatches")
    assert n_bad >= 1


def test_bins_and_count_against_the_reference():
    """accumulate_spectra with column subsets (slice / index array) and a count=False
    back-fill, replayed against vectors from the unmodified reference
    (tests/golden/make_golden_bins.py)."""
    from pathlib import Path
    g = np.load(Path(__file__).resolve().parent / "golden" / "bins_count.npz")
    spectra = g["spectra"]
    K, C, nb = spectra.shape
    acc = S.SpectrumSet(C, 2 * (nb - 1))
    for i in range(int(g["n_plan"])):
        b = g[f"plan_{i}_bins"]
        bins = None if (b.size == 1 and b[0] == -1) else b
        S.accumulate_spectra(acc, spectra[int(g[f"plan_{i}_trial"])], bins=bins, count=bool(g[f"plan_{i}_count"]))
    assert acc.n_trials_accumulated == int(g["n_trials"])
    fns = {"COHY": M.cohy_bins, **{m: f[0] for m, f in FAM.items()}}
    tol = {"COHY": 1e-4, **{m: f[2] for m, f in FAM.items()}}
    for m, fn in fns.items():
        got, want = fn(acc), g["bins_" + m]
        assert got.shape == want.shape, m
        err = np.abs(got - want)
        assert err.max() <= tol[m], f"{m}: max err {err.max():.3g} at {np.unravel_index(err.argmax(), err.shape)}"
    kk = int(g["n_trials"])
    assert np.array_equal(np.rint(M.pli_bins(acc) * kk), np.rint(g["bins_PLI"] * kk))


@pytest.mark.parametrize("metric", ["COH", "IMAGCOHY", "PLV", "PLI", "USPLI", "WPLI", "DSWPLI", "COHY"])
def test_compute_metric_epochs_of_different_lengths(metric):
    """compute_metric over epochs of different lengths (some cropped to nfft, some padded):
    every epoch is conditioned on its own, as in the reference (metrics.py:541-551)."""
    from paper_2303_03279_b200 import EpochMatrix, MetricId, compute_metric
    rng = np.random.default_rng(5)
    C, nfft = 9, 128
    data = [rng.standard_normal((C, T)) for T in (90, 128, 200, 64, 128, 300, 150)]
    data[2][3] = 0.5 * data[2][1]
    net = compute_metric([EpochMatrix(d, 500.0) for d in data], MetricId.parse(metric), nfft)
    want, _ = O.compute(data, nfft, 0, nfft // 2, (metric,))
    ref = want[metric]["band"] if metric != "COHY" else np.abs(want[metric]["cband"])
    tol = 1e-4 if metric in ("COH", "IMAGCOHY", "PLV", "COHY") else 1e-3
    assert np.abs(np.asarray(net.weights) - ref).max() <= tol
