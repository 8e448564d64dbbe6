"""ConnectivityEngine fed trials of different lengths, as the reference's engine
accepts them (metrics.py:335-357: every trial goes through accumulate_epoch on its
own; the spontaneous-mode pipeline hands it a shorter last block, pipeline.py:276-281).

* fixed mode: each trial cropped / zero-padded to nfft on its own;
* welch mode: the per-trial rule of spectral.py:272-286 -- n_samples >= 2 nfft folds
  the mean CSD of its n_samples // nfft segments, shorter trials fold like fixed mode --
  with segment counts that grow past the ring's (the ring is widened) and a
  trial-window rebuild that re-folds the cached first segments (metrics.py:450-460);
* multitaper (DPSS) with each length's own taper stack;
* XCOR without a max_lag: each trial's own n_samples - 1 (metrics.py:385).
Every finalize is compared with the oracle over exactly the trials folded so far.
"""
import copy

import numpy as np
import pytest

import oracle as O
from paper_2303_03279_b200 import ConnectivityEngine, EpochMatrix, FrequencyBand, MetricId
from paper_2303_03279_b200.plan import make_taper

pytestmark = pytest.mark.gpu
SPECTRAL = ("COH", "IMAGCOHY", "PLV", "PLI", "USPLI", "WPLI", "DSWPLI", "COHY")
TOL = {"COH": 1e-4, "IMAGCOHY": 1e-4, "PLV": 1e-4, "PLI": 1e-3, "USPLI": 1e-3, "WPLI": 1e-3, "DSWPLI": 1e-3,
       "COHY": 1e-4}


def _data(lengths, C=10, seed=0):
    rng = np.random.default_rng(seed)
    out = []
    for T in lengths:
        x = rng.standard_normal((C, T))
        x[4] = 0.7 * x[1]                    # zero-lag copy: exact zeros on the guard path
        t = np.arange(T)
        x[6:9] += np.sin(2 * np.pi * 0.11 * t[None, :] + np.array([[0.0], [0.4], [0.9]]) + rng.uniform(0, 6))
        out.append(x)
    return out


def _want(acc, metric):
    pb = {"COH": O.coh_bins, "IMAGCOHY": O.imagcohy_bins, "PLV": O.plv_bins, "PLI": O.pli_bins,
          "USPLI": O.uspli_bins, "WPLI": O.wpli_bins, "DSWPLI": O.dswpli_bins, "COHY": O.cohy_bins}[metric](acc)
    w, cw = O.band_reduce(metric, pb)
    return np.abs(cw) if metric == "COHY" else w


def _band(acc, lo, hi):
    """Oracle sums restricted to bins [lo, hi]."""
    sub = copy.copy(acc)
    for k in ("csd_sum", "psd_sum", "plv_sum", "pli_sum", "abs_im_sum"):
        setattr(sub, k, getattr(acc, k)[:, lo:hi + 1])
    return sub


def _fold(acc, ep, nfft, mode, taper=None):
    if mode == "welch" and ep.shape[1] >= 2 * nfft:
        O.accumulate_multitaper(acc, np.stack([O.trial_spectra(s, nfft) for s in O.segments(ep, nfft)]))
    elif taper is not None:
        tp = make_taper(taper, min(ep.shape[1], nfft))
        O.accumulate_multitaper(acc, np.stack([O.trial_spectra(ep, nfft, t) for t in tp]))
    else:
        O.accumulate(acc, O.trial_spectra(ep, nfft))


@pytest.mark.parametrize("storage,cap", [(True, 64), (False, 64), (True, 1)])
def test_fixed_mode_trials_of_different_lengths(storage, cap):
    C, nfft, sfreq = 10, 128, 250.0
    lengths = (100, 128, 256, 60, 128, 300, 131)
    data = _data(lengths, C)
    eng = ConnectivityEngine(C, nfft, sfreq, storage_mode=storage, slot_capacity=cap)
    acc = O.Sums(C, nfft // 2 + 1)
    lo, hi = 4, 30
    band = FrequencyBand(lo, hi, sfreq / nfft)
    for k, x in enumerate(data):
        metric = SPECTRAL[k % len(SPECTRAL)]
        net = eng.update_and_finalize(EpochMatrix(x, sfreq, trial_index=k), MetricId.parse(metric), band)
        _fold(acc, x, nfft, "fixed")
        want = _want(_band(acc, lo, hi), metric)
        err = np.abs(np.asarray(net.weights) - want).max()
        assert err <= TOL[metric], (k, metric, err)
    for metric in SPECTRAL:
        net = eng.finalize(MetricId.parse(metric), band)
        assert np.abs(np.asarray(net.weights) - _want(_band(acc, lo, hi), metric)).max() <= TOL[metric], metric
    net = eng.finalize(MetricId.COR, band)
    assert np.abs(np.asarray(net.weights) - O.cor(data)[0]).max() <= 1e-9


@pytest.mark.parametrize("cap", [64, 1])
def test_welch_mode_segment_counts_grow_past_the_ring(cap):
    """First trial shorter than 2 nfft (a one-segment ring), then 2, 4 and 3 segments
    and a short trial again; rebuild_last re-folds the cached first segments.  cap = 1:
    the ring also doubles its slots while it is widened."""
    C, nfft, sfreq = 10, 64, 250.0
    lengths = (100, 130, 256, 64, 200, 90)
    data = _data(lengths, C, seed=3)
    eng = ConnectivityEngine(C, nfft, sfreq, storage_mode=True, spectral_mode="welch", slot_capacity=cap)
    acc = O.Sums(C, nfft // 2 + 1)
    lo, hi = 2, 20
    band = FrequencyBand(lo, hi, sfreq / nfft)
    for k, x in enumerate(data):
        metric = SPECTRAL[(3 * k) % len(SPECTRAL)]
        net = eng.update_and_finalize(EpochMatrix(x, sfreq, trial_index=k), MetricId.parse(metric), band)
        _fold(acc, x, nfft, "welch")
        err = np.abs(np.asarray(net.weights) - _want(_band(acc, lo, hi), metric)).max()
        assert err <= TOL[metric], (k, metric, err)
    # the reference's trial-window rebuild re-adds the kept trials from the cache:
    # welch trials fold their first segment only, as fixed-mode spectra
    eng.rebuild_last(4)
    acc = O.Sums(C, nfft // 2 + 1)
    for x in data[-4:]:
        O.accumulate(acc, O.trial_spectra(O.segments(x, nfft)[0] if x.shape[1] >= 2 * nfft else x, nfft))
    for metric in SPECTRAL:
        net = eng.finalize(MetricId.parse(metric), band)
        err = np.abs(np.asarray(net.weights) - _want(_band(acc, lo, hi), metric)).max()
        assert err <= TOL[metric], (metric, err)


def test_multitaper_trials_of_different_lengths():
    C, nfft, sfreq = 10, 128, 250.0
    taper = ("dpss", 2.0, 3)
    lengths = (128, 90, 200, 128)
    data = _data(lengths, C, seed=5)
    eng = ConnectivityEngine(C, nfft, sfreq, storage_mode=True, taper=taper)
    acc = O.Sums(C, nfft // 2 + 1)
    for k, x in enumerate(data):
        eng.add_trial(EpochMatrix(x, sfreq, trial_index=k))
        _fold(acc, x, nfft, "fixed", taper)
    band = FrequencyBand(3, 25, sfreq / nfft)
    for metric in SPECTRAL:
        net = eng.finalize(MetricId.parse(metric), band)
        err = np.abs(np.asarray(net.weights) - _want(_band(acc, 3, 25), metric)).max()
        assert err <= TOL[metric], (metric, err)


def test_xcor_uses_each_trials_own_max_lag():
    C, nfft, sfreq = 9, 64, 250.0
    lengths = (50, 80, 33)
    data = _data(lengths, C, seed=9)
    eng = ConnectivityEngine(C, nfft, sfreq, storage_mode=True)
    for k, x in enumerate(data):
        eng.add_trial(EpochMatrix(x, sfreq, trial_index=k))
    net = eng.finalize(MetricId.XCOR, FrequencyBand(1, 5, sfreq / nfft))
    pi, pj = O.pair_index(C)
    pk = np.zeros(len(pi))
    for x in data:
        for q in range(len(pi)):
            pk[q] += O.xcor_pair(x[pi[q]], x[pj[q]], x.shape[1] - 1)[0]
    assert np.abs(np.asarray(net.weights) - np.abs(pk / len(data))).max() <= 1e-9
