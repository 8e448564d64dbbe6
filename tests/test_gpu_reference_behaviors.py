"""Behaviours the reference's own metric tests pin (reference pkg/tests/test_metrics.py,
TestCor / TestXcor / TestEngine / TestConvergence), restated on this package's
public API with independent data and checked against the oracle where a number is
involved: COR and XCOR (metrics.py:141-260), the engine's time-domain switch and
back-fill rules, reset, band hints and the FFT-count contract (metrics.py:285-460),
and convergence_curve (metrics.py:501-528)."""
import numpy as np
import pytest

import oracle as O
from paper_2303_03279_b200 import ConnectivityEngine, EpochMatrix, FrequencyBand, MetricId, compute_metric
from paper_2303_03279_b200 import metrics as M
from paper_2303_03279_b200 import spectral as S
from paper_2303_03279_b200.core import ParameterError

pytestmark = pytest.mark.gpu


def _epochs(K, C, T, seed, sfreq=600.0):
    rng = np.random.default_rng(seed)
    return [EpochMatrix(rng.standard_normal((C, T)), sfreq, trial_index=k) for k in range(K)]


# -- COR (metrics.py:141-177) ---------------------------------------------------
def test_cor_hand_computed_value():
    # x = (0, 1, 2, 3), y = (0, 2, 1, 3): cov = 4, var = 5 each -> r = 0.8
    d = np.array([[0.0, 1.0, 2.0, 3.0], [0.0, 2.0, 1.0, 3.0]])
    assert M.cor([EpochMatrix(d, 20.0)]).weights[0] == pytest.approx(0.8, abs=1e-14)


def test_cor_mean_over_trials_against_oracle():
    eps = _epochs(6, 5, 33, seed=101)
    got = M.cor(eps).weights
    want, dead = O.cor([e.data for e in eps])
    assert not dead
    assert np.abs(got - want).max() <= 1e-12


def test_cor_zero_variance_channel_warns():
    d = np.vstack([np.arange(20.0), np.full(20, 2.5), np.sin(np.arange(20.0))])
    net = M.cor([EpochMatrix(d, 20.0)])
    assert net.weights[0] == 0.0 and net.weights[2] == 0.0        # pairs (0,1) and (1,2)
    assert any("zero-variance" in w and "1" in w for w in net.warnings)


@pytest.mark.parametrize("seed", range(6))
def test_cor_bounded_and_duplicate_is_one(seed):
    d = np.random.default_rng(seed).standard_normal((4, 19))
    assert np.all(np.abs(M.cor([EpochMatrix(d, 20.0)]).weights) <= 1.0)
    dup = np.vstack([d[2], d[2]])
    assert M.cor([EpochMatrix(dup, 20.0)]).weights[0] == pytest.approx(1.0, abs=1e-12)


# -- XCOR (metrics.py:180-260) --------------------------------------------------
def test_xcor_pair_recovers_a_known_delay():
    base = np.random.default_rng(8).standard_normal(300)
    d = 9
    x, y = base[30:-30], np.roll(base, d)[30:-30]    # y lags x by d samples
    v, lag = M.xcor_pair(x, y, 20)
    assert lag == -d and v > 0.9                      # negative lag: x leads


def test_xcor_pair_identical_constant_and_bound():
    x = np.random.default_rng(9).standard_normal(70)
    v, lag = M.xcor_pair(x, x.copy(), 15)
    assert v == pytest.approx(1.0, abs=1e-10) and lag == 0
    assert M.xcor_pair(np.full(24, 4.0), np.arange(24.0), 6) == (0.0, 0)
    with pytest.raises(ParameterError):
        M.xcor_pair(np.ones(10), np.ones(10), 10)


def test_xcor_pair_methods_agree_with_oracle():
    rng = np.random.default_rng(12)
    for _ in range(6):
        x, y = rng.standard_normal(45), rng.standard_normal(45)
        ml = int(rng.integers(1, 44))
        ov, ol = O.xcor_pair(x, y, ml)
        for method in ("fft", "direct"):
            v, l = M.xcor_pair(x, y, ml, method=method)
            assert v == pytest.approx(ov, abs=1e-10) and l == ol


def test_xcor_network_mean_peak_and_lag():
    eps = _epochs(4, 4, 50, seed=13)
    net = M.xcor(eps, max_lag=12)
    w, lags = O.xcor([e.data for e in eps], max_lag=12)
    assert np.abs(net.weights - w).max() <= 1e-10
    assert np.array_equal(np.asarray(net.lags), lags)


# -- engine rules (metrics.py:285-460) ------------------------------------------
def test_late_switch_to_xcor_backfills_from_the_cache():
    eps = _epochs(5, 4, 45, seed=14)
    band = FrequencyBand(0, 5, 1.0)
    eng = ConnectivityEngine(4, 48, 600.0, storage_mode=True, max_lag=11)
    for e in eps:
        eng.update_and_finalize(e, MetricId.PLV, band)
    net = eng.finalize(MetricId.XCOR, band)
    w, lags = O.xcor([e.data for e in eps], max_lag=11)
    assert np.abs(net.weights - w).max() <= 1e-10
    assert np.array_equal(np.asarray(net.lags), lags)


def test_late_switch_to_xcor_without_storage_raises():
    eng = ConnectivityEngine(4, 32, 600.0, storage_mode=False)
    eng.add_trial(_epochs(1, 4, 32, seed=15)[0])
    with pytest.raises(ParameterError):
        eng.finalize(MetricId.XCOR, FrequencyBand(0, 3, 1.0))


def test_reset_clears_trials_sums_and_cache():
    eng = ConnectivityEngine(4, 32, 600.0)
    for e in _epochs(2, 4, 32, seed=16):
        eng.add_trial(e)
    eng.reset()
    assert eng.n_trials == 0
    assert eng.acc.n_trials_accumulated == 0
    assert not eng.cache.spectra and eng.cache.memory_bytes() == 0
    e = _epochs(1, 4, 32, seed=17)[0]
    eng.add_trial(e)
    assert eng.n_trials == 1 and eng.cache.memory_bytes() > 0


def test_band_backfill_needs_no_new_ffts_and_matches_batch():
    eps = _epochs(5, 4, 40, seed=18)
    eng = ConnectivityEngine(4, 48, 600.0, storage_mode=True, accumulate_band=(8, 14))
    for e in eps:
        eng.add_trial(e)
    S.reset_fft_call_count()
    wide = FrequencyBand(0, 24, 12.5)
    got = eng.finalize(MetricId.COH, wide)
    assert S.fft_call_count() == 0
    want, _ = O.compute([e.data for e in eps], 48, 0, 24, ("COH",))
    assert np.abs(got.weights - want["COH"]["band"]).max() <= 1e-4


def test_band_hint_is_ignored_without_storage():
    eps = _epochs(3, 4, 40, seed=19)
    eng = ConnectivityEngine(4, 48, 600.0, storage_mode=False, accumulate_band=(8, 14))
    for e in eps:
        eng.add_trial(e)
    got = eng.finalize(MetricId.COH, FrequencyBand(0, 24, 12.5))
    want = compute_metric(eps, MetricId.COH, 48, FrequencyBand(0, 24, 12.5))
    assert np.abs(got.weights - want.weights).max() <= 1e-6


def test_band_hint_outside_the_spectrum_is_rejected():
    with pytest.raises(ParameterError):
        ConnectivityEngine(4, 48, 600.0, accumulate_band=(20, 25))
    with pytest.raises(ParameterError):
        ConnectivityEngine(4, 48, 600.0, accumulate_band=(-1, 3))


# -- convergence_curve (metrics.py:501-528) -------------------------------------
def test_convergence_curve_counts_and_last_point():
    eps = _epochs(8, 5, 40, seed=20)
    band = FrequencyBand(2, 9, 600.0 / 48)
    counts, curve = M.convergence_curve(eps, MetricId.PLV, 48, band, n_top=4)
    assert counts.tolist() == list(range(1, 9)) and curve.shape == (8,)
    want, _ = O.compute([e.data for e in eps], 48, 2, 9, ("PLV",))
    w = want["PLV"]["band"] / want["PLV"]["band"].max()
    assert curve[-1] == pytest.approx(np.sort(w)[-4:].mean(), abs=1e-5)


@pytest.mark.parametrize("metric", [MetricId.COR, MetricId.XCOR])
def test_convergence_curve_time_domain(metric):
    eps = _epochs(5, 4, 40, seed=21)
    counts, curve = M.convergence_curve(eps, metric, 32, FrequencyBand(0, 3, 1.0), max_lag=7)
    assert len(curve) == 5 and np.all(np.isfinite(curve))


# -- SpectrumSet / fft_real (spectral.py:65-201) --------------------------------
def test_csd_entry_is_hermitian_and_matches_oracle():
    eps = _epochs(4, 6, 45, seed=22)
    acc = S.SpectrumSet(6, 32)
    ref = O.Sums(6, 17)
    for e in eps:
        S.accumulate_epoch(acc, e)
        O.accumulate(ref, O.trial_spectra(e.data, 32))
    pi, pj = O.pair_index(6)
    for i in range(6):
        assert np.abs(acc.csd_entry(i, i).imag).max() == 0.0          # diagonal: the PSD sum
        assert np.abs(acc.csd_entry(i, i).real - ref.psd_sum[i]).max() <= 1e-9
        for j in range(6):
            if i != j:
                assert np.array_equal(acc.csd_entry(i, j), np.conj(acc.csd_entry(j, i)))
    k = 7
    assert np.abs(acc.csd_entry(pi[k], pj[k]) - ref.csd_sum[k]).max() <= 1e-9


def test_merge_of_mismatched_sets_is_rejected():
    with pytest.raises(ParameterError):
        S.SpectrumSet(3, 24).merge(S.SpectrumSet(4, 24))
    with pytest.raises(ParameterError):
        S.SpectrumSet(3, 24).merge(S.SpectrumSet(3, 32))


def test_fft_real_parseval_and_crop_pad():
    rng = np.random.default_rng(23)
    x = rng.standard_normal(64)
    X = S.fft_real(x, 64)
    xd = x - x.mean()
    # one-sided spectrum: interior bins count twice, DC (zero) and Nyquist once
    energy = (np.abs(X[0]) ** 2 + 2 * np.sum(np.abs(X[1:-1]) ** 2) + np.abs(X[-1]) ** 2) / 64
    assert energy == pytest.approx(np.sum(xd ** 2), rel=1e-12)
    y = rng.standard_normal(100)                                    # cropped to nfft
    assert np.abs(S.fft_real(y, 64) - O.trial_spectra(y[None, :64], 64)[0]).max() <= 1e-9
    z = np.array([2.0, -1.0, 0.5, 3.0, -0.25])                      # zero-padded to nfft
    got = S.fft_real(z, 16)
    assert got.shape == (9,) and np.abs(got - O.trial_spectra(z[None], 16)[0]).max() <= 1e-12


@pytest.mark.parametrize("nfft,T", [(63, 50), (63, 80), (9, 9), (255, 300)])
def test_odd_nfft_has_no_nyquist_bin(nfft, T):
    """Odd nfft (np.fft.rfft: nfft // 2 + 1 bins, the last one complex, not a Nyquist bin):
    every spectral metric over all bins against the oracle, including the last bin's
    phase-lag terms."""
    rng = np.random.default_rng(nfft + T)
    data = [rng.standard_normal((7, T)) for _ in range(9)]
    data[0][3] = 0.5 * data[0][2]
    hi = nfft // 2
    want, _ = O.compute(data, nfft, 0, hi, ("COH", "IMAGCOHY", "PLV", "PLI", "WPLI", "DSWPLI", "USPLI"))
    assert np.abs(want["PLI"]["bins"][:, -1]).max() > 0          # the last bin carries phase
    band = FrequencyBand(0, hi, 500.0 / nfft)
    for m, tol in (("COH", 1e-4), ("IMAGCOHY", 1e-4), ("PLV", 1e-4), ("PLI", 1e-3), ("WPLI", 1e-3),
                   ("DSWPLI", 1e-3), ("USPLI", 1e-3)):
        net = compute_metric([EpochMatrix(d, 500.0) for d in data], MetricId.parse(m), nfft, band)
        assert np.abs(net.weights - want[m]["band"]).max() <= tol, m
    acc = S.SpectrumSet(7, nfft)
    for d in data:
        S.accumulate_epoch(acc, EpochMatrix(d, 500.0))
    assert acc.n_bins == hi + 1
    assert np.abs(M.pli_bins(acc) - want["PLI"]["bins"]).max() <= 1e-3
    assert np.abs(M.imagcohy_bins(acc) - want["IMAGCOHY"]["bins"]).max() <= 1e-4


@pytest.mark.parametrize("n_last,kept", [(2, [3, 4]), (0, [0, 1, 2, 3, 4]), (-2, [2, 3, 4]), (9, [0, 1, 2, 3, 4])])
def test_rebuild_last_slices_like_the_reference(n_last, kept):
    """rebuild_last keeps sorted(cache)[-n_last:] (metrics.py:450-460): n_last = 0 keeps
    every cached trial, a negative count drops the oldest |n_last|."""
    eps = _epochs(5, 5, 48, seed=30)
    eng = ConnectivityEngine(5, 48, 600.0, storage_mode=True)
    for e in reversed(eps):                       # cache order is by trial index, not arrival
        eng.add_trial(e)
    eng.rebuild_last(n_last)
    assert eng.n_trials == len(kept) and eng.acc.n_trials_accumulated == len(kept)
    band = FrequencyBand(2, 10, 12.5)
    want, _ = O.compute([eps[k].data for k in kept], 48, 2, 10, ("PLV", "WPLI"))
    for m in ("PLV", "WPLI"):
        assert np.abs(eng.finalize(MetricId.parse(m), band).weights - want[m]["band"]).max() <= 1e-3, m
    w, _ = O.cor([eps[k].data for k in kept])
    assert np.abs(eng.finalize(MetricId.COR, band).weights - w).max() <= 1e-12


def test_convergence_curve_xcor_uses_each_trial_even_with_repeated_indices():
    """convergence_curve folds XCOR peaks from every epoch it is given (metrics.py:517-518),
    so epochs that share the default trial_index still count one by one."""
    rng = np.random.default_rng(31)
    data = [rng.standard_normal((4, 40)) for _ in range(5)]
    eps = [EpochMatrix(d, 600.0) for d in data]            # all trial_index 0
    counts, curve = M.convergence_curve(eps, MetricId.XCOR, 32, FrequencyBand(0, 3, 1.0), n_top=3, max_lag=6)
    assert counts.tolist() == [1, 2, 3, 4, 5]
    snaps = []
    for k in range(1, 6):
        w, _ = O.xcor(data[:k], max_lag=6)
        snaps.append(w / w.max())
    top = np.argsort(-snaps[-1])[:3]
    assert np.abs(curve - np.array([s[top].mean() for s in snaps])).max() <= 1e-9


def test_repeated_trial_index_folds_cached_spectra_but_cor_sees_each_epoch():
    """With storage on, an epoch whose trial_index is already cached re-folds the cached
    spectra (metrics.py:341-343) -- here every epoch has the default index 0, so the
    spectral sums hold K copies of the first epoch (PLV = 1) -- while COR sums each given
    epoch's own correlation (metrics.py:355-357)."""
    rng = np.random.default_rng(32)
    data = [rng.standard_normal((5, 48)) for _ in range(4)]
    eng = ConnectivityEngine(5, 48, 600.0, storage_mode=True)
    for d in data:
        eng.add_trial(EpochMatrix(d, 600.0))
    band = FrequencyBand(2, 10, 12.5)
    assert eng.n_trials == 4
    assert np.abs(eng.finalize(MetricId.PLV, band).weights - 1.0).max() <= 1e-5
    want, _ = O.compute([data[0]] * 4, 48, 2, 10, ("COH",))
    assert np.abs(eng.finalize(MetricId.COH, band).weights - want["COH"]["band"]).max() <= 1e-4
    w, _ = O.cor(data)
    assert np.abs(eng.finalize(MetricId.COR, band).weights - w).max() <= 1e-12


def test_band_past_the_last_bin_like_the_reference():
    """The reference slices per-bin arrays with the band (metrics.py:121-127): COHY's
    complex mean then runs over the bins that exist, every other metric hits band_average's
    range check (core.py:208-215).  Same through SpectrumSet and the engine."""
    eps = _epochs(4, 5, 48, seed=33)
    nb = 25
    over = FrequencyBand(18, nb + 6, 12.5)
    inside = FrequencyBand(18, nb - 1, 12.5)
    acc = S.SpectrumSet(5, 48)
    eng = ConnectivityEngine(5, 48, 600.0, storage_mode=True)
    for e in eps:
        S.accumulate_epoch(acc, e)
        eng.add_trial(e)
    want, _ = O.compute([e.data for e in eps], 48, 18, nb - 1, ("COHY",))
    for got in (M.finalize_spectral(acc, MetricId.COHY, over), eng.finalize(MetricId.COHY, over)):
        assert got.band == over
        assert np.abs(got.weights - np.abs(want["COHY"]["cband"])).max() <= 1e-4
        ref = M.finalize_spectral(acc, MetricId.COHY, inside)
        assert np.abs(got.complex_weights - ref.complex_weights).max() <= 1e-6
    for fn in (lambda: M.finalize_spectral(acc, MetricId.COH, over), lambda: eng.finalize(MetricId.WPLI, over),
               lambda: eng.finalize(MetricId.COHY, FrequencyBand(nb, nb + 2, 12.5))):
        with pytest.raises(ParameterError):
            fn()


def test_engine_cache_holds_the_reference_cached_spectra():
    """engine.cache.spectra[idx] is what the reference caches (metrics.py:341-347): the
    trial's spectra, or a welch trial's first segment; read from the HBM ring on access."""
    rng = np.random.default_rng(34)
    fixed = ConnectivityEngine(4, 32, 250.0, storage_mode=True)
    welch = ConnectivityEngine(4, 32, 250.0, storage_mode=True, spectral_mode="welch")
    data = [rng.standard_normal((4, T)) for T in (40, 100, 20)]
    for k, d in enumerate(data):
        fixed.add_trial(EpochMatrix(d, 250.0, trial_index=k))
        welch.add_trial(EpochMatrix(d, 250.0, trial_index=k))
    assert sorted(fixed.cache.spectra) == [0, 1, 2] and len(welch.cache.spectra) == 3
    for k, d in enumerate(data):
        assert np.abs(fixed.cache.spectra[k] - O.trial_spectra(d, 32)).max() <= 1e-9
        first = O.segments(d, 32)[0] if d.shape[1] >= 64 else d
        assert np.abs(welch.cache.spectra[k] - O.trial_spectra(first, 32)).max() <= 1e-9


def test_incremental_equals_batch_over_trial_orderings():
    """Acceptance criterion 2 of the reference (test_acceptance.py:99-124): trial-by-trial
    updates without storage, in random trial orders, equal the batch result for all ten
    metrics.  COR / XCOR run in fp64 and meet the reference's 1e-10 relative; the spectral
    metrics' fp32 sums depend on the trial order in their last bits, so they are held to
    2e-6 absolute (far inside the north-star 1e-4 / 1e-3), and K PLI stays an exact integer."""
    eps = _epochs(6, 4, 40, seed=202)
    band = FrequencyBand(2, 8, 600.0 / 48)
    batch = {m: compute_metric(eps, m, 48, band, max_lag=12) for m in MetricId}
    rng = np.random.default_rng(0)
    for _ in range(6):
        perm = rng.permutation(len(eps))
        for m in MetricId:
            eng = ConnectivityEngine(4, 48, 600.0, storage_mode=False, max_lag=12)
            net = None
            for k in perm:
                try:
                    net = eng.update_and_finalize(eps[k], m, band)
                except M.DegenerateTrialCountError:
                    assert m is MetricId.USPLI
            ref = batch[m].weights
            if m in (MetricId.COR, MetricId.XCOR):
                rel = np.max(np.abs(net.weights - ref) / np.maximum(np.abs(ref), 1e-12))
                assert rel <= 1e-10, (m, rel)
                if m is MetricId.XCOR:
                    assert np.array_equal(np.asarray(net.lags), np.asarray(batch[m].lags))
            else:
                assert np.abs(net.weights - ref).max() <= 2e-6, m
            if m is MetricId.PLI:
                assert np.array_equal(np.rint(net.weights * 7 * 6), np.rint(ref * 7 * 6))
