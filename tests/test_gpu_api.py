"""The reference's own test strategy (pkg/tests/test_spectral.py, test_metrics.py,
test_acceptance.py) replayed against the drop-in package on the GPU, with the
pinned oracle as the checker.  Tolerances: north_star (1e-4 coherency family,
1e-3 phase-lag family; fp32 outputs vs fp64)."""
import numpy as np
import pytest
import torch

import oracle as O
from paper_2303_03279_b200 import core
from paper_2303_03279_b200.core import (DegenerateTrialCountError, EpochMatrix, FrequencyBand, MetricId,
                                        ParameterError)
from paper_2303_03279_b200 import metrics as M
from paper_2303_03279_b200 import spectral as S

pytestmark = pytest.mark.gpu
TOL = {"COHY": 1e-4, "COH": 1e-4, "IMAGCOHY": 1e-4, "PLV": 1e-4, "PLI": 1e-3, "USPLI": 1e-3, "WPLI": 1e-3,
       "DSWPLI": 1e-3}


def make_epochs(n_trials, n_channels, n_samples, seed=0, sfreq=600.0):
    rng = np.random.default_rng(seed)
    return [EpochMatrix(data=rng.standard_normal((n_channels, n_samples)), sfreq=sfreq, trial_index=k)
            for k in range(n_trials)]


def accumulated(epochs, nfft):
    acc = S.SpectrumSet(epochs[0].n_channels, nfft)
    for ep in epochs:
        S.accumulate_epoch(acc, ep)
    return acc


# ---------------------------------------------------------------- spectral (test_spectral.py)
class TestFftReal:
    def test_matches_naive_dft(self):
        rng = np.random.default_rng(0)
        for n, nfft in [(64, 64), (100, 64), (40, 64)]:
            x = rng.standard_normal(n)
            got = S.fft_real(x, nfft)
            want = O.trial_spectra(x[None], nfft, method="dft")[0]
            np.testing.assert_allclose(got, want, atol=1e-9)

    def test_mean_removed(self):
        assert abs(S.fft_real(np.full(32, 3.7), 32)[0]) < 1e-12

    def test_invalid(self):
        with pytest.raises(ParameterError):
            S.fft_real(np.ones(8), 1)
        with pytest.raises(ParameterError):
            S.fft_real(np.array([]), 8)

    def test_trial_spectra_matches_numpy_rfft(self):
        ep = make_epochs(1, 6, 300, seed=4)[0]
        got = S.trial_spectra(ep, 256)
        want = O.trial_spectra(ep.data, 256)
        assert got.shape == (6, 129)
        np.testing.assert_allclose(got, want, atol=1e-9)
        assert np.all(got[:, 0] == 0)
        assert np.all(got[:, -1].imag == 0)


class TestSpectrumSet:
    def test_shapes(self):
        acc = S.SpectrumSet(4, 64)
        assert acc.n_bins == 33 and acc.n_pairs == 6

    def test_sums_match_direct_accumulation(self):
        eps = make_epochs(4, 3, 24, seed=5)
        acc = S.SpectrumSet(3, 24)
        specs = [S.trial_spectra(ep, 24) for ep in eps]
        for s in specs:
            S.accumulate_spectra(acc, s)
        pi, pj = S.pair_index(3)
        np.testing.assert_allclose(acc.csd_sum, sum(s[pi] * np.conj(s[pj]) for s in specs), atol=1e-10)
        np.testing.assert_allclose(acc.psd_sum, sum(np.abs(s) ** 2 for s in specs), atol=1e-10)
        np.testing.assert_array_equal(acc.im_sum, acc.csd_sum.imag)
        assert acc.n_trials_accumulated == 4

    def test_merge_associative(self):
        eps = make_epochs(6, 3, 24, seed=9)
        whole = accumulated(eps, 24)
        a, b = accumulated(eps[:2], 24), accumulated(eps[2:], 24)
        a.merge(b)
        np.testing.assert_allclose(a.csd_sum, whole.csd_sum, atol=1e-10)
        np.testing.assert_allclose(M.wpli_bins(a), M.wpli_bins(whole), atol=1e-6)
        assert a.n_trials_accumulated == 6
        with pytest.raises(ParameterError):
            S.SpectrumSet(3, 24).merge(S.SpectrumSet(4, 24))

    def test_copy_independent(self):
        acc = S.SpectrumSet(3, 16)
        cp = acc.copy()
        S.accumulate_epoch(acc, make_epochs(1, 3, 16)[0])
        assert cp.n_trials_accumulated == 0

    def test_fft_counter_counts_per_channel(self):
        S.reset_fft_call_count()
        S.accumulate_epoch(S.SpectrumSet(7, 32), make_epochs(1, 7, 32)[0])
        assert S.fft_call_count() == 7

    def test_pair_row_slices_tile_pair_axis(self):
        for C in range(2, 31):
            pi, pj = S.pair_index(C)
            for i in range(C - 1):
                sl = S.pair_row_slice(C, i)
                assert pi[sl].tolist() == [i] * (C - 1 - i)


# ---------------------------------------------------------------- metrics (test_metrics.py)
class TestSpectralAgainstOracle:
    @pytest.mark.parametrize("name", list(TOL))
    def test_matches_reference_restatement(self, name):
        epochs = make_epochs(6, 4, 32, seed=11)
        acc = accumulated(epochs, 32)
        got = M._SPECTRAL_BINS[MetricId[name]](acc)
        want = O.compute([e.data for e in epochs], 32, 0, 16, metrics=(name,))[0][name]["bins"]
        assert np.abs(got - want).max() <= TOL[name]


class TestMetricBounds:
    @pytest.mark.parametrize("seed", range(8))
    def test_ranges(self, seed):
        acc = accumulated(make_epochs(4, 3, 24, seed=seed), 24)
        eps = 1e-6
        assert np.all(M.coh_bins(acc) <= 1 + eps) and np.all(M.coh_bins(acc) >= 0)
        assert np.all(np.abs(M.imagcohy_bins(acc)) <= 1 + eps)
        assert np.all((M.plv_bins(acc) >= 0) & (M.plv_bins(acc) <= 1 + eps))
        assert np.all((M.pli_bins(acc) >= 0) & (M.pli_bins(acc) <= 1 + eps))
        assert np.all((M.wpli_bins(acc) >= 0) & (M.wpli_bins(acc) <= 1 + eps))
        assert np.all(M.dswpli_bins(acc) <= M.wpli_bins(acc) + eps)
        assert np.all(M.uspli_bins(acc) >= -1.0 / (acc.n_trials_accumulated - 1) - eps)

    def test_uspli_needs_two_trials(self):
        with pytest.raises(DegenerateTrialCountError):
            M.uspli_bins(accumulated(make_epochs(1, 3, 24), 24))

    def test_no_trials_degenerate(self):
        acc = S.SpectrumSet(3, 24)
        for fn in M._SPECTRAL_BINS.values():
            with pytest.raises(DegenerateTrialCountError):
                fn(acc)

    def test_wpli_zero_over_zero_is_zero(self):
        data = np.tile(np.sin(np.arange(32) * 0.3), (2, 1))
        acc = accumulated([EpochMatrix(data=data, sfreq=100.0)] * 3, 32)
        assert np.all(M.wpli_bins(acc) == 0.0)
        assert np.all(M.pli_bins(acc) == 0.0)


class TestFinalizeSpectral:
    def test_band_average(self):
        acc = accumulated(make_epochs(4, 3, 32, seed=51), 32)
        band = FrequencyBand(3, 7, 600.0 / 32)
        net = M.finalize_spectral(acc, MetricId.COH, band)
        np.testing.assert_allclose(net.weights, M.coh_bins(acc)[:, 3:8].mean(axis=1), atol=1e-6)
        assert net.n_trials == 4

    def test_cohy_weight_is_magnitude_of_mean(self):
        acc = accumulated(make_epochs(4, 3, 32, seed=52), 32)
        band = FrequencyBand(2, 6, 600.0 / 32)
        net = M.finalize_spectral(acc, MetricId.COHY, band)
        cmean = M.cohy_bins(acc)[:, 2:7].mean(axis=1)
        np.testing.assert_allclose(net.complex_weights, cmean, atol=1e-6)
        np.testing.assert_allclose(net.weights, np.abs(cmean), atol=1e-6)

    def test_band_limited_equals_full_then_crop(self):
        acc = accumulated(make_epochs(4, 3, 32, seed=53), 32)
        np.testing.assert_allclose(M.wpli_bins(acc, FrequencyBand(4, 9, 1.0)), M.wpli_bins(acc)[:, 4:10], atol=1e-6)

    def test_non_spectral_rejected(self):
        acc = accumulated(make_epochs(2, 3, 32), 32)
        with pytest.raises(ParameterError):
            M.finalize_spectral(acc, MetricId.COR, FrequencyBand(0, 3, 1.0))


class TestEngine:
    SPECTRAL = [m for m in MetricId if m.is_spectral]

    def test_incremental_equals_batch_all_metrics(self):
        epochs = make_epochs(8, 4, 40, seed=61)
        band = FrequencyBand(2, 8, 600.0 / 48)
        for metric in self.SPECTRAL:
            engine = M.ConnectivityEngine(4, 48, 600.0, storage_mode=False)
            net = None
            for ep in epochs:
                try:
                    net = engine.update_and_finalize(ep, metric, band)
                except DegenerateTrialCountError:
                    assert metric is MetricId.USPLI and engine.n_trials == 1
            batch = M.compute_metric(epochs, metric, 48, band)
            np.testing.assert_allclose(net.weights, batch.weights, atol=1e-6, err_msg=metric.value)

    def test_metric_switch_zero_new_ffts(self):
        epochs = make_epochs(6, 4, 40, seed=62)
        engine = M.ConnectivityEngine(4, 48, 600.0, storage_mode=True)
        band = FrequencyBand(2, 8, 600.0 / 48)
        for ep in epochs:
            engine.add_trial(ep)
        S.reset_fft_call_count()
        for metric in (MetricId.COH, MetricId.WPLI, MetricId.PLV, MetricId.PLI, MetricId.DSWPLI):
            engine.finalize(metric, band)
        assert S.fft_call_count() == 0

    def test_rebuild_last_window(self):
        epochs = make_epochs(6, 3, 32, seed=64)
        band = FrequencyBand(1, 6, 1.0)
        engine = M.ConnectivityEngine(3, 32, 600.0, storage_mode=True)
        for ep in epochs:
            engine.add_trial(ep)
        S.reset_fft_call_count()
        engine.rebuild_last(3)
        net = engine.finalize(MetricId.COH, band)
        assert S.fft_call_count() == 0
        batch = M.compute_metric(epochs[-3:], MetricId.COH, 32, band)
        np.testing.assert_allclose(net.weights, batch.weights, atol=1e-6)
        assert net.n_trials == 3

    def test_rebuild_requires_storage(self):
        with pytest.raises(ParameterError):
            M.ConnectivityEngine(3, 32, 600.0, storage_mode=False).rebuild_last(2)

    def test_reset_and_channel_mismatch(self):
        engine = M.ConnectivityEngine(3, 32, 600.0)
        engine.add_trial(make_epochs(1, 3, 32)[0])
        engine.reset()
        assert engine.n_trials == 0 and not engine.cache.spectra
        with pytest.raises(ParameterError):
            engine.add_trial(make_epochs(1, 4, 32)[0])

    def test_band_limited_accumulation_matches_full(self):
        epochs = make_epochs(6, 4, 40, seed=65)
        limited = M.ConnectivityEngine(4, 48, 600.0, storage_mode=True, accumulate_band=(10, 15))
        for ep in epochs:
            limited.add_trial(ep)
        S.reset_fft_call_count()
        for band in (FrequencyBand(10, 15, 12.5), FrequencyBand(0, 24, 12.5)):
            for metric in (MetricId.COH, MetricId.WPLI, MetricId.PLV):
                got = limited.finalize(metric, band)
                want = M.compute_metric(epochs, metric, 48, band)
                np.testing.assert_allclose(got.weights, want.weights, atol=1e-6)
        with pytest.raises(ParameterError):
            M.ConnectivityEngine(4, 48, 600.0, accumulate_band=(10, 99))

    def test_cache_memory_accounting(self):
        engine = M.ConnectivityEngine(3, 32, 600.0, storage_mode=True)
        assert engine.cache.memory_bytes() == 0
        engine.add_trial(make_epochs(1, 3, 32)[0])
        assert engine.cache.memory_bytes() > 0

    def test_convergence_curve_final_value(self):
        epochs = make_epochs(10, 4, 40, seed=71)
        band = FrequencyBand(2, 8, 600.0 / 48)
        counts, curve = M.convergence_curve(epochs, MetricId.COH, 48, band, n_top=3)
        assert counts.tolist() == list(range(1, 11))
        net = M.compute_metric(epochs, MetricId.COH, 48, band)
        w = net.weights / net.weights.max()
        assert np.isclose(curve[-1], np.sort(w)[-3:].mean(), atol=1e-6)


# ---------------------------------------------------------------- acceptance (test_acceptance.py)
@pytest.mark.parametrize("C", [1, 2, 3])
def test_smallest_node_counts(C):
    """One channel -> an empty network (no pairs), as the reference returns; two and
    three channels (a single partial tile) match the oracle for every metric."""
    eps = make_epochs(3, C, 64, seed=20 + C, sfreq=100.0)
    band = FrequencyBand(2, 5, 100.0 / 32)
    for m in ("COHY", "COH", "IMAGCOHY", "PLV", "PLI", "USPLI", "WPLI", "DSWPLI", "COR", "XCOR"):
        net = M.compute_metric(eps, MetricId[m], 32, band=None if m in ("COR", "XCOR") else band)
        w = np.asarray(net.weights)
        assert w.shape == (C * (C - 1) // 2,), m
        if C == 1 or m in ("COR", "XCOR"):
            continue
        want, _ = O.compute([e.data for e in eps], 32, 2, 5, (m,))
        np.testing.assert_allclose(w, want[m]["band"], rtol=0, atol=TOL[m], err_msg=m)
        if m == "COHY":  # weight = |mean coherency| (metrics.py:126-130)
            np.testing.assert_allclose(np.abs(np.asarray(net.complex_weights)), w, rtol=1e-6, atol=1e-7)


def test_criterion_1_oracle_equivalence():
    epochs = make_epochs(20, 8, 64, seed=101)
    acc = accumulated(epochs, 64)
    want, _ = O.compute([e.data for e in epochs], 64, 0, 32)
    for metric, fn in M._SPECTRAL_BINS.items():
        assert np.abs(fn(acc) - want[metric.value]["bins"]).max() <= TOL[metric.value], metric.value


def test_criterion_3_zero_lag_copies():
    rng = np.random.default_rng(7)
    t = np.arange(96) / 600.0
    eps = []
    for k in range(60):
        s = np.sin(2 * np.pi * 18.0 * t + rng.uniform(0, 2 * np.pi))
        eps.append(EpochMatrix(data=np.vstack([s, 0.7 * s, 0.4 * s]), sfreq=600.0, trial_index=k))
    band = FrequencyBand(15, 21, 1.0)
    for metric in (MetricId.IMAGCOHY, MetricId.PLI, MetricId.WPLI):
        net = M.compute_metric(eps, metric, 600, band)
        assert np.all(np.abs(net.weights) <= 1e-9), (metric, net.weights)
    for metric in (MetricId.COH, MetricId.PLV):
        assert np.all(M.compute_metric(eps, metric, 600, band).weights >= 0.99)


@pytest.mark.parametrize("metric", ["COH", "IMAGCOHY"])
def test_reference_threshold_fixture(metric):
    """The reference's golden network (export_threshold_fixtures.py) through compute_metric."""
    from conftest import GOLDEN
    g = np.load(GOLDEN / "sim2024_thresh.npz")
    eps = [EpochMatrix(data=e, sfreq=600.0, trial_index=k) for k, e in enumerate(g["epochs"])]
    net = M.compute_metric(eps, MetricId[metric], 600, FrequencyBand(15, 21, 1.0))
    want = g["band_" + metric]
    assert np.abs(net.weights - want).max() <= 1e-4
    assert np.abs(net.weights / np.abs(net.weights).max() - want / np.abs(want).max()).max() <= 1e-4


@pytest.mark.parametrize("nfft,T,lo,hi,taper", [(64, 64, 0, 32, None), (128, 100, 3, 60, "hann"),
                                                (512, 500, 0, 256, "hann"), (1024, 1000, 8, 13, "hann"),
                                                (256, 300, 5, 20, ("dpss", 2.0, 3))])
def test_fft_and_dft_spectra_agree(monkeypatch, nfft, T, lo, hi, taper):
    """Both K1 variants (direct DFT and real FFT) against the oracle's rfft spectra."""
    from paper_2303_03279_b200.plan import DevicePlan, make_taper
    rng = np.random.default_rng(nfft + T)
    x = rng.standard_normal((3, 5, T)) + 7.0
    tap = make_taper(taper, min(T, nfft))
    want = np.stack([np.stack([O.trial_spectra(e, nfft, None if tap is None else tp)[:, lo:hi + 1]
                               for tp in ([None] if tap is None else tap)]) for e in x])  # [K, L, C, nb]
    for mode in ("fft", "dft"):
        monkeypatch.setenv("CSCONN_SPECTRA", mode)
        plan = DevicePlan(5, T, nfft, lo, hi, taper=taper, slot_capacity=3, device="cuda")
        plan.spectra(torch.tensor(x, device="cuda"), 0)
        got = plan.ring()[0].cpu().numpy()                 # [S, L, nb, N]
        got = np.transpose(got, (0, 1, 3, 2))               # [K, L, C, nb]
        np.testing.assert_allclose(got, want, atol=1e-9 * np.abs(want).max(), err_msg=mode)


def test_host_pipeline_matches_device_path():
    """HostPipeline (chunked uploads, row-chunked kernels + downloads, back-to-back
    submits) returns the band means of the one-shot device path."""
    from paper_2303_03279_b200.plan import DevicePlan, HostPipeline, SEVEN, pow2_scale
    rng = np.random.default_rng(11)
    K, N, T, nfft, lo, hi = 9, 300, 200, 256, 4, 20
    x = torch.tensor(rng.standard_normal((K, N, T)), dtype=torch.float32)
    scale = pow2_scale(float(x.abs().max()), min(T, nfft))
    ref = DevicePlan(N, T, nfft, lo, hi, taper="hann", slot_capacity=K, device="cuda", scale=scale)
    ref.spectra(x.cuda(), 0)
    want = ref.pair_metrics(torch.arange(K, dtype=torch.int32, device="cuda"), SEVEN + ("COHY",), 0, ref.n_bins,
                            per_bin=False, band=True)
    hp = HostPipeline(N, T, nfft, lo, hi, K, metrics=SEVEN + ("COHY",), taper="hann", scale=scale, device="cuda",
                      in_chunks=4, row_chunks=5)
    xh = x.pin_memory()
    outs = [hp.alloc_host() for _ in range(3)]
    for o in outs:                       # three calls in flight
        ev = hp.submit(xh, o)
    ev.synchronize()
    for o in outs:
        for m in SEVEN + ("COHY",):
            # same kernels; only the band-mean summation order may differ (bins split over CTAs)
            np.testing.assert_allclose(o[m].numpy(), want[m]["band"].cpu().numpy(), rtol=0, atol=2e-6, err_msg=m)


def test_window_graph_matches_eager_windows():
    """WindowGraph (CUDA-graph replays, one graph per ring phase, the ring = the
    window) returns, update after update, the metrics of a fresh eager plan over
    the same window of trials -- including after the phases wrap around."""
    from paper_2303_03279_b200.plan import DevicePlan, WindowGraph, pow2_scale
    rng = np.random.default_rng(12)
    win, new, N, T, nfft, lo, hi = 10, 4, 150, 128, 128, 3, 20
    n_up = 9                                          # 5 phases (10 / gcd(10, 4)), wrapped once
    x = torch.tensor(rng.standard_normal((win + new * n_up, N, T)), dtype=torch.float32, device="cuda")
    scale = pow2_scale(float(x.abs().max()), min(T, nfft))
    metrics = ("COH", "IMAGCOHY", "PLV", "PLI", "USPLI", "WPLI", "DSWPLI")
    plan = DevicePlan(N, T, nfft, lo, hi, taper="hann", slot_capacity=win, device="cuda", scale=scale)
    wg = WindowGraph(plan, new, metrics)
    assert wg.n_phases == 5
    wg.prime(x[:win])
    for u in range(1, n_up + 1):
        got = wg.update(x[win + new * (u - 1): win + new * u])
        if u in (1, 4, 5, 6, 9):
            ref = DevicePlan(N, T, nfft, lo, hi, taper="hann", slot_capacity=win, device="cuda", scale=scale)
            ref.spectra(x[new * u: new * u + win], 0)
            want = ref.pair_metrics(torch.arange(win, dtype=torch.int32, device="cuda"), metrics)
            for m in metrics:
                for part in ("bins", "band"):
                    # same kernels, the trials in ring (not stream) order: fp32 summation order only
                    np.testing.assert_allclose(got[m][part].cpu().numpy(), want[m][part].cpu().numpy(),
                                               rtol=0, atol=2e-5, err_msg=f"{m} {part} update {u}")
    assert len(wg._graphs) == 9 and wg.graph_kernels() > 0  # (phase, buffer) keys: lcm(5, 2) = 10 > 9 updates
    with pytest.raises(ParameterError):
        wg.update(x[:new + 1])


def test_window_graph_submit_pipelined_host_io():
    """WindowGraph.submit from pinned host samples into pinned host band buffers,
    many updates in flight (no host sync in between): every window's downloaded
    band results equal a fresh eager plan's over the same trials."""
    from paper_2303_03279_b200.plan import DevicePlan, WindowGraph, pow2_scale
    rng = np.random.default_rng(13)
    win, new, N, T, nfft, lo, hi = 12, 3, 140, 100, 128, 2, 30
    n_up = 10
    xh = torch.tensor(rng.standard_normal((win + new * n_up, N, T)), dtype=torch.float32).pin_memory()
    scale = pow2_scale(float(xh.abs().max()), min(T, nfft))
    metrics = ("COH", "PLV", "WPLI")
    plan = DevicePlan(N, T, nfft, lo, hi, taper="hann", slot_capacity=win, device="cuda", scale=scale)
    wg = WindowGraph(plan, new, metrics)
    wg.prime(xh[:win])
    P = N * (N - 1) // 2
    outs = [{m: torch.empty(P, dtype=torch.float32).pin_memory() for m in metrics} for _ in range(n_up)]
    evs = [wg.submit(xh[win + new * (u - 1): win + new * u], outs[u - 1]) for u in range(1, n_up + 1)]
    for ev in evs:
        ev.synchronize()
    for u in (1, 2, 7, n_up):
        ref = DevicePlan(N, T, nfft, lo, hi, taper="hann", slot_capacity=win, device="cuda", scale=scale)
        ref.spectra(xh[new * u: new * u + win].cuda(), 0)
        want = ref.pair_metrics(torch.arange(win, dtype=torch.int32, device="cuda"), metrics)
        for m in metrics:
            np.testing.assert_allclose(outs[u - 1][m].numpy(), want[m]["band"].cpu().numpy(), rtol=0, atol=2e-5,
                                       err_msg=f"{m} update {u}")


# ---------------------------------------------------------------- welch mode (test_spectral.py:138-160)
class TestWelchMode:
    def test_welch_averages_segments(self):
        ep = make_epochs(1, 2, 64, seed=4)[0]
        acc = S.SpectrumSet(2, 16)
        S.accumulate_epoch(acc, ep, mode="welch")
        pi, pj = S.pair_index(2)
        csd = np.zeros((1, 9), np.complex128)
        psd = np.zeros((2, 9))
        for k in range(4):
            s = S.trial_spectra(EpochMatrix(data=ep.data[:, k * 16:(k + 1) * 16], sfreq=ep.sfreq), 16)
            csd += s[pi] * np.conj(s[pj])
            psd += np.abs(s) ** 2
        np.testing.assert_allclose(acc.csd_sum, csd / 4, atol=1e-10)
        np.testing.assert_allclose(acc.psd_sum, psd / 4, atol=1e-10)

    def test_welch_falls_back_for_short_trials(self):
        ep = make_epochs(1, 2, 20, seed=4)[0]
        a, b = S.SpectrumSet(2, 16), S.SpectrumSet(2, 16)
        S.accumulate_epoch(a, ep, mode="welch")
        S.accumulate_epoch(b, ep, mode="fixed")
        np.testing.assert_allclose(a.csd_sum, b.csd_sum)

    def test_segment_spectra_and_fft_counter(self):
        ep = make_epochs(1, 3, 70, seed=5)[0]
        S.reset_fft_call_count()
        segs = S.segment_spectra(ep, 16)
        assert len(segs) == 4 and S.fft_call_count() == 4 * 3
        want = [O.trial_spectra(ep.data[:, k * 16:(k + 1) * 16], 16) for k in range(4)]
        for g, w in zip(segs, want):
            np.testing.assert_allclose(g, w, atol=1e-9 * np.abs(w).max())

    def test_mixed_welch_and_fixed_trials(self):
        """A welch trial folds its segment-mean CSD, a fixed one its own CSD
        (weights of spectral.py:272-283), in one accumulator."""
        eps = make_epochs(4, 5, 96, seed=9)
        acc = S.SpectrumSet(5, 32)
        ref = O.Sums(5, 17)
        for k, ep in enumerate(eps):
            mode = "welch" if k % 2 == 0 else "fixed"
            S.accumulate_epoch(acc, ep, mode=mode)
            if mode == "welch":
                O.accumulate_multitaper(ref, np.stack([O.trial_spectra(sg, 32) for sg in O.segments(ep.data, 32)]))
            else:
                O.accumulate(ref, O.trial_spectra(ep.data, 32))
        band = FrequencyBand(0, 16, 1.0)
        for metric, fn in M._SPECTRAL_BINS.items():
            want = O.BINS[metric.value](ref)
            assert np.abs(fn(acc, band) - want).max() <= TOL[metric.value], metric.value

    def test_engine_welch_then_rebuild_uses_cached_first_segments(self):
        """ConnectivityEngine(spectral_mode="welch"): first folds are segment means;
        rebuild_last re-folds the cached first-segment spectra in fixed mode
        (metrics.py:337-341, 450-460), exactly as the reference does."""
        eps = make_epochs(6, 6, 128, seed=13)
        band = FrequencyBand(2, 12, 1.0)
        eng = M.ConnectivityEngine(6, 32, 600.0, storage_mode=True, spectral_mode="welch")
        for ep in eps:
            eng.add_trial(ep)
        for metric in ("COH", "PLV", "WPLI", "IMAGCOHY"):
            got = eng.finalize(MetricId[metric], band).weights
            want, _ = O.compute([e.data for e in eps], 32, 2, 12, metrics=(metric,), mode="welch")
            assert np.abs(got - want[metric]["band"]).max() <= TOL[metric], metric
        eng.rebuild_last(4)
        for metric in ("COH", "PLI", "WPLI"):
            got = eng.finalize(MetricId[metric], band).weights
            want, _ = O.compute([e.data[:, :32] for e in eps[-4:]], 32, 2, 12, metrics=(metric,))
            assert np.abs(got - want[metric]["band"]).max() <= TOL[metric], metric


@pytest.mark.parametrize("case", ["rect_crop_oddk", "rect_accept", "welch3", "zerolag_dead"])
def test_running_sums_match_reference(case):
    """SpectrumSet attributes (cs_pair_sums over the fp64 ring) against the
    reference-pinned oracle's sums (spectral.py:136-141, 216-241)."""
    from conftest import GOLDEN
    g = np.load(GOLDEN / f"{case}.npz")
    mode = str(g["mode"]) if "mode" in g.files else "fixed"
    nfft = int(g["nfft"])
    eps = [EpochMatrix(data=e, sfreq=1000.0, trial_index=k) for k, e in enumerate(g["epochs"])]
    acc = S.SpectrumSet(eps[0].n_channels, nfft)
    for ep in eps:
        S.accumulate_epoch(acc, ep, mode=mode)
    _, ref = O.compute([e.data for e in eps], nfft, 0, nfft // 2, mode=mode)
    scale = np.abs(ref.csd_sum).max()
    np.testing.assert_allclose(acc.csd_sum, ref.csd_sum, atol=1e-9 * scale)
    np.testing.assert_allclose(acc.psd_sum, ref.psd_sum, atol=1e-9 * np.abs(ref.psd_sum).max())
    np.testing.assert_allclose(acc.abs_im_sum, ref.abs_im_sum, atol=1e-9 * scale)
    np.testing.assert_allclose(acc.plv_sum, ref.plv_sum, atol=1e-9)
    # sign sums are integers: exact wherever the entry is not decided by the 1e-13 flush
    sens = O.flush_sensitive([e.data for e in eps], nfft, 0, nfft // 2, mode=mode)
    assert np.array_equal(acc.pli_sum[~sens], ref.pli_sum[~sens])
    assert acc.n_trials_accumulated == len(eps)


# ---------------------------------------------------------------- device network post-processing
@pytest.mark.parametrize("P,ties", [(6, False), (5000, True), (3_000_000, True), (1_000_001, False)])
def test_device_threshold_matches_host_semantics(P, ties):
    """cs_net_threshold (radix select + ordered compaction) = the reference's
    lexsort selection (core.py:184-205) on the same fp32 weights."""
    from paper_2303_03279_b200.core import ConnectivityNetwork, pair_to_ij, threshold_network, normalize_network
    rng = np.random.default_rng(P)
    w = rng.standard_normal(P).astype(np.float32)
    if ties:
        w = np.round(w, 1).astype(np.float32)                 # many exact ties
    n = int((1 + np.sqrt(1 + 8 * P)) / 2) + 1
    while n * (n - 1) // 2 < P:
        n += 1
    wd = torch.tensor(w, device="cuda")
    net = ConnectivityNetwork(MetricId.COH, FrequencyBand(0, 1, 1.0), 2, tuple(range(n)), np.zeros((n, 3)), weights=wd)
    for f in (1e-6, 0.01, 0.37, 1.0):
        k = int(np.ceil(f * P))
        got = threshold_network(net, f)
        order = np.lexsort((np.arange(P), -np.abs(w.astype(np.float64))))
        want = np.sort(order[:k])
        assert got.n_edges == k
        assert np.array_equal(got._pairs.cpu().numpy(), want), f
        wi, wj = pair_to_ij(want, n)
        assert np.array_equal(got.edge_i, wi) and np.array_equal(got.edge_j, wj)
        assert np.array_equal(got.weights, w[want].astype(np.float64))
    nn = normalize_network(net)
    np.testing.assert_allclose(nn.weights, w / np.abs(w).max(), rtol=1e-6)


def test_threshold_fixture_selections_on_device():
    """The reference's threshold fixture (normalised COH / IMAGCOHY networks and
    their kept edge sets, regenerated from the reference into the golden file)
    through compute_metric -> normalize_network -> threshold_network on the device."""
    from conftest import GOLDEN
    from paper_2303_03279_b200.core import normalize_network, threshold_network
    g = np.load(GOLDEN / "sim2024_thresh.npz")
    eps = [EpochMatrix(data=e, sfreq=600.0, trial_index=k) for k, e in enumerate(g["epochs"])]
    for nm in ("COH", "IMAGCOHY"):
        dense = normalize_network(M.compute_metric(eps, MetricId[nm], 600, FrequencyBand(15, 21, 1.0)))
        assert np.abs(dense.weights - g["norm_" + nm]).max() <= 1e-4
        for f in (0.05, 0.10, 0.25):
            t = threshold_network(dense, f)
            want = g[f"thresh_{nm}_{f:.2f}"]
            assert np.array_equal(np.stack([t.edge_i, t.edge_j], 1), want), (nm, f)


# ---------------------------------------------------------------- time-domain metrics (metrics.py:140-260)
def test_cor_xcor_match_reference_golden():
    from conftest import GOLDEN
    g = np.load(GOLDEN / "timedomain.npz")
    eps = [EpochMatrix(data=e, sfreq=100.0, trial_index=k) for k, e in enumerate(g["epochs"])]
    net = M.compute_metric(eps, MetricId.COR, 64)
    assert np.abs(net.weights - g["cor_w"]).max() <= 1e-12
    assert list(net.warnings) == list(g["cor_warn"])
    for ml, key in ((10, "10"), (None, "all")):
        net = M.compute_metric(eps, MetricId.XCOR, 64, max_lag=ml)
        assert np.abs(net.weights - g["xcor_w_" + key]).max() <= 1e-12
        assert np.array_equal(net.lags, g["xcor_lag_" + key])


def test_xcor_pair_and_engine_time_domain():
    rng = np.random.default_rng(21)
    x = rng.standard_normal(50)
    y = np.roll(x, -4) + 0.1 * rng.standard_normal(50)       # x leads y
    assert M.xcor_pair(x, y, 10) == pytest.approx(O.xcor_pair(x, y, 10), abs=1e-12)
    assert M.xcor_pair(x, np.full(50, 3.0), 5) == (0.0, 0)
    with pytest.raises(ParameterError):
        M.xcor_pair(x, y, 50)
    eps = make_epochs(7, 5, 60, seed=22)
    for storage in (True, False):
        eng = M.ConnectivityEngine(5, 32, 600.0, storage_mode=storage, max_lag=12)
        for ep in eps:
            if storage:
                eng.add_trial(ep)
            else:
                eng.update_and_finalize(ep, MetricId.XCOR, FrequencyBand(0, 0, 0.0))
        w, _ = O.cor([e.data for e in eps])
        assert np.abs(eng.finalize(MetricId.COR, FrequencyBand(0, 0, 0.0)).weights - w).max() <= 1e-12
        a, lags = O.xcor([e.data for e in eps], 12)
        net = eng.finalize(MetricId.XCOR, FrequencyBand(0, 0, 0.0))
        assert np.abs(net.weights - a).max() <= 1e-12 and np.array_equal(net.lags, lags)
    # storage mode: a late switch to XCOR after rebuild_last back-fills from ALL cached epochs
    eng2 = M.ConnectivityEngine(5, 32, 600.0, storage_mode=True, max_lag=12)
    for ep in eps:
        eng2.add_trial(ep)
    eng2.rebuild_last(3)
    w3, _ = O.cor([e.data for e in eps[-3:]])
    assert np.abs(eng2.finalize(MetricId.COR, FrequencyBand(0, 0, 0.0)).weights - w3).max() <= 1e-12
    net = eng2.finalize(MetricId.XCOR, FrequencyBand(0, 0, 0.0))
    a, lags = O.xcor([e.data for e in eps], 12)                # reference quirk: all cached epochs
    assert net.n_trials == len(eps)
    assert np.abs(net.weights - a).max() <= 1e-12 and np.array_equal(net.lags, lags)


# ---------------------------------------------------------------- upstream
@pytest.mark.parametrize("taper", [None, "hann", ("dpss", 2.0, 3)])
def test_source_connectivity_projects_the_spectra(taper):
    """K1 on sensors + spectral projection = the reference path on M @ x."""
    from paper_2303_03279_b200.plan import make_taper
    from paper_2303_03279_b200.upstream import source_connectivity
    rng = np.random.default_rng(31)
    K, C, T, Ns, nfft, lo, hi = 8, 6, 96, 11, 128, 3, 20
    x = rng.standard_normal((K, C, T))
    Mx = rng.standard_normal((Ns, C))
    out, _ = source_connectivity(torch.tensor(x, device="cuda"), Mx, nfft, lo, hi, taper=taper)
    tp = make_taper(taper, min(T, nfft))
    tp = None if tp is None else (tp[0] if tp.shape[0] == 1 else tp)
    want, _ = O.compute([Mx @ e for e in x], nfft, lo, hi, taper=tp)
    for m in ("COH", "IMAGCOHY", "PLV", "PLI", "WPLI"):
        got = out[m]["bins"].T.cpu().numpy()
        assert np.abs(got - want[m]["bins"]).max() <= TOL[m], m


def test_apply_inverse_and_overlap_add_filter():
    from paper_2303_03279_b200.upstream import OverlapAddFilter, apply_inverse, filter_offline
    rng = np.random.default_rng(32)
    M_ = rng.standard_normal((9, 4))
    ep = EpochMatrix(data=rng.standard_normal((4, 50)), sfreq=100.0, trial_index=3)
    src = apply_inverse(M_, ep)
    np.testing.assert_allclose(src.data.cpu().numpy(), M_ @ ep.data, atol=1e-12)
    assert src.trial_index == 3
    taps = rng.standard_normal(21)
    sig = rng.standard_normal((3, 257))
    want = np.stack([np.convolve(s, taps)[:257] for s in sig])
    f = OverlapAddFilter(taps)
    got = np.concatenate([f.process(sig[:, a:b]).cpu().numpy() for a, b in ((0, 40), (40, 41), (41, 200), (200, 257))], 1)
    np.testing.assert_allclose(got, want, atol=1e-10)
    np.testing.assert_allclose(filter_offline(taps, sig).cpu().numpy(), want, atol=1e-10)
    with pytest.raises(ParameterError):
        f.process(sig[:2, :5])
