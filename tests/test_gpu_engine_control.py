"""The reference Pipeline's control path driven through the drop-in engine, and
ring-wrapped online windows, both checked against the oracle (not against
another GPU run).

The reference Pipeline cannot travel to the GPU box, so ``_ControlDriver``
restates exactly the engine calls it makes:

* ``submit_control`` (pipeline.py:157-166): a ``set_band`` whose hi bin is
  >= ``engine.acc.n_bins`` is rejected with the reference's message;
  ``set_average_count`` needs storage mode;
* ``_apply_pending_controls`` (pipeline.py:168-184): set_metric / set_band /
  set_average_count -> ``engine.rebuild_last(count)`` / reset_accumulators ->
  ``engine.reset()``;
* the backend step (pipeline.py:304-309): ``update_and_finalize`` and, while
  more trials than the average count are held, ``rebuild_last`` + ``finalize``.

After every step the network weights equal the oracle's band means over exactly
the trials the reference accumulator holds at that point.
"""
import queue

import numpy as np
import pytest
import torch

import oracle as O
from paper_2303_03279_b200 import ConnectivityEngine, EpochMatrix, FrequencyBand, MetricId
from paper_2303_03279_b200.core import ParameterError

pytestmark = pytest.mark.gpu
TOL = {"COH": 1e-4, "IMAGCOHY": 1e-4, "PLV": 1e-4, "PLI": 1e-3, "USPLI": 1e-3, "WPLI": 1e-3, "DSWPLI": 1e-3,
       "COHY": 1e-4}


class _Msg:
    def __init__(self, kind, **kw):
        self.kind = kind
        self.__dict__.update(kw)


class _ControlDriver:
    """pipeline.py:143-184 and 304-309, restated around a ConnectivityEngine."""

    def __init__(self, n_nodes, nfft, sfreq, band, metric, storage_mode=True):
        self.storage_mode = storage_mode
        self.engine = ConnectivityEngine(n_nodes, nfft, sfreq, storage_mode=storage_mode,
                                         accumulate_band=band if storage_mode else None)
        self.metric = MetricId.parse(metric)
        self.band = FrequencyBand(band[0], band[1], sfreq / nfft)
        self.average_count = None
        self.q = queue.Queue()

    def submit_control(self, msg):
        if msg.kind == "set_band":
            if msg.hi >= self.engine.acc.n_bins:
                return False, f"band exceeds {self.engine.acc.n_bins} bins"
        if msg.kind == "set_average_count" and not self.storage_mode:
            return False, "trial window control requires storage mode"
        self.q.put(msg)
        return True, ""

    def _apply(self):
        while not self.q.empty():
            msg = self.q.get_nowait()
            if msg.kind == "set_metric":
                self.metric = MetricId.parse(msg.metric)
            elif msg.kind == "set_band":
                self.band = FrequencyBand(msg.lo, msg.hi, self.band.bin_hz)
            elif msg.kind == "set_average_count":
                self.average_count = msg.count
                self.engine.rebuild_last(msg.count)
            elif msg.kind == "reset_accumulators":
                self.engine.reset()

    def step(self, ep):
        self._apply()
        net = self.engine.update_and_finalize(ep, self.metric, self.band)
        if self.average_count is not None and self.engine.n_trials > self.average_count:
            self.engine.rebuild_last(self.average_count)
            net = self.engine.finalize(self.metric, self.band)
        return net


def test_pipeline_control_path_against_oracle():
    rng = np.random.default_rng(31)
    K, N, T, nfft, fs = 26, 48, 200, 256, 256.0
    x = rng.standard_normal((K, N, T))
    x[:, 5] += 0.7 * np.roll(x[:, 4], 3, axis=-1)          # a lagged coupling
    drv = _ControlDriver(N, nfft, fs, (8, 20), "WPLI")
    assert drv.engine.acc.n_bins == nfft // 2 + 1
    # control schedule (applied before the step's trial, as in the backend loop)
    schedule = {
        3: [_Msg("set_metric", metric="PLI")],
        5: [_Msg("set_band", lo=2, hi=40)],
        8: [_Msg("set_average_count", count=4)],
        12: [_Msg("set_metric", metric="COH"), _Msg("set_band", lo=30, hi=60)],
        15: [_Msg("reset_accumulators")],
        18: [_Msg("set_metric", metric="IMAGCOHY")],
        21: [_Msg("set_average_count", count=3), _Msg("set_metric", metric="USPLI")],
    }
    ok, why = drv.submit_control(_Msg("set_band", lo=1, hi=nfft // 2 + 1))
    assert not ok and why == f"band exceeds {nfft // 2 + 1} bins"
    held = []                       # trial indices the reference accumulator holds
    for k in range(K):
        for msg in schedule.get(k, []):
            assert drv.submit_control(msg) == (True, "")
            if msg.kind == "set_average_count":
                held = sorted(held)[-msg.count:]
            elif msg.kind == "reset_accumulators":
                held = []
        net = drv.step(EpochMatrix(x[k], fs, trial_index=k))
        held.append(k)
        if drv.average_count is not None and len(held) > drv.average_count:
            held = sorted(held)[-drv.average_count:]
        m, b = drv.metric.value, drv.band
        if m == "USPLI" and len(held) < 2:
            continue
        want, _ = O.compute([x[i] for i in held], nfft, b.lo_bin, b.hi_bin, (m,))
        got = np.asarray(net.weights)
        err = np.abs(got - want[m]["band"]).max()
        assert err <= TOL[m], f"step {k} {m} {b.lo_bin}-{b.hi_bin} trials {held}: err {err:.3g}"
        assert net.n_trials == len(held)
        assert drv.engine.acc.n_trials_accumulated == len(held)
    # the accumulator view's running sums are the reference fold over the held trials
    acc = drv.engine.acc
    ref = O.Sums(N, acc.n_bins)
    for i in held:
        O.accumulate(ref, O.trial_spectra(x[i], nfft)[:, :])
    cols = np.zeros(acc.n_bins, bool)
    cols[8:21] = True       # rebuild_last resets to the accumulate band (metrics.py:450-460) ...
    cols[30:61] = True      # ... widened by the band finalized since (ensure_band, metrics.py:363-380)
    np.testing.assert_allclose(acc.csd_sum[:, cols], ref.csd_sum[:, cols], rtol=1e-9, atol=1e-9)
    np.testing.assert_array_equal(acc.pli_sum[:, cols], ref.pli_sum[:, cols])
    assert np.all(acc.csd_sum[:, ~cols] == 0)


def test_set_average_count_requires_storage_mode():
    drv = _ControlDriver(8, 64, 64.0, (1, 5), "PLV", storage_mode=False)
    assert drv.submit_control(_Msg("set_average_count", count=3)) == (False,
                                                                       "trial window control requires storage mode")
    with pytest.raises(ParameterError):
        drv.engine.rebuild_last(3)


def test_ring_wrapped_online_windows_against_oracle():
    """WindowGraph (the ring = the window, new trials overwrite the ones that left)
    over a stream: windows long after the ring wrapped equal the oracle's metrics
    over trials [step u, step u + window)."""
    from paper_2303_03279_b200.plan import DevicePlan, WindowGraph, pow2_scale
    rng = np.random.default_rng(41)
    win, new, N, T, nfft, lo, hi = 12, 5, 80, 128, 128, 4, 18
    n_up = 11                                        # 12 / gcd(12, 5) = 12 phases; the ring wraps 4 times
    x = rng.standard_normal((win + new * n_up, N, T))
    x[:, 7] += 0.6 * np.roll(x[:, 3], 2, axis=-1)
    xt = torch.tensor(x, dtype=torch.float32, device="cuda")
    scale = pow2_scale(float(np.abs(x).max()), min(T, nfft))
    metrics = ("COH", "IMAGCOHY", "PLV", "PLI", "USPLI", "WPLI", "DSWPLI")
    plan = DevicePlan(N, T, nfft, lo, hi, taper="hann", slot_capacity=win, device="cuda", scale=scale)
    wg = WindowGraph(plan, new, metrics)
    wg.prime(xt[:win])
    xf = xt.double().cpu().numpy()                   # the fp32 samples the GPU saw
    for u in range(1, n_up + 1):
        got = wg.update(xt[win + new * (u - 1): win + new * u])
        if u in (3, 6, 10, 11):
            want, _ = O.compute(list(xf[new * u: new * u + win]), nfft, lo, hi, metrics, taper=np.hanning(T))
            for m in metrics:
                e = np.abs(got[m]["bins"].T.cpu().numpy() - want[m]["bins"]).max()
                eb = np.abs(got[m]["band"].cpu().numpy() - want[m]["band"]).max()
                assert max(e, eb) <= TOL[m], f"update {u} {m}: {e:.3g} / {eb:.3g}"
