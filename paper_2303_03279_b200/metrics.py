"""Drop-in for connstream.metrics (reference src/metrics.py) on the B200 path.

Per-bin finalisers, band-averaged networks, the batch entry point and the
storage-mode engine, with the reference's names, signatures and errors.  Every
spectral metric is computed by the fused device kernels (cs_pair_metrics):
  COH / COHY / PLV      -> tcgen05 tensor-core kernel (K2)
  IMAGCOHY / PLI family -> FP32 pair x trial kernel with fp64 exact-sign guard (K3)

Reference anchors: metrics.py:32-98 (*_bins, _SPECTRAL_BINS), :101-134
(_build_network, finalize_spectral), :267-460 (TrialCache, ConnectivityEngine),
:465-498 (one-shot wrappers), :501-528 (convergence_curve), :531-551
(compute_metric).  COR / XCOR (time-domain, :137-260) in timedomain.py.
"""
from __future__ import annotations

from collections.abc import MutableMapping
from dataclasses import dataclass, field

import numpy as np
import torch

from . import spectral, timedomain
from .core import (ConnectivityNetwork, DegenerateTrialCountError, EpochMatrix, FrequencyBand, MetricId,
                   ParameterError, default_positions)
from .plan import DevicePlan, pow2_scale
from .spectral import SpectrumSet, pair_index


def _full_band(acc, band):
    return band if band is not None else FrequencyBand(0, acc.n_bins - 1, 0.0)


def _check_k(K: int, metric: str):
    if K < 1:
        raise DegenerateTrialCountError("no trials accumulated")
    if metric == "USPLI" and K < 2:
        raise DegenerateTrialCountError("USPLI needs at least 2 trials")


def _bins_from_sums(acc: SpectrumSet, metric: str, band, want_band=False):
    """The reference's finalisers (metrics.py:32-98) over the running sums of every fold
    (cs_pair_sums, fp64 reference arithmetic) -- the path for an accumulator whose columns
    were folded from different trial sets (accumulate_spectra ``bins`` / ``count=False``,
    spectral.py:216-261), where no single slot list serves every column.  The sums'
    normalisation is the reference's: n_trials_accumulated for PLV / PLI / USPLI."""
    plan = acc.plan
    lo, nbb = band.lo_bin, band.n_bins
    slots = torch.tensor([s for s, _ in acc._entries], dtype=torch.int32, device=plan.device)
    o = plan.pair_sums(slots, lo, nbb)                   # bin-major [nbb, P] / [nbb, C]
    K = float(acc.n_trials_accumulated)
    pi, pj = (torch.as_tensor(v, device=plan.device) for v in pair_index(acc.n_channels))
    tiny = float(np.finfo(np.float64).tiny)
    if metric in ("COHY", "COH", "IMAGCOHY"):
        den = torch.sqrt(o["psd"][:, pi] * o["psd"][:, pj])
        cohy_v = torch.where(den > tiny, o["csd"] / torch.where(den > tiny, den, 1.0), torch.zeros_like(o["csd"]))
        val = cohy_v if metric == "COHY" else (cohy_v.abs() if metric == "COH" else cohy_v.imag)
    elif metric == "PLV":
        val = o["plv"].abs() / K
    elif metric in ("PLI", "USPLI"):
        pli = o["pli"].to(torch.float64).abs() / K
        val = pli if metric == "PLI" else (K * pli * pli - 1.0) / (K - 1.0)
    else:  # WPLI, DSWPLI
        num, den = o["csd"].imag.abs(), o["abs_im"]
        w = torch.where(den > 0.0, num / torch.where(den > 0.0, den, 1.0), torch.zeros_like(num))
        val = w if metric == "WPLI" else w * w
    bins = val.to(torch.complex64 if metric == "COHY" else torch.float32)
    out = {"bins": bins}
    if want_band:  # core.py:208-215 / metrics.py:124-134: arithmetic mean over the band
        out["band"] = val.mean(dim=0).to(bins.dtype)
    return out


def _device_bins(acc: SpectrumSet, metric: str, band, want_band=False):
    """Run the pair kernels for ``metric`` over acc's folded trials -> device
    tensors (bins [nb, P], band [P])."""
    band = _full_band(acc, band)
    _check_k(acc.n_trials_accumulated, metric)
    if band.hi_bin >= acc.n_bins:
        raise ParameterError(f"band [{band.lo_bin}, {band.hi_bin}] exceeds {acc.n_bins} bins")
    slots = acc.slots_for(band.lo_bin, band.hi_bin)
    if slots is None or len(slots) != acc.n_trials_accumulated:
        return _bins_from_sums(acc, metric, band, want_band)
    plan = acc.plan
    st = torch.tensor(slots, dtype=torch.int32, device=plan.device)
    out = plan.pair_metrics(st, (metric,), band.lo_bin, band.n_bins, per_bin=True, band=want_band)
    return out[metric]


def _host_bins(acc, metric, band):
    o = _device_bins(acc, metric, band)["bins"]
    arr = o.t().contiguous().cpu().numpy()
    return arr.astype(np.complex128 if metric == "COHY" else np.float64)


def cohy_bins(acc: SpectrumSet, band: FrequencyBand | None = None) -> np.ndarray:
    """Complex coherency per pair and bin [P, nb] (metrics.py:32-42)."""
    return _host_bins(acc, "COHY", band)


def coh_bins(acc, band=None):
    return _host_bins(acc, "COH", band)


def imagcohy_bins(acc, band=None):
    return _host_bins(acc, "IMAGCOHY", band)


def plv_bins(acc, band=None):
    return _host_bins(acc, "PLV", band)


def pli_bins(acc, band=None):
    return _host_bins(acc, "PLI", band)


def uspli_bins(acc, band=None):
    return _host_bins(acc, "USPLI", band)


def wpli_bins(acc, band=None):
    return _host_bins(acc, "WPLI", band)


def dswpli_bins(acc, band=None):
    return _host_bins(acc, "DSWPLI", band)


_SPECTRAL_BINS = {
    MetricId.COHY: cohy_bins,
    MetricId.COH: coh_bins,
    MetricId.IMAGCOHY: imagcohy_bins,
    MetricId.PLV: plv_bins,
    MetricId.PLI: pli_bins,
    MetricId.USPLI: uspli_bins,
    MetricId.WPLI: wpli_bins,
    MetricId.DSWPLI: dswpli_bins,
}


def _build_network(metric, band, n_trials, n_channels, weights, complex_weights=None, lags=None, positions=None,
                   node_ids=None, warnings=()):
    if positions is None:
        positions = default_positions(n_channels)
    if node_ids is None:
        node_ids = tuple(range(n_channels))
    return ConnectivityNetwork(metric=metric, band=band, n_trials=n_trials, node_ids=node_ids,
                               positions=positions, weights=weights, complex_weights=complex_weights,
                               lags=lags, warnings=tuple(warnings))


def _network_from_band(metric: MetricId, band, n_trials, n_channels, band_out, positions, node_ids):
    if metric is MetricId.COHY:
        cm = band_out.to(torch.complex128)
        return _build_network(metric, band, n_trials, n_channels, cm.abs(), cm, positions=positions,
                              node_ids=node_ids)
    return _build_network(metric, band, n_trials, n_channels, band_out.double(), positions=positions,
                          node_ids=node_ids)


def finalize_spectral(acc: SpectrumSet, metric: MetricId, band: FrequencyBand, positions=None,
                      node_ids=None) -> ConnectivityNetwork:
    """Band-averaged network for one spectral metric (metrics.py:115-134)."""
    if metric not in _SPECTRAL_BINS:
        raise ParameterError(f"{metric} is not a spectral metric")
    band = out_band = _full_band(acc, band)
    if metric is MetricId.COHY and band.lo_bin < acc.n_bins <= band.hi_bin:
        # the reference's numpy slice clips the band and its COHY mean has no range
        # check (metrics.py:121-127): the mean runs over the bins that exist
        band = FrequencyBand(band.lo_bin, acc.n_bins - 1, band.bin_hz)
    _check_k(acc.n_trials_accumulated, metric.value)
    slots = acc.slots_for(band.lo_bin, band.hi_bin)
    if slots is None or len(slots) != acc.n_trials_accumulated:  # mixed column sets: the sums path
        if band.hi_bin >= acc.n_bins:
            raise ParameterError(f"band [{band.lo_bin}, {band.hi_bin}] exceeds {acc.n_bins} bins")
        w = _bins_from_sums(acc, metric.value, band, want_band=True)["band"]
        return _network_from_band(metric, out_band, acc.n_trials_accumulated, acc.n_channels, w, positions, node_ids)
    if band.hi_bin >= acc.n_bins:   # core.py:208-215 on the reference's clipped per-bin array
        raise ParameterError(f"band [{band.lo_bin}, {band.hi_bin}] exceeds {acc.n_bins} bins")
    plan = acc.plan
    st = torch.tensor(slots, dtype=torch.int32, device=plan.device)
    out = plan.pair_metrics(st, (metric.value,), band.lo_bin, band.n_bins, per_bin=False, band=True)
    return _network_from_band(metric, out_band, acc.n_trials_accumulated, acc.n_channels, out[metric.value]["band"],
                              positions, node_ids)


# one-shot wrappers (metrics.py:465-498)
def cohy(acc, band=None, **kw):
    return finalize_spectral(acc, MetricId.COHY, _full_band(acc, band), **kw)


def coh(acc, band=None, **kw):
    return finalize_spectral(acc, MetricId.COH, _full_band(acc, band), **kw)


def imagcohy(acc, band=None, **kw):
    return finalize_spectral(acc, MetricId.IMAGCOHY, _full_band(acc, band), **kw)


def plv(acc, band=None, **kw):
    return finalize_spectral(acc, MetricId.PLV, _full_band(acc, band), **kw)


def pli(acc, band=None, **kw):
    return finalize_spectral(acc, MetricId.PLI, _full_band(acc, band), **kw)


def uspli(acc, band=None, **kw):
    return finalize_spectral(acc, MetricId.USPLI, _full_band(acc, band), **kw)


def wpli(acc, band=None, **kw):
    return finalize_spectral(acc, MetricId.WPLI, _full_band(acc, band), **kw)


def dswpli(acc, band=None, **kw):
    return finalize_spectral(acc, MetricId.DSWPLI, _full_band(acc, band), **kw)


def _stack_epochs(epochs):
    ts = [e.data if isinstance(e.data, torch.Tensor) else torch.as_tensor(e.data) for e in epochs]
    T = ts[0].shape[1]
    if any(t.shape != ts[0].shape for t in ts):
        raise ParameterError("epochs must have equal shapes")
    dt = torch.float32 if all(t.dtype == torch.float32 for t in ts) else torch.float64
    return torch.stack([t.to(dt) for t in ts]).to(spectral._device()), T


def compute_metric(epochs, metric: MetricId, nfft: int, band: FrequencyBand | None = None,
                   max_lag: int | None = None, positions=None, node_ids=None, taper=None) -> ConnectivityNetwork:
    """One-shot batch computation over a list of epochs (metrics.py:531-551):
    K1 over every node x trial, then the fused pair kernels over all trials."""
    metric = metric if isinstance(metric, MetricId) else MetricId.parse(metric)
    if metric is MetricId.COR:
        return cor(epochs, band=band, positions=positions, node_ids=node_ids)
    if metric is MetricId.XCOR:
        return xcor(epochs, max_lag=max_lag, band=band, positions=positions, node_ids=node_ids)
    if not epochs:
        raise ParameterError("need at least one epoch")
    if nfft < 2:
        raise ParameterError(f"nfft must be >= 2, got {nfft}")
    if len({tuple(e.data.shape) for e in epochs}) > 1:
        # epochs of different lengths: each is cropped / padded to nfft on its own, as the
        # reference's per-trial path does (spectral.py:49-97, metrics.py:541-551)
        acc = SpectrumSet(epochs[0].n_channels, nfft)
        for e in epochs:
            spectral.accumulate_epoch(acc, e, taper=taper)
        if band is None:
            band = FrequencyBand(0, acc.n_bins - 1, epochs[0].sfreq / nfft)
        return finalize_spectral(acc, metric, band, positions=positions, node_ids=node_ids)
    x, T = _stack_epochs(epochs)
    K, C = x.shape[0], x.shape[1]
    if band is None:
        band = FrequencyBand(0, nfft // 2, epochs[0].sfreq / nfft)
    if band.hi_bin > nfft // 2:
        raise ParameterError(f"band [{band.lo_bin}, {band.hi_bin}] exceeds {nfft // 2 + 1} bins")
    _check_k(K, metric.value)
    plan = DevicePlan(C, T, nfft, band.lo_bin, band.hi_bin, taper=taper, slot_capacity=K, device=x.device,
                      scale=pow2_scale(float(x.abs().amax()), min(T, nfft)))
    plan.spectra(x, 0)
    spectral._count_ffts(K * C * plan.n_tapers)
    slots = torch.arange(K, dtype=torch.int32, device=x.device)
    out = plan.pair_metrics(slots, (metric.value,), 0, plan.n_bins, per_bin=False, band=True)
    return _network_from_band(metric, band, K, C, out[metric.value]["band"], positions, node_ids)


def cor(epochs, band: FrequencyBand | None = None, positions=None, node_ids=None) -> ConnectivityNetwork:
    """Pearson correlation per pair averaged over epochs (metrics.py:158-177)."""
    if not epochs:
        raise ParameterError("need at least one epoch")
    C = epochs[0].n_channels
    if any(ep.n_channels != C for ep in epochs):
        raise ParameterError("epochs must have equal channel counts")
    total, dead = timedomain.cor_sums([ep.data for ep in epochs], C)
    if band is None:
        band = FrequencyBand(0, 0, 0.0)
    return _build_network(MetricId.COR, band, len(epochs), C, total / len(epochs), positions=positions,
                          node_ids=node_ids, warnings=tuple(f"zero-variance channel {c}" for c in dead))


def xcor(epochs, max_lag: int | None = None, band: FrequencyBand | None = None, positions=None, node_ids=None,
         method: str = "fft") -> ConnectivityNetwork:
    """Cross-correlation peak per pair averaged over epochs; weight = |mean peak|,
    lag = rounded mean peak lag (metrics.py:229-260)."""
    if not epochs:
        raise ParameterError("need at least one epoch")
    if method not in ("fft", "direct"):
        raise ParameterError(f"unknown xcor method {method!r}")
    C = epochs[0].n_channels
    n = epochs[0].n_samples
    if max_lag is None:
        max_lag = n - 1
    peak, lag = timedomain.xcor_sums([ep.data for ep in epochs], C, max_lag)
    K = len(epochs)
    lags = np.rint(lag.cpu().numpy() / K).astype(np.int64)
    if band is None:
        band = FrequencyBand(0, 0, 0.0)
    return _build_network(MetricId.XCOR, band, K, C, (peak / K).abs(), lags=lags, positions=positions,
                          node_ids=node_ids)


xcor_pair = timedomain.xcor_pair


@dataclass
class TrialCache:
    """Storage mode (metrics.py:267-282).  In an engine ``spectra`` maps trial_index to
    the cached spectra (complex128 [C, n_bins], read from the ring slot on access)."""

    enabled: bool = True
    spectra: dict = field(default_factory=dict)
    epochs: dict = field(default_factory=dict)
    bytes_per_trial: int = 0

    def memory_bytes(self) -> int:
        """Cached spectra (their ring slots) plus the cached epochs' samples, as the
        reference counts them (metrics.py:279-282)."""
        return len(self.spectra) * self.bytes_per_trial + sum(int(e.data.nbytes) for e in self.epochs.values())


class _RingSpectra(MutableMapping):
    """trial_index -> the spectra the reference caches for it (metrics.py:341-347: the trial
    spectra, or a welch trial's first segment), kept in the engine's HBM ring and copied
    to the host only when an entry is read."""

    def __init__(self, engine: "ConnectivityEngine"):
        self._e = engine
        self._slots: dict = {}

    def __setitem__(self, idx, slot: int) -> None:
        self._slots[idx] = slot

    def __getitem__(self, idx):
        e = self._e
        slot = e._seg0_of.get(idx, self._slots[idx])
        sp = e._plan.get_spectra(torch.tensor([slot], dtype=torch.int32, device=e._plan.device))
        return sp[0].cpu().numpy()

    def __delitem__(self, idx) -> None:
        del self._slots[idx]

    def __iter__(self):
        return iter(self._slots)

    def __len__(self) -> int:
        return len(self._slots)


class ConnectivityEngine:
    """Storage-mode engine over an HBM spectrum ring (metrics.py:285-460).

    Every added trial's full-bin spectra are computed once (K1) into a ring
    slot.  finalize() runs the fused pair kernels over the slots of the trials
    currently folded, so switching metric or band issues no new FFTs, and
    rebuild_last(n) is a change of slot list (no re-fold).
    """

    def __init__(self, n_channels: int, nfft: int, sfreq: float, storage_mode: bool = True,
                 max_lag: int | None = None, spectral_mode: str = "fixed", positions=None, node_ids=None,
                 accumulate_band: tuple | None = None, taper=None, slot_capacity: int = 64):
        if spectral_mode not in ("fixed", "welch"):
            raise ParameterError(f"unknown spectral mode {spectral_mode!r}")
        if spectral_mode == "welch" and taper is not None:
            raise ParameterError("welch mode takes no taper")
        self.n_channels = n_channels
        self.nfft = nfft
        self.sfreq = sfreq
        self.bin_hz = sfreq / nfft
        self.spectral_mode = spectral_mode
        self.max_lag = max_lag
        self.positions = positions
        self.node_ids = node_ids
        self.taper = taper
        self.n_bins = nfft // 2 + 1
        if accumulate_band is not None and storage_mode and spectral_mode == "fixed":
            lo, hi = accumulate_band
            if not (0 <= lo <= hi < self.n_bins):
                raise ParameterError(f"accumulate_band [{lo}, {hi}] outside {self.n_bins} bins")
        self._accumulate_band = accumulate_band
        # columns the reference's accumulator holds (metrics.py:314-322, 363-380): the
        # accumulate band in storage mode, widened by ensure_band; the ring keeps all bins
        self._storage_mode = storage_mode
        self._init_cols()
        self.cache = TrialCache(enabled=storage_mode)
        self.cache.spectra = _RingSpectra(self)
        self._slot_capacity = max(int(slot_capacity), 1)
        self._plan: DevicePlan | None = None
        self._T = None
        self._next_slot = 0
        self._slot_of: dict = {}
        self._seg0_of: dict = {}     # welch: slot holding only the first segment (the cached spectra)
        self._mixed = False          # widened ring: every trial through _slot_other_length
        self._plans_by_length: dict = {}
        self._sum_trials: list = []
        self._fold_epochs: list = []  # the epoch given at each fold (COR sums, metrics.py:355-357)
        self._fold_slots: list = []  # ring slot of every fold, in order
        self.n_trials = 0
        # time-domain state (metrics.py:320-326): COR sums are kept eagerly only
        # without storage mode (with it they are recomputed from the cached epochs of
        # the folded trials); XCOR peaks follow the reference's lazy/backfill rules
        self._cor_sum = None
        self._dead_channels: set = set()
        self._xcor_peak_sum = None
        self._xcor_lag_sum = None
        self._xcor_trials = 0
        self._pending: list = []     # device epochs whose finiteness flag is not read yet

    def _init_cols(self) -> None:
        self._acc_cols = np.ones(self.n_bins, dtype=bool)
        ab = self._accumulate_band
        if ab is not None and self._storage_mode and self.spectral_mode == "fixed":
            self._acc_cols[:] = False
            self._acc_cols[ab[0]:ab[1] + 1] = True

    def _validate_pending(self) -> None:
        """One host read for all device epochs added since the last finalize
        (core.py:97-100 raises ParameterError for non-finite samples)."""
        if self._pending:
            flags = torch.stack([e.__dict__["_finite_dev"] for e in self._pending])
            pend, self._pending = self._pending, []
            if not bool(flags.all()):
                for e in pend:
                    e.validate()

    # -- ring ------------------------------------------------------------------
    def _ensure_plan(self, T: int, scale: float, n_tapers: int = 0):
        """Room for two more slots (and ``n_tapers`` taper slots per trial).  The ring
        is grown by doubling; it is widened only for a welch trial with more segments
        than the ring holds, after which it is a rectangular ring filled through
        per-length plans (``_mixed``)."""
        need = self._next_slot + 2
        grow = self._plan is None or need > self._plan.slot_capacity
        widen = self._plan is not None and n_tapers > self._plan.n_tapers
        if not (grow or widen):
            return
        dev = spectral._device()
        if self._plan is None:
            new = DevicePlan(self.n_channels, T, self.nfft, 0, self.n_bins - 1, taper=self.taper,
                             slot_capacity=max(self._slot_capacity, need), device=dev, scale=scale,
                             welch=self.spectral_mode == "welch")
            self._T = T
        else:
            cap = max(2 * self._plan.slot_capacity, need) if grow else self._plan.slot_capacity
            self._mixed = self._mixed or widen
            if self._mixed:
                new = DevicePlan(self.n_channels, self._T, self.nfft, 0, self.n_bins - 1, slot_capacity=cap,
                                 device=dev, scale=self._plan.scale,
                                 n_tapers=max(n_tapers, self._plan.n_tapers))
            else:
                new = DevicePlan(self.n_channels, self._T, self.nfft, 0, self.n_bins - 1, taper=self.taper,
                                 slot_capacity=cap, device=dev, scale=self._plan.scale,
                                 welch=self.spectral_mode == "welch")
            o64, o32 = self._plan.ring()
            n64, n32 = new.ring()
            L = o64.shape[1]
            n64[: o64.shape[0], :L].copy_(o64)
            n32[: o32.shape[0], :L].copy_(o32)
            n64[: o64.shape[0], L:].zero_()    # segments a widened ring adds: nothing folded
            n32[: o32.shape[0], L:].zero_()
        self._plan = new
        self.cache.bytes_per_trial = self.n_channels * self.n_bins * 24 * new.n_tapers

    def _length_plan(self, T: int) -> DevicePlan:
        """K1 plan for trials of ``T`` samples other than the ring's own length
        (same taper / welch rule and fp32 scale as the ring)."""
        p = self._plans_by_length.get(T)
        if p is None:
            if len(self._plans_by_length) >= 8:      # bounded: one plan per recent length
                self._plans_by_length.pop(next(iter(self._plans_by_length)))
            p = DevicePlan(self.n_channels, T, self.nfft, 0, self.n_bins - 1, taper=self.taper, slot_capacity=1,
                           device=spectral._device(), scale=self._plan.scale, welch=self.spectral_mode == "welch")
            self._plans_by_length[T] = p
        return p

    def _slot_other_length(self, x: torch.Tensor, idx) -> int:
        """A trial whose length differs from the ring's: its own plan computes the
        spectra (crop / pad to nfft, or welch segments when n_samples >= 2 nfft --
        spectral.py:264-286 decides per trial), copied into a ring slot; taper slots
        past its own segments stay zero, which adds nothing to any sum."""
        aux = self._length_plan(x.shape[1])
        L = aux.n_tapers
        self._ensure_plan(self._T, 1.0, n_tapers=L)
        aux.spectra(x[None].contiguous(), 0)
        spectral._count_ffts(self.n_channels * L)
        a64, a32 = aux.ring()
        r64, r32 = self._plan.ring()
        slot = self._next_slot
        self._next_slot += 1
        r64[slot, L:].zero_()
        r32[slot, L:].zero_()
        r64[slot, :L].copy_(a64[0])
        r32[slot, :L].copy_(a32[0])
        if aux.welch:
            s0 = self._next_slot
            self._next_slot += 1
            r64[s0].zero_()
            r32[s0].zero_()
            r64[s0, 0].copy_(a64[0, 0])
            r32[s0, 0].copy_(a32[0, 0])
            w = 1.0 / float(np.sqrt(L))
            r64[slot].mul_(w)
            r32[slot].mul_(w)
            self._seg0_of[idx] = s0
        return slot

    def _slot_ring_length(self, x: torch.Tensor, idx, data) -> int:
        # the fp32 scale is fixed by the first trial (host data: no device sync)
        scale = 1.0 if self._plan is not None else pow2_scale(_abs_max(data), min(x.shape[1], self.nfft))
        self._ensure_plan(x.shape[1], scale)
        slot = self._next_slot
        self._next_slot += 1
        self._plan.spectra(x[None].contiguous(), slot)
        spectral._count_ffts(self.n_channels * self._plan.n_tapers)
        if self._plan.welch:
            # the reference caches the first segment's spectra (spectral.py:286) and
            # re-folds cached trials in fixed mode (metrics.py:337-341, 450-460):
            # keep that segment in a slot of its own, then weight the welch slot's
            # S segments by 1/sqrt(S) so its summed CSD is the segment mean
            S = self._plan.n_tapers
            r64, r32 = self._plan.ring()
            s0 = self._next_slot
            self._next_slot += 1
            r64[s0].zero_()
            r32[s0].zero_()
            r64[s0, 0].copy_(r64[slot, 0])
            r32[s0, 0].copy_(r32[slot, 0])
            w = 1.0 / float(np.sqrt(S))
            r64[slot].mul_(w)
            r32[slot].mul_(w)
            self._seg0_of[idx] = s0
        return slot

    # -- accumulation -------------------------------------------------------------
    def add_trial(self, epoch: EpochMatrix) -> None:
        if epoch.n_channels != self.n_channels:
            raise ParameterError(f"epoch has {epoch.n_channels} channels, engine expects {self.n_channels}")
        idx = epoch.trial_index
        if not (self.cache.enabled and idx in self._slot_of):
            x = spectral._as_device_samples(epoch.data)
            if self._plan is not None and (self._mixed or x.shape[1] != self._T):
                slot = self._slot_other_length(x, idx)
            else:
                slot = self._slot_ring_length(x, idx, epoch.data)
            self._slot_of[idx] = slot
            if self.cache.enabled:
                self.cache.spectra[idx] = slot
            fold_slot = slot
        else:  # cached trial: the reference folds its cached (first-segment) spectra
            fold_slot = self._seg0_of.get(idx, self._slot_of[idx])
        if epoch.__dict__.get("_finite_dev") is not None:
            self._pending.append(epoch)       # device samples: finiteness checked at finalize
        if self.cache.enabled:
            self.cache.epochs[idx] = epoch
        else:  # no cache to recompute from: fold the trial's Pearson matrix now
            w, dead = timedomain.cor_sums([epoch.data], self.n_channels)
            self._cor_sum = w if self._cor_sum is None else self._cor_sum + w
            self._dead_channels.update(dead)
        self._sum_trials.append(idx)
        self._fold_epochs.append(epoch)
        self._fold_slots.append(fold_slot)
        self.n_trials += 1

    def _xcor_add(self, epochs) -> None:
        # without a max_lag each trial uses its own n_samples - 1 (metrics.py:385)
        groups: dict = {}
        for e in epochs:
            groups.setdefault(self.max_lag if self.max_lag is not None else e.n_samples - 1, []).append(e)
        for max_lag, grp in groups.items():
            pk, lg = timedomain.xcor_sums([e.data for e in grp], self.n_channels, max_lag)
            if self._xcor_peak_sum is None:
                self._xcor_peak_sum, self._xcor_lag_sum = pk, lg
            else:
                self._xcor_peak_sum += pk
                self._xcor_lag_sum += lg
        self._xcor_trials += len(epochs)

    def _finalize_time_domain(self, metric: MetricId, band: FrequencyBand) -> ConnectivityNetwork:
        if self.n_trials < 1:
            raise DegenerateTrialCountError("no trials accumulated")
        if metric is MetricId.COR:
            if self.cache.enabled:
                total, dead = timedomain.cor_sums([e.data for e in self._fold_epochs],
                                                  self.n_channels)
            else:
                total, dead = self._cor_sum, sorted(self._dead_channels)
            warnings = tuple(f"zero-variance channel {c}" for c in dead)
            return _build_network(MetricId.COR, band, self.n_trials, self.n_channels, total / self.n_trials,
                                  positions=self.positions, node_ids=self.node_ids, warnings=warnings)
        # XCOR: backfill from the cached epochs (sorted by index) past the ones
        # already processed, as the reference does (metrics.py:418-428)
        if self._xcor_trials < self.n_trials:
            if not self.cache.enabled:
                raise ParameterError("switching to XCOR mid-session requires storage mode")
            todo = [self.cache.epochs[i] for i in sorted(self.cache.epochs)[self._xcor_trials:]]
            if todo:
                self._xcor_add(todo)
        mean_peak = self._xcor_peak_sum / self._xcor_trials
        lags = np.rint(self._xcor_lag_sum.cpu().numpy() / self._xcor_trials).astype(np.int64)
        return _build_network(MetricId.XCOR, band, self._xcor_trials, self.n_channels, mean_peak.abs(), lags=lags,
                              positions=self.positions, node_ids=self.node_ids)

    def ensure_band(self, band: FrequencyBand) -> None:
        """All bins are cached on the device, so back-fill needs no FFT (metrics.py:363-380);
        only the accumulator's column set widens."""
        self._acc_cols[band.lo_bin:band.hi_bin + 1] = True   # a numpy slice: clipped at n_bins

    @property
    def acc(self) -> "EngineSpectrumSet":
        """The reference engine's ``acc`` (a SpectrumSet over the folded trials,
        metrics.py:306): shape attributes, and the running sums on access."""
        return EngineSpectrumSet(self)

    # -- finalization ---------------------------------------------------------------
    def _slots(self):
        return torch.tensor(self._fold_slots, dtype=torch.int32, device=self._plan.device)

    def finalize(self, metric: MetricId, band: FrequencyBand) -> ConnectivityNetwork:
        metric = metric if isinstance(metric, MetricId) else MetricId.parse(metric)
        self._validate_pending()
        if not metric.is_spectral:
            return self._finalize_time_domain(metric, band)
        self.ensure_band(band)
        _check_k(len(self._sum_trials), metric.value)
        calc = band
        if band.hi_bin >= self.n_bins:   # as finalize_spectral: COHY over the bins that exist, else an error
            if metric is not MetricId.COHY or band.lo_bin >= self.n_bins:
                raise ParameterError(f"band [{band.lo_bin}, {band.hi_bin}] exceeds {self.n_bins} bins")
            calc = FrequencyBand(band.lo_bin, self.n_bins - 1, band.bin_hz)
        out = self._plan.pair_metrics(self._slots(), (metric.value,), calc.lo_bin, calc.n_bins, per_bin=False,
                                      band=True)
        return _network_from_band(metric, band, len(self._sum_trials), self.n_channels, out[metric.value]["band"],
                                  self.positions, self.node_ids)

    def update_and_finalize(self, new_epoch: EpochMatrix, metric: MetricId, band: FrequencyBand):
        metric = metric if isinstance(metric, MetricId) else MetricId.parse(metric)
        self.add_trial(new_epoch)
        if metric is MetricId.XCOR and not self.cache.enabled:
            # without storage nothing can be back-filled later: keep XCOR in lockstep
            self._xcor_add([new_epoch])
        return self.finalize(metric, band)

    def reset(self) -> None:
        self.__init__(self.n_channels, self.nfft, self.sfreq, storage_mode=self.cache.enabled,
                      max_lag=self.max_lag, spectral_mode=self.spectral_mode, positions=self.positions,
                      node_ids=self.node_ids, accumulate_band=self._accumulate_band, taper=self.taper,
                      slot_capacity=self._slot_capacity)

    def rebuild_last(self, n_last: int) -> None:
        """Sums over the most recent ``n_last`` cached trials (metrics.py:450-460):
        a new slot list over the cached spectra, no FFTs and no re-fold."""
        if not self.cache.enabled:
            raise ParameterError("trial-window rebuild requires storage mode")
        keep = sorted(self.cache.epochs)[-n_last:]   # as the reference slices: n_last = 0 keeps all
        # the reference resets (time-domain sums included) and re-adds the kept trials
        self._xcor_peak_sum = self._xcor_lag_sum = None
        self._xcor_trials = 0
        self._sum_trials = list(keep)
        self._fold_epochs = [self.cache.epochs[i] for i in keep]
        self._init_cols()   # the reference's reset() restores the accumulate-band mask
        # re-added from the cache: fixed-mode folds of the cached spectra
        self._fold_slots = [self._seg0_of.get(i, self._slot_of[i]) for i in keep]
        self.n_trials = len(keep)


def _abs_max(data) -> float:
    if isinstance(data, torch.Tensor):
        return float(data.abs().amax()) if data.numel() else 0.0
    a = np.asarray(data)
    return float(np.abs(a).max()) if a.size else 0.0


class EngineSpectrumSet:
    """Read-only SpectrumSet view of a ConnectivityEngine (the reference Pipeline
    reads ``engine.acc.n_bins``, pipeline.py:161-162).  The sums are the
    reference's fold over the engine's current trials (cs_pair_sums, fp64),
    zero outside the columns the reference accumulator would hold."""

    def __init__(self, engine: "ConnectivityEngine"):
        self._e = engine
        self._cache = None

    n_channels = property(lambda self: self._e.n_channels)
    nfft = property(lambda self: self._e.nfft)
    n_bins = property(lambda self: self._e.n_bins)
    n_pairs = property(lambda self: self._e.n_channels * (self._e.n_channels - 1) // 2)
    n_trials_accumulated = property(lambda self: len(self._e._sum_trials))

    def _sums(self) -> dict:
        if self._cache is None:
            e = self._e
            C, B, P = self.n_channels, self.n_bins, self.n_pairs
            out = {"csd": np.zeros((P, B), np.complex128), "psd": np.zeros((C, B)),
                   "plv": np.zeros((P, B), np.complex128), "pli": np.zeros((P, B)), "abs_im": np.zeros((P, B))}
            if e._fold_slots:
                o = e._plan.pair_sums(e._slots())
                cols = e._acc_cols
                for k in ("csd", "plv", "pli", "abs_im", "psd"):
                    v = o[k].T.cpu().numpy()
                    out[k][:, cols] = v[:, cols]
            self._cache = out
        return self._cache

    csd_sum = property(lambda self: self._sums()["csd"])
    psd_sum = property(lambda self: self._sums()["psd"])
    plv_sum = property(lambda self: self._sums()["plv"])
    pli_sum = property(lambda self: self._sums()["pli"])
    abs_im_sum = property(lambda self: self._sums()["abs_im"])
    im_sum = property(lambda self: self.csd_sum.imag)

    def csd_entry(self, i: int, j: int) -> np.ndarray:
        if i == j:
            return self.psd_sum[i].astype(np.complex128)
        if i < j:
            return self.csd_sum[spectral.pair_row_slice(self.n_channels, i)][j - i - 1]
        return np.conj(self.csd_entry(j, i))

    def nbytes(self) -> int:
        e = self._e
        return 0 if e._plan is None else len(e._slot_of) * e._plan.n_tapers * e.n_channels * e.n_bins * 24


def convergence_curve(epochs, metric: MetricId, nfft: int, band: FrequencyBand, n_top: int = 20,
                      max_lag: int | None = None):
    """Stability-of-the-final-network curve over trial count (metrics.py:501-528)."""
    engine = ConnectivityEngine(epochs[0].n_channels, nfft, epochs[0].sfreq, storage_mode=True, max_lag=max_lag,
                                slot_capacity=len(epochs))
    snapshots, counts = [], []
    for k, ep in enumerate(epochs, start=1):
        engine.add_trial(ep)
        if metric is MetricId.XCOR:
            engine._xcor_add([ep])     # the trial itself, as the reference does (not the cache by index)
        try:
            net = engine.finalize(metric, band)
        except DegenerateTrialCountError:
            continue
        w = np.abs(net.weights)
        wmax = w.max()
        snapshots.append(w / wmax if wmax > 0 else w)
        counts.append(k)
    top = np.argsort(-snapshots[-1])[:n_top]
    curve = np.array([s[top].mean() for s in snapshots])
    return np.array(counts), curve
