"""Drop-in for connstream.spectral (reference src/spectral.py) on the B200 path.

Same names, arguments and errors; the arithmetic runs in libcsconn.so:
  * trial_spectra / fft_real      -> K1 (cs_spectra), fp64 demean + taper + DFT
  * SpectrumSet                    -> a device accumulator: the folded trials'
    spectra live in an HBM slot ring; metric finalisers run the fused pair
    kernels over those slots (the reference's running sums are materialised
    only when an attribute such as ``csd_sum`` is read).
  * accumulate_spectra / accumulate_epoch keep the bins/count semantics of
    spectral.py:244-286, fixed and welch mode (segments on the ring's taper
    axis, a welch trial stored with weight 1/sqrt(S) so its summed CSD is the
    segment mean of spectral.py:272-283).

Reference anchors: spectral.py:18-30 (FFT counter), :49-97 (spectra),
:114-122 (pair order), :125-201 (SpectrumSet), :204-286 (fold).
"""
from __future__ import annotations

import os

import numpy as np
import torch

from .core import EpochMatrix, ParameterError
from .plan import DevicePlan, pow2_scale

_FFT_CALLS = 0


def fft_call_count() -> int:
    return _FFT_CALLS


def reset_fft_call_count() -> None:
    global _FFT_CALLS
    _FFT_CALLS = 0


def _count_ffts(n: int) -> None:
    global _FFT_CALLS
    _FFT_CALLS += int(n)


def n_bins_for(nfft: int) -> int:
    return nfft // 2 + 1


def worker_count() -> int:
    """CONNSTREAM_THREADS-capped pool size (spectral.py:37-46); kept for callers
    that size host pools -- the device path does not use host threads."""
    n = os.cpu_count() or 1
    cap = os.environ.get("CONNSTREAM_THREADS")
    if cap:
        try:
            n = min(n, max(1, int(cap)))
        except ValueError:
            pass
    return n


def _device():
    if not torch.cuda.is_available():
        raise RuntimeError("paper_2303_03279_b200 needs a CUDA device; there is no CPU fallback")
    return torch.device("cuda", torch.cuda.current_device())


def _as_device_samples(data) -> torch.Tensor:
    if isinstance(data, torch.Tensor):
        t = data
        if t.dtype not in (torch.float32, torch.float64):
            t = t.double()
        return t.to(_device())
    return torch.as_tensor(np.asarray(data, dtype=np.float64), device=_device())


_SPEC_PLANS: dict = {}


def _spectra_plan(C: int, T: int, nfft: int, taper) -> DevicePlan:
    key = (C, T, nfft, None if taper is None else (taper if isinstance(taper, str) else id(taper)))
    plan = _SPEC_PLANS.get(key)
    if plan is None:
        if len(_SPEC_PLANS) > 16:
            _SPEC_PLANS.clear()
        plan = DevicePlan(C, T, nfft, 0, nfft // 2, taper=taper, slot_capacity=1, device=_device())
        _SPEC_PLANS[key] = plan
    return plan


def device_trial_spectra(data, nfft: int, taper=None) -> torch.Tensor:
    """complex128 [C, nfft//2+1] on the device (K1 over all bins)."""
    x = _as_device_samples(data)
    if x.dim() == 1:
        x = x[None]
    C, T = x.shape
    plan = _spectra_plan(C, T, nfft, taper)
    plan.spectra(x[None].contiguous(), 0)
    _count_ffts(C)
    return plan.get_spectra(torch.zeros(1, dtype=torch.int32, device=plan.device))[0]


def fft_real(signal, nfft: int, taper=None) -> np.ndarray:
    """One-sided DFT of a real signal after mean removal (spectral.py:65-79)."""
    if nfft < 2:
        raise ParameterError(f"nfft must be >= 2, got {nfft}")
    sig = np.asarray(signal, dtype=np.float64).reshape(-1)
    if sig.size < 1:
        raise ParameterError("empty signal")
    return device_trial_spectra(sig[None], nfft, taper)[0].cpu().numpy()


def trial_spectra(epoch: EpochMatrix, nfft: int, mode: str = "fixed", taper=None) -> np.ndarray:
    """Per-channel one-sided spectra, rows = channels (spectral.py:82-97).  As in
    the reference, ``mode`` is validated and the fixed-resolution spectra are
    returned for both modes (the welch average lives in accumulate_epoch)."""
    if nfft < 2:
        raise ParameterError(f"nfft must be >= 2, got {nfft}")
    if mode not in ("fixed", "welch"):
        raise ParameterError(f"unknown spectral mode {mode!r}")
    return device_trial_spectra(epoch.data, nfft, taper).cpu().numpy()


def device_segment_spectra(data, nfft: int) -> torch.Tensor:
    """complex128 [S, C, nfft//2+1] on the device: K1 over the S = max(1, T // nfft)
    consecutive non-overlapping nfft segments, each demeaned (spectral.py:100-111)."""
    x = _as_device_samples(data)
    if x.dim() == 1:
        x = x[None]
    C, T = x.shape
    S = max(1, T // nfft)
    if T < nfft:
        return device_trial_spectra(x, nfft)[None]
    x = x.contiguous()
    segs = x.as_strided((S, C, nfft), (nfft, T, 1))       # segment s = samples [s nfft, (s+1) nfft)
    key = ("seg", C, nfft, S)
    plan = _SPEC_PLANS.get(key)
    if plan is None:
        if len(_SPEC_PLANS) > 16:
            _SPEC_PLANS.clear()
        plan = DevicePlan(C, nfft, nfft, 0, nfft // 2, slot_capacity=S, device=_device())
        _SPEC_PLANS[key] = plan
    plan.spectra(segs, 0)
    _count_ffts(S * C)
    return plan.get_spectra(torch.arange(S, dtype=torch.int32, device=plan.device))


def segment_spectra(epoch: EpochMatrix, nfft: int) -> list:
    """Spectra of consecutive non-overlapping nfft segments ("welch" mode, spectral.py:100-111)."""
    if nfft < 2:
        raise ParameterError(f"nfft must be >= 2, got {nfft}")
    return list(device_segment_spectra(epoch.data, nfft).cpu().numpy())


def pair_index(n_channels: int):
    """Upper-triangle (i < j) channel pairs in row-major order (spectral.py:114-116)."""
    return np.triu_indices(n_channels, k=1)


def pair_row_slice(n_channels: int, i: int) -> slice:
    """Slice of the pair axis holding pairs (i, i+1) .. (i, n-1) (spectral.py:119-122)."""
    off = i * (n_channels - 1) - i * (i - 1) // 2
    return slice(off, off + n_channels - 1 - i)


def trial_csd_psd(spectra, n_channels: int):
    """Upper-triangle CSD [P, B] and PSD [C, B] of one trial's spectra
    (spectral.py:204-213; no Im flush -- that belongs to the fold).  Computed on
    the device; returns numpy arrays like the reference."""
    x = torch.as_tensor(spectra, dtype=torch.complex128, device=_device())
    if x.dim() != 2 or x.shape[0] != n_channels:
        raise ParameterError(f"spectra must be [{n_channels}, bins], got {tuple(x.shape)}")
    i, j = (torch.as_tensor(a, device=x.device) for a in pair_index(n_channels))
    csd = x[i] * x[j].conj()
    psd = x.abs() ** 2
    return csd.cpu().numpy(), psd.cpu().numpy()


class SpectrumSet:
    """Device accumulator with the reference's SpectrumSet interface.

    The folded trials' full-bin spectra are held in an HBM slot ring together
    with the column mask each fold covered (``bins``) and whether it counted
    (``count``).  Metric finalisers (metrics.py) run the fused pair kernels over
    the slots; the reference's [P, B] running sums are built on first access.
    """

    def __init__(self, n_channels: int, nfft: int):
        if nfft < 2:
            raise ParameterError("nfft must be >= 2")
        if n_channels < 1:
            raise ParameterError("need at least one channel")
        self.n_channels = int(n_channels)
        self.nfft = int(nfft)
        self.n_trials_accumulated = 0
        self._entries: list[tuple[int, np.ndarray]] = []   # (slot, column mask)
        self._plan: DevicePlan | None = None
        self._next_slot = 0
        self._sums_cache = None

    # -- shape -------------------------------------------------------------
    @property
    def n_bins(self) -> int:
        return n_bins_for(self.nfft)

    @property
    def n_pairs(self) -> int:
        return self.n_channels * (self.n_channels - 1) // 2

    # -- storage -------------------------------------------------------------
    def _ensure_capacity(self, extra: int, scale: float = 1.0, n_tapers: int = 1) -> None:
        """Room for ``extra`` more slots with at least ``n_tapers`` taper (welch
        segment) entries per slot; grows by re-planning and copying the ring."""
        need = self._next_slot + extra
        L_old = self._plan.n_tapers if self._plan is not None else 1
        L = max(L_old, int(n_tapers))
        if self._plan is not None and need <= self._plan.slot_capacity and L == L_old:
            return
        cap = max(8, 1 << max(need - 1, 1).bit_length())
        if self._plan is not None:
            cap = max(cap, self._plan.slot_capacity)
        new = DevicePlan(self.n_channels, self.nfft, self.nfft, 0, self.n_bins - 1, slot_capacity=cap,
                         device=_device(), scale=self._plan.scale if self._plan is not None else scale,
                         n_tapers=L)
        if self._plan is not None and self._next_slot:
            o64, o32 = self._plan.ring()
            n64, n32 = new.ring()
            n64[: self._next_slot, :L_old].copy_(o64[: self._next_slot])
            n32[: self._next_slot, :L_old].copy_(o32[: self._next_slot])
        self._plan = new

    def _first_scale(self, spectra: torch.Tensor) -> float:
        amax = float(spectra.abs().amax()) if spectra.numel() else 0.0
        return pow2_scale(amax / max(self.nfft, 1) ** 0.5, self.nfft) if amax > 0 else 1.0

    def _fold(self, spectra: torch.Tensor, cols: np.ndarray, count: bool) -> None:
        """spectra: complex128 device [C, n_bins] (zeros outside ``cols``)."""
        self._fold_segments(spectra[None], cols, count)

    def _fold_segments(self, segs: torch.Tensor, cols: np.ndarray, count: bool) -> None:
        """segs: complex128 device [S, C, n_bins]; S > 1 is a welch trial whose CSD /
        PSD contribution is the mean over segments (spectral.py:272-283): each
        segment is stored with weight 1/sqrt(S) on the slot's taper axis."""
        S = int(segs.shape[0])
        if self._plan is None:
            self._ensure_capacity(1, self._first_scale(segs), n_tapers=S)
        else:
            self._ensure_capacity(1, n_tapers=S)
        slot = self._next_slot
        w = 1.0 / float(np.sqrt(S))
        for l in range(S):
            self._plan.put_spectra(segs[l:l + 1], slot, taper=l, weight=w if S > 1 else 1.0)
        self._next_slot += 1
        self._entries.append((slot, cols.copy()))
        if count:
            self.n_trials_accumulated += 1
        self._sums_cache = None

    def slots_for(self, lo: int, hi: int):
        """Slots whose folds cover every column of [lo, hi] (or None if the
        column sets differ inside the band)."""
        sel = [s for s, m in self._entries if m[lo:hi + 1].all()]
        part = [s for s, m in self._entries if m[lo:hi + 1].any() and not m[lo:hi + 1].all()]
        return None if part else sel

    @property
    def plan(self) -> DevicePlan | None:
        return self._plan

    # -- reference attributes (materialised on access) ----------------------
    def _sums(self):
        if self._sums_cache is None:
            self._sums_cache = _materialise_sums(self)
        return self._sums_cache

    @property
    def csd_sum(self):
        return self._sums()["csd"]

    @property
    def psd_sum(self):
        return self._sums()["psd"]

    @property
    def plv_sum(self):
        return self._sums()["plv"]

    @property
    def pli_sum(self):
        return self._sums()["pli"]

    @property
    def abs_im_sum(self):
        return self._sums()["abs_im"]

    @property
    def im_sum(self):
        return self.csd_sum.imag

    def csd_entry(self, i: int, j: int) -> np.ndarray:
        if i == j:
            return self.psd_sum[i].astype(np.complex128)
        if i < j:
            return self.csd_sum[pair_row_slice(self.n_channels, i)][j - i - 1]
        return np.conj(self.csd_entry(j, i))

    def nbytes(self) -> int:
        if self._plan is None:
            return 0
        return self._next_slot * self._plan.n_tapers * self.n_channels * self.n_bins * (16 + 8)

    def copy(self) -> "SpectrumSet":
        out = SpectrumSet(self.n_channels, self.nfft)
        out.merge(self)
        out.n_trials_accumulated = self.n_trials_accumulated
        return out

    def merge(self, other: "SpectrumSet") -> None:
        """Fold another partial accumulation into this one (associative)."""
        if (other.n_channels, other.nfft) != (self.n_channels, self.nfft):
            raise ParameterError("cannot merge accumulators of different shape")
        if other._plan is not None and other._entries:
            o64, _ = other._plan.ring()                       # [S, L, nb, N] complex128
            Lo = other._plan.n_tapers
            for s_o, m in other._entries:
                if self._plan is None:
                    self._ensure_capacity(len(other._entries), other._plan.scale, n_tapers=Lo)
                self._ensure_capacity(1, n_tapers=Lo)
                for l in range(Lo):   # stored values already carry their weights
                    self._plan.put_spectra(o64[s_o, l].transpose(0, 1)[None], self._next_slot, taper=l)
                self._entries.append((self._next_slot, m.copy()))
                self._next_slot += 1
        self.n_trials_accumulated += other.n_trials_accumulated
        self._sums_cache = None


def _materialise_sums(acc: SpectrumSet) -> dict:
    """The reference's running sums (spectral.py:136-141, fold of :216-241) from
    the cached spectra by cs_pair_sums (fp64, reference arithmetic) -- an accessor
    for callers that read the sums directly; the finalisers never use it.  Folds
    that covered only some columns stored zeros elsewhere, which contribute 0 to
    every sum (CSD 0, no phasor, sign(0) = 0)."""
    C, B = acc.n_channels, acc.n_bins
    P = acc.n_pairs
    out = {"csd": np.zeros((P, B), np.complex128), "psd": np.zeros((C, B)), "plv": np.zeros((P, B), np.complex128),
           "pli": np.zeros((P, B)), "abs_im": np.zeros((P, B))}
    if not acc._entries:
        return out
    slots = torch.tensor([s for s, _ in acc._entries], dtype=torch.int32, device=acc._plan.device)
    o = acc._plan.pair_sums(slots)
    out["csd"] = o["csd"].T.cpu().numpy().copy()
    out["plv"] = o["plv"].T.cpu().numpy().copy()
    out["pli"] = o["pli"].T.to(torch.float64).cpu().numpy().copy()
    out["abs_im"] = o["abs_im"].T.cpu().numpy().copy()
    out["psd"] = o["psd"].T.cpu().numpy().copy()
    return out


def _cols_mask(n_bins: int, bins) -> np.ndarray:
    m = np.zeros(n_bins, dtype=bool)
    if bins is None:
        m[:] = True
    else:
        m[np.arange(n_bins)[bins]] = True
    return m


def accumulate_spectra(acc: SpectrumSet, spectra, bins=None, count: bool = True) -> SpectrumSet:
    """Fold one trial's spectra into the accumulator (spectral.py:244-261)."""
    if isinstance(spectra, torch.Tensor):
        shape = tuple(spectra.shape)
    else:
        spectra = np.asarray(spectra)
        shape = spectra.shape
    if shape != (acc.n_channels, acc.n_bins):
        raise ParameterError(f"spectra shape {shape} does not match accumulator ({acc.n_channels}, {acc.n_bins})")
    cols = _cols_mask(acc.n_bins, bins)
    spec = torch.as_tensor(spectra, dtype=torch.complex128, device=_device())
    if not cols.all():
        spec = spec * torch.as_tensor(cols, device=spec.device)[None, :]
    acc._fold(spec, cols, count)
    return acc


def accumulate_epoch(acc: SpectrumSet, epoch: EpochMatrix, mode: str = "fixed", bins=None, taper=None):
    """Compute and accumulate one trial; returns the spectra (spectral.py:264-286).
    Welch mode with n_samples >= 2 nfft folds the segment-mean CSD / PSD and
    returns the first segment's spectra, as the reference does."""
    if mode not in ("fixed", "welch"):
        raise ParameterError(f"unknown spectral mode {mode!r}")
    cols = _cols_mask(acc.n_bins, bins)
    cmask = None if cols.all() else torch.as_tensor(cols)
    if mode == "welch" and epoch.n_samples >= 2 * acc.nfft:
        if taper is not None:
            raise ParameterError("welch mode takes no taper")
        segs = device_segment_spectra(epoch.data, acc.nfft)          # [S, C, B]
        acc._fold_segments(segs if cmask is None else segs * cmask.to(segs.device)[None, None, :], cols, True)
        return segs[0].cpu().numpy()
    spec = device_trial_spectra(epoch.data, acc.nfft, taper)
    acc._fold(spec if cmask is None else spec * cmask.to(spec.device)[None, :], cols, True)
    return spec.cpu().numpy()
