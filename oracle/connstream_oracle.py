"""numpy restatement of the reference's spectral-connectivity hot path.

TEST INFRASTRUCTURE: the checker for the CUDA path, never shipped or measured as
the product.  Every function follows the reference (``/root/reference/pkg/src/
connstream``) operation-for-operation in complex128/float64 so that, on the same
inputs, it reproduces the reference bit-for-bit (pinned by tests/test_oracle.py).

Reference anchors (paths relative to pkg/src/connstream/):
  * conditioning          spectral.py:49-62   (_crop_pad_demean)
  * per-trial spectra     spectral.py:82-97   (trial_spectra; DC := 0 at :96)
  * pair order            spectral.py:114-122 (pair_index, pair_row_slice)
  * running sums          spectral.py:125-201 (SpectrumSet)
  * per-trial CSD/PSD     spectral.py:204-213 (trial_csd_psd)
  * nonlinear fold        spectral.py:216-241 (_fold_csd; Im flush at :227-228)
  * welch-style averaging spectral.py:264-286 (precedent for the multitaper mean)
  * finalizers            metrics.py:32-98    (*_bins, _SPECTRAL_BINS)
  * band reduction        metrics.py:115-134, core.py:208-215

Documented extensions (conventions item 11), absent from the
reference and applied *outside* its arithmetic:
  * taper: demean over the real samples, multiply by the taper over those samples,
    zero-pad to nfft, rFFT, DC := 0.  Hann = np.hanning(T_eff).
  * multitaper (DPSS): per-trial CSD/PSD = uniform mean over the L tapers, then the
    reference's own nonlinear fold (the welch precedent, spectral.py:272-283).
"""
from __future__ import annotations

import numpy as np

TINY = np.finfo(np.float64).tiny
METRICS = ("COHY", "COH", "IMAGCOHY", "PLV", "PLI", "USPLI", "WPLI", "DSWPLI")


class DegenerateTrialCount(ValueError):
    """Mirror of the reference's DegenerateTrialCountError (core.py:21)."""


# --------------------------------------------------------------------------
# spectra
# --------------------------------------------------------------------------
def crop_pad_demean(data: np.ndarray, nfft: int, taper: np.ndarray | None = None) -> np.ndarray:
    """spectral.py:49-62, plus the taper extension (applied after the demean,
    over the real samples only, before zero padding)."""
    data = np.atleast_2d(np.asarray(data, dtype=np.float64))
    n = data.shape[1]
    if n >= nfft:
        seg = data[:, :nfft]
        out = seg - seg.mean(axis=1, keepdims=True)
        if taper is not None:
            out = out * taper[None, :]
        return out
    out = np.zeros((data.shape[0], nfft))
    dm = data - data.mean(axis=1, keepdims=True)
    if taper is not None:
        dm = dm * taper[None, :]
    out[:, :n] = dm
    return out


def hann(n: int) -> np.ndarray:
    """Conventions item 11: symmetric Hann = np.hanning(n)."""
    return np.hanning(n)


def dpss(n: int, nw: float, k: int) -> np.ndarray:
    """Conventions item 11: scipy.signal.windows.dpss(n, nw, Kmax=k) (L2-normalised)."""
    from scipy.signal import windows
    return np.atleast_2d(windows.dpss(n, nw, Kmax=k))


def trial_spectra(data: np.ndarray, nfft: int, taper: np.ndarray | None = None,
                  method: str = "fft") -> np.ndarray:
    """spectral.py:82-97: one-sided spectra [C, nfft//2+1], DC forced to 0.

    ``method="dft"`` evaluates the same transform as a direct O(n^2) DFT (the
    reference's own test oracle, tests/oracles.py:9-27).  Two fp64 algorithms
    agreeing is the definition of a *well-conditioned* entry: where they differ
    by more than the parity tolerance the reference's value is rounding noise
    (e.g. the Im-flush threshold of spectral.py:227-228 at leakage-level bins).
    """
    seg = crop_pad_demean(data, nfft, taper)
    if method == "fft":
        out = np.fft.rfft(seg, n=nfft, axis=1)
    else:
        nb = nfft // 2 + 1
        m = np.outer(np.arange(nfft), np.arange(nb)) % nfft
        tw = np.exp(-2j * np.pi * m / nfft)
        if nfft % 2 == 0:
            tw[:, -1] = (-1.0) ** np.arange(nfft)
        out = seg @ tw
    out[:, 0] = 0.0
    return out


def pair_index(n: int):
    """spectral.py:114-116."""
    return np.triu_indices(n, k=1)


def pair_row_slice(n: int, i: int) -> slice:
    """spectral.py:119-122."""
    off = i * (n - 1) - i * (i - 1) // 2
    return slice(off, off + n - 1 - i)


# --------------------------------------------------------------------------
# accumulation (SpectrumSet restated over band columns)
# --------------------------------------------------------------------------
class Sums:
    """spectral.py:125-201 restricted to the accumulated columns."""

    def __init__(self, n_channels: int, n_cols: int):
        P = n_channels * (n_channels - 1) // 2
        self.n_channels = n_channels
        self.csd_sum = np.zeros((P, n_cols), dtype=np.complex128)
        self.psd_sum = np.zeros((n_channels, n_cols))
        self.plv_sum = np.zeros((P, n_cols), dtype=np.complex128)
        self.pli_sum = np.zeros((P, n_cols))
        self.abs_im_sum = np.zeros((P, n_cols))
        self.n_trials_accumulated = 0

    @property
    def im_sum(self):
        return self.csd_sum.imag


def trial_csd_psd(spectra: np.ndarray, n_channels: int):
    """spectral.py:204-213."""
    psd = np.abs(spectra) ** 2
    csd = np.empty((n_channels * (n_channels - 1) // 2, spectra.shape[1]), dtype=np.complex128)
    conj = np.conj(spectra)
    for i in range(n_channels - 1):
        csd[pair_row_slice(n_channels, i)] = spectra[i][None, :] * conj[i + 1:]
    return csd, psd


def fold_csd(acc: Sums, csd: np.ndarray, psd: np.ndarray, bins=None, count: bool = True) -> None:
    """spectral.py:216-241: ``bins`` selects the accumulator columns csd / psd cover (None =
    all); ``count=False`` back-fills columns of trials already counted."""
    im = csd.imag
    im[np.abs(im) <= 1e-13 * np.abs(csd.real)] = 0.0
    mag = np.abs(csd)
    nz = mag > TINY
    unit = np.zeros_like(csd)
    np.divide(csd, mag, out=unit, where=nz)
    sl = slice(None) if bins is None else bins
    acc.psd_sum[:, sl] += psd
    acc.csd_sum[:, sl] += csd
    acc.plv_sum[:, sl] += unit
    acc.pli_sum[:, sl] += np.sign(im)
    acc.abs_im_sum[:, sl] += np.abs(im)
    if count:
        acc.n_trials_accumulated += 1


def accumulate(acc: Sums, spectra_cols: np.ndarray, bins=None, count: bool = True) -> None:
    """spectral.py:244-261: spectra over all of acc's columns, folded into ``bins`` (None =
    all) -- or, with bins None, spectra already restricted to acc's columns."""
    sub = spectra_cols if bins is None else spectra_cols[:, bins]
    csd, psd = trial_csd_psd(sub, acc.n_channels)
    fold_csd(acc, csd, psd, bins=bins, count=count)


def accumulate_multitaper(acc: Sums, spectra_l: np.ndarray) -> None:
    """Multitaper extension: spectra_l [L, C, ncols]; CSD/PSD = mean over tapers,
    then the reference fold (welch precedent, spectral.py:272-283)."""
    L = spectra_l.shape[0]
    csd = np.zeros((acc.csd_sum.shape[0], spectra_l.shape[2]), dtype=np.complex128)
    psd = np.zeros((acc.n_channels, spectra_l.shape[2]))
    for spec in spectra_l:
        c, p = trial_csd_psd(spec, acc.n_channels)
        csd += c
        psd += p
    fold_csd(acc, csd / L, psd / L)


# --------------------------------------------------------------------------
# finalizers (metrics.py:32-98) over all accumulated columns
# --------------------------------------------------------------------------
def _need(acc: Sums, k: int = 1):
    if acc.n_trials_accumulated < k:
        raise DegenerateTrialCount("no trials accumulated" if k == 1 else "USPLI needs at least 2 trials")


def cohy_bins(acc: Sums) -> np.ndarray:
    _need(acc)
    pi, pj = pair_index(acc.n_channels)
    denom = np.sqrt(acc.psd_sum[pi] * acc.psd_sum[pj])
    out = np.zeros_like(acc.csd_sum)
    np.divide(acc.csd_sum, denom, out=out, where=denom > TINY)
    return out


def coh_bins(acc):
    return np.abs(cohy_bins(acc))


def imagcohy_bins(acc):
    return cohy_bins(acc).imag


def plv_bins(acc):
    _need(acc)
    return np.abs(acc.plv_sum) / acc.n_trials_accumulated


def pli_bins(acc):
    _need(acc)
    return np.abs(acc.pli_sum) / acc.n_trials_accumulated


def uspli_bins(acc):
    K = acc.n_trials_accumulated
    _need(acc, 2)
    pli = pli_bins(acc)
    return (K * pli ** 2 - 1.0) / (K - 1.0)


def wpli_bins(acc):
    _need(acc)
    num = np.abs(acc.im_sum)
    den = acc.abs_im_sum
    out = np.zeros_like(num)
    np.divide(num, den, out=out, where=den > 0.0)
    return out


def dswpli_bins(acc):
    return wpli_bins(acc) ** 2


BINS = {"COHY": cohy_bins, "COH": coh_bins, "IMAGCOHY": imagcohy_bins, "PLV": plv_bins,
        "PLI": pli_bins, "USPLI": uspli_bins, "WPLI": wpli_bins, "DSWPLI": dswpli_bins}


def band_reduce(metric: str, per_bin: np.ndarray):
    """metrics.py:124-134 / core.py:208-215: arithmetic mean over the band; COHY
    keeps the complex mean and reports |mean| as the weight."""
    if metric == "COHY":
        cmean = per_bin.mean(axis=1)
        return np.abs(cmean), cmean
    return per_bin.mean(axis=1), None


# --------------------------------------------------------------------------
# whole-path driver
# --------------------------------------------------------------------------
def segments(ep: np.ndarray, nfft: int) -> list:
    """Welch mode (spectral.py:100-111): consecutive non-overlapping nfft segments."""
    n_seg = max(1, ep.shape[1] // nfft)
    return [ep[:, s * nfft:(s + 1) * nfft] for s in range(n_seg)]


def compute(epochs, nfft: int, lo: int, hi: int, metrics=METRICS, taper=None, method: str = "fft",
            mode: str = "fixed"):
    """All requested metrics for trials ``epochs`` (list/array of [C, T]) over the
    inclusive bin range [lo, hi].

    ``taper``: None (reference rectangular), a 1-D taper, or a 2-D [L, T_eff]
    DPSS stack (multitaper extension).  ``mode="welch"``: trials with
    T >= 2 nfft fold the segment-mean CSD / PSD (spectral.py:264-283).
    Returns {metric: {"bins": [P, nb], "band": [P], "cband": complex [P] | None}}.
    """
    epochs = [np.asarray(e, dtype=np.float64) for e in epochs]
    C = epochs[0].shape[0]
    acc = Sums(C, hi - lo + 1)
    for ep in epochs:
        if mode == "welch" and ep.shape[1] >= 2 * nfft:
            spec_l = np.stack([trial_spectra(sg, nfft, None, method)[:, lo:hi + 1] for sg in segments(ep, nfft)])
            accumulate_multitaper(acc, spec_l)
        elif taper is not None and np.ndim(taper) == 2:
            spec_l = np.stack([trial_spectra(ep, nfft, tp, method)[:, lo:hi + 1] for tp in taper])
            accumulate_multitaper(acc, spec_l)
        else:
            accumulate(acc, trial_spectra(ep, nfft, taper, method)[:, lo:hi + 1])
    out = {}
    for m in metrics:
        try:
            pb = BINS[m](acc)
        except DegenerateTrialCount:
            out[m] = None
            continue
        w, cw = band_reduce(m, pb)
        out[m] = {"bins": pb, "band": w, "cband": cw}
    return out, acc


def well_conditioned(epochs, nfft, lo, hi, metrics, tol, taper=None, ref=None, mode="fixed"):
    """Per-metric boolean masks [P, nb] of entries on which two independent fp64
    spectral algorithms (rfft vs direct DFT) agree within tol[m]/2."""
    a = ref if ref is not None else compute(epochs, nfft, lo, hi, metrics, taper, mode=mode)[0]
    b = compute(epochs, nfft, lo, hi, metrics, taper, method="dft", mode=mode)[0]
    out = {}
    for m in metrics:
        if a.get(m) is None:
            continue
        out[m] = np.abs(a[m]["bins"] - b[m]["bins"]) <= 0.5 * tol[m]
    return out


def flush_sensitive(epochs, nfft, lo, hi, taper=None, lo_ratio=1e-15, hi_ratio=1e-11, mode="fixed"):
    """Boolean [P, nb]: (pair, bin) entries where some trial has
    |Im CSD| / |Re CSD| within two decades of the reference's 1e-13 flush
    threshold (spectral.py:227-228).  There the reference's sign(Im) is decided
    by last-ulp rounding of its own spectra, so no other arithmetic (a different
    FFT, summation order or taper placement) can reproduce it."""
    epochs = [np.asarray(e, dtype=np.float64) for e in epochs]
    C = epochs[0].shape[0]
    out = np.zeros((C * (C - 1) // 2, hi - lo + 1), dtype=bool)
    for ep in epochs:
        if mode == "welch" and ep.shape[1] >= 2 * nfft:
            csd = 0
            for sg in segments(ep, nfft):
                c, _ = trial_csd_psd(trial_spectra(sg, nfft, None)[:, lo:hi + 1], C)
                csd = csd + c
        elif taper is not None and np.ndim(taper) == 2:
            csd = 0
            for tp in taper:
                c, _ = trial_csd_psd(trial_spectra(ep, nfft, tp)[:, lo:hi + 1], C)
                csd = csd + c
        else:
            csd, _ = trial_csd_psd(trial_spectra(ep, nfft, taper)[:, lo:hi + 1], C)
        r = np.abs(csd.imag) / np.maximum(np.abs(csd.real), TINY)
        out |= (r >= lo_ratio) & (r <= hi_ratio)
    return out


# --------------------------------------------------------------------------
# time-domain metrics (metrics.py:140-260), restated
# --------------------------------------------------------------------------
def epoch_cor(data: np.ndarray):
    """Clipped upper-triangle Pearson matrix of one epoch and its zero-variance
    channels (metrics.py:140-155)."""
    d = data - data.mean(axis=1, keepdims=True)
    norms = np.sqrt(np.sum(d * d, axis=1))
    dead = np.flatnonzero(norms == 0.0)
    u = d / np.where(norms == 0.0, 1.0, norms)[:, None]
    full = u @ u.T
    full[dead, :] = 0.0
    full[:, dead] = 0.0
    pi, pj = pair_index(data.shape[0])
    return np.clip(full[pi, pj], -1.0, 1.0), list(dead)


def cor(epochs):
    """Mean Pearson correlation per pair (metrics.py:158-177): (weights, dead channels)."""
    tot, dead = 0.0, set()
    for ep in epochs:
        w, d = epoch_cor(np.asarray(ep, dtype=np.float64))
        tot = tot + w
        dead.update(d)
    return tot / len(epochs), sorted(dead)


def xcor_pair(x: np.ndarray, y: np.ndarray, max_lag: int):
    """Peak (value, lag) of the overlap-normalised cross-correlation by direct
    sliding sums (the reference's method="direct" checker, metrics.py:180-226)."""
    n = len(x)
    dx, dy = x - x.mean(), y - y.mean()
    ey = float(np.sum(dy * dy))
    if ey == 0.0 or not np.any(dx):
        return 0.0, 0
    best, best_lag = None, 0
    for tau in range(-max_lag, max_lag + 1):
        a, b = (dx[tau:], dy[:n - tau]) if tau >= 0 else (dx[:n + tau], dy[-tau:])
        den = np.sqrt(np.sum(a * a) * ey)
        v = np.sum(a * b) / den if den > 0.0 else 0.0
        if best is None or v > best:
            best, best_lag = v, tau
    return float(best), int(best_lag)


def xcor(epochs, max_lag=None):
    """|mean peak| and rounded mean lag per pair (metrics.py:229-260)."""
    C, n = np.asarray(epochs[0]).shape
    max_lag = n - 1 if max_lag is None else max_lag
    pi, pj = pair_index(C)
    pk, lg = np.zeros(len(pi)), np.zeros(len(pi))
    for ep in epochs:
        ep = np.asarray(ep, dtype=np.float64)
        for k in range(len(pi)):
            v, l = xcor_pair(ep[pi[k]], ep[pj[k]], max_lag)
            pk[k] += v
            lg[k] += l
    K = len(epochs)
    return np.abs(pk / K), np.rint(lg / K).astype(np.int64)
