"""Time-domain metrics COR and XCOR on the device (reference metrics.py:137-260).

COR: per trial the Pearson matrix of the demeaned, normalised channels is one
Gram product (cuBLAS DGEMM, fp64 like the reference); the clipped upper
triangle is accumulated by ``cs_cor_accumulate``.  XCOR: per trial one real FFT
per channel (cuFFT, fp64), an inverse FFT per pair of X_i conj X_j gives every
lag's numerator at once, and ``cs_xcor_peaks`` normalises by the overlap
energies and takes the first maximum over [-max_lag, max_lag] (one warp per
pair).  Both keep the reference's edge cases: zero-variance channels give
zero-weight COR edges and a warning; an XCOR pair with a constant x or y gives
(0, lag 0).
"""
from __future__ import annotations

import ctypes

import numpy as np
import torch

from . import _lib
from .core import ParameterError


def _sp():
    return ctypes.c_void_p(torch.cuda.current_stream().cuda_stream)


def _dev_f64(data) -> torch.Tensor:
    from .spectral import _device
    t = data if isinstance(data, torch.Tensor) else torch.as_tensor(np.asarray(data, dtype=np.float64))
    return t.to(device=_device(), dtype=torch.float64)


def cor_sums(epochs_data, n_channels: int):
    """(sum over epochs of the clipped Pearson upper triangle [P] fp64 device,
    sorted zero-variance channels) -- metrics.py:140-177."""
    C = int(n_channels)
    P = C * (C - 1) // 2
    total = None
    dead = set()
    for data in epochs_data:
        x = _dev_f64(data)
        if x.shape[0] != C:
            raise ParameterError("epochs must have equal channel counts")
        if total is None:
            total = torch.zeros(P, dtype=torch.float64, device=x.device)
        d = x - x.mean(dim=1, keepdim=True)
        norms = torch.sqrt((d * d).sum(dim=1))
        z = norms == 0.0
        if bool(z.any()):
            dead.update(torch.nonzero(z).flatten().tolist())
        u = d / torch.where(z, torch.ones_like(norms), norms)[:, None]
        G = (u @ u.T).contiguous()                       # cuBLAS DGEMM
        if P:
            _lib.check(_lib.lib().cs_cor_accumulate(ctypes.c_void_p(G.data_ptr()), C, 0, P,
                                                    ctypes.c_void_p(total.data_ptr()), _sp()))
    return total, sorted(dead)


def xcor_sums(epochs_data, n_channels: int, max_lag: int, pair_chunk: int | None = None):
    """(sum of per-epoch peak values [P], sum of peak lags [P], n_epochs), fp64
    device -- metrics.py:180-260 (peak of the overlap-normalised
    cross-correlation, negative lag = x leads y)."""
    C = int(n_channels)
    P = C * (C - 1) // 2
    peak = lag = None
    pi = pj = None
    for data in epochs_data:
        x = _dev_f64(data)
        n = x.shape[1]
        if max_lag >= n:
            raise ParameterError("max_lag must be < n_samples")
        if peak is None:
            peak = torch.zeros(P, dtype=torch.float64, device=x.device)
            lag = torch.zeros(P, dtype=torch.float64, device=x.device)
            a, b = np.triu_indices(C, 1)
            pi = torch.as_tensor(a, dtype=torch.int64, device=x.device)
            pj = torch.as_tensor(b, dtype=torch.int64, device=x.device)
        nfft = 1 << max(1, (2 * n - 1 - 1).bit_length())      # >= 2 n - 1: no circular wrap
        d = x - x.mean(dim=1, keepdim=True)
        xz = (d == 0).all(dim=1).to(torch.uint8).contiguous()
        csq = torch.cat([torch.zeros((C, 1), dtype=torch.float64, device=x.device), torch.cumsum(d * d, 1)], 1)
        csq = csq.contiguous()
        X = torch.fft.rfft(d, n=nfft, dim=1)                  # cuFFT, fp64
        chunk = pair_chunk or max(1, min(P, (1 << 28) // (8 * nfft)))
        for p0 in range(0, P, chunk):
            a, b = pi[p0:p0 + chunk], pj[p0:p0 + chunk]
            cc = torch.fft.irfft(X[a] * torch.conj(X[b]), n=nfft, dim=1).contiguous()
            _lib.check(_lib.lib().cs_xcor_peaks(
                ctypes.c_void_p(cc.data_ptr()), int(a.numel()), nfft, n, int(max_lag),
                ctypes.c_void_p(a.data_ptr()), ctypes.c_void_p(b.data_ptr()), ctypes.c_void_p(csq.data_ptr()),
                ctypes.c_void_p(xz.data_ptr()), ctypes.c_void_p(peak[p0:].data_ptr()),
                ctypes.c_void_p(lag[p0:].data_ptr()), _sp()))
    return peak, lag


def xcor_pair(x, y, max_lag: int, method: str = "fft"):
    """Peak of the normalised cross-correlation of one pair (metrics.py:180-226);
    the device path for both ``method`` values (the reference's "direct" is its
    O(n^2) checker)."""
    if method not in ("fft", "direct"):
        raise ParameterError(f"unknown xcor method {method!r}")
    x = np.asarray(x, dtype=np.float64)
    y = np.asarray(y, dtype=np.float64)
    if max_lag >= len(x):
        raise ParameterError("max_lag must be < n_samples")
    pk, lg = xcor_sums([np.vstack([x, y])], 2, max_lag)
    return float(pk[0]), int(round(float(lg[0])))
