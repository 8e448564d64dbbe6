"""Time-domain metrics COR and XCOR on the device (reference metrics.py:137-260).

Both run in the hand-written kernels of csrc/timedomain.cu on the fp64 tensor
cores (DMMA): COR as the Gram product of the demeaned unit-norm channels with the
clip fused in (``cs_cor_sums``), XCOR as per-lag "shifted Gram" products of the
demeaned channels with the overlap normalisation and the first-maximum argmax
fused in (``cs_xcor_sums``), every trial of a call in one launch.  Both keep the
reference's edge cases: zero-variance channels give zero-weight COR edges and a
warning; an XCOR pair with a constant x or y gives (0, lag 0).
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


def _groups(epochs_data, C: int):
    """Device fp64 stacks [k, C, T] of consecutive epochs sharing n_samples (the
    reference allows epochs of different lengths; each stack is one launch)."""
    out, cur = [], []
    for data in epochs_data:
        x = _dev_f64(data)
        if x.dim() != 2 or x.shape[0] != C:
            raise ParameterError("epochs must have equal channel counts")
        if cur and x.shape[1] != cur[0].shape[1]:
            out.append(torch.stack(cur))
            cur = []
        cur.append(x)
        if len(cur) == 65535:
            out.append(torch.stack(cur))
            cur = []
    if cur:
        out.append(torch.stack(cur))
    return out


def cor_sums(epochs_data, n_channels: int):
    """(sum over epochs of the clipped Pearson upper triangle [P] fp64 device,
    sorted zero-variance channels) -- metrics.py:140-177."""
    C = int(n_channels)
    P = C * (C - 1) // 2
    total = None
    dead = set()
    for xs in _groups(epochs_data, C):
        K, _, T = xs.shape
        if total is None:
            total = torch.zeros(P, dtype=torch.float64, device=xs.device)
        if P == 0:  # one channel: no pairs, only the zero-variance warning
            flags = (xs == xs[..., :1]).all(dim=-1)
        else:
            flags = torch.zeros((K, C), dtype=torch.uint8, device=xs.device)
            _lib.check(_lib.lib().cs_cor_sums(ctypes.c_void_p(xs.data_ptr()), K, C, T,
                                              ctypes.c_void_p(total.data_ptr()), ctypes.c_void_p(flags.data_ptr()),
                                              _sp()))
        dead.update(torch.nonzero(flags.any(dim=0)).flatten().tolist())
    return total, sorted(dead)


def xcor_sums(epochs_data, n_channels: int, max_lag: int):
    """(sum of per-epoch peak values [P], sum of peak lags [P]), fp64 device --
    metrics.py:180-260 (peak of the overlap-normalised cross-correlation,
    negative lag = x leads y)."""
    C = int(n_channels)
    P = C * (C - 1) // 2
    peak = lag = None
    for xs in _groups(epochs_data, C):
        K, _, T = xs.shape
        if max_lag >= T:
            raise ParameterError("max_lag must be < n_samples")
        if peak is None:
            peak = torch.zeros(P, dtype=torch.float64, device=xs.device)
            lag = torch.zeros(P, dtype=torch.float64, device=xs.device)
        if P == 0:
            continue
        _lib.check(_lib.lib().cs_xcor_sums(ctypes.c_void_p(xs.data_ptr()), K, C, T, int(max_lag),
                                           ctypes.c_void_p(peak.data_ptr()), ctypes.c_void_p(lag.data_ptr()), None,
                                           _sp()))
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
