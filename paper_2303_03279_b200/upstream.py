"""Upstream of the spectra: source projection and FIR filtering,
on the hand-written kernels of csrc/upstream.cu (fp64).

* Inverse projection (reference inverse.py:147-154: source data = M @ sensor
  data, then the spectral path on the sources).  Demean, taper and the DFT are
  linear per channel, so the source spectra equal M times the sensor spectra:
  ``source_connectivity`` runs K1 on the C sensors and projects the HBM spectrum
  ring ([K L nb] complex rows x C sensors -> N_src sources; ``cs_project_ring``, a
  DMMA GEMM whose epilogue writes the source plan's fp64 and fp32 rings) instead
  of projecting K x T samples and transforming N_src >> C channels.
  ``apply_inverse`` is the same GEMM engine on samples (``cs_apply_inverse``).
* Streaming FIR (reference preprocess.py:109-142): direct-form causal convolution
  with the previous block's last n_taps - 1 input samples carried
  (``cs_fir_apply``), equal to the reference's overlap-add output.
"""
from __future__ import annotations

import ctypes

import numpy as np
import torch

from . import _lib
from .core import EpochMatrix, ParameterError
from .plan import SEVEN, DevicePlan, _stream_ptr, pow2_scale


def _dev(a, dtype=torch.float64):
    from .spectral import _device
    t = a if isinstance(a, torch.Tensor) else torch.as_tensor(np.asarray(a, dtype=np.float64))
    return t.to(device=_device(), dtype=dtype)


def apply_inverse(op, epoch: EpochMatrix) -> EpochMatrix:
    """Project a sensor-space epoch to source space on the device (inverse.py:147-154);
    ``op`` is an operator with ``.M`` [n_sources, n_sensors] or the matrix itself."""
    M = _dev(op.M if hasattr(op, "M") else op).contiguous()
    if epoch.n_channels != M.shape[1]:
        raise ParameterError(f"operator expects {M.shape[1]} sensors, got {epoch.n_channels}")
    x = _dev(epoch.data).contiguous()
    y = torch.empty((M.shape[0], x.shape[1]), dtype=torch.float64, device=x.device)
    _lib.check(_lib.lib().cs_apply_inverse(ctypes.c_void_p(M.data_ptr()), int(M.shape[0]), int(M.shape[1]),
                                           ctypes.c_void_p(x.data_ptr()), int(x.shape[1]),
                                           ctypes.c_void_p(y.data_ptr()), _stream_ptr(None)))
    return EpochMatrix(data=y, sfreq=epoch.sfreq, t0_offset=epoch.t0_offset, trial_index=epoch.trial_index)


def source_connectivity(x_sensors: torch.Tensor, M, nfft: int, lo: int, hi: int, metrics=SEVEN, taper=None,
                        per_bin=True, band=True, mode: str = "fixed"):
    """Connectivity between the N_src sources of ``M @ x`` for sensor trials
    x [K, C, T] (device), computed as K1 on the sensors + a spectral projection
    of the ring + the fused pair kernels on the sources.  Returns
    (outputs, source_plan) like ``compute_connectivity``."""
    K, C, T = x_sensors.shape
    Md = _dev(M).contiguous()
    if Md.dim() != 2 or Md.shape[1] != C:
        raise ParameterError(f"operator must be [n_sources, {C}], got {tuple(Md.shape)}")
    N = Md.shape[0]
    sens_scale = pow2_scale(float(x_sensors.abs().amax()), min(T, nfft))
    sens = DevicePlan(C, T, nfft, lo, hi, taper=taper, slot_capacity=K, device=x_sensors.device,
                      scale=sens_scale, welch=(mode == "welch"))
    sens.spectra(x_sensors, 0)
    # fp32 scale of the source ring: a power of two from the projection's gain bound
    # (|y| <= max_n sum_c |M_nc| max|x|); every metric is invariant to it
    gain = float(Md.abs().sum(dim=1).max())
    scale = sens_scale * (2.0 ** -int(np.ceil(np.log2(gain))) if gain > 0 else 1.0)
    src = DevicePlan(N, nfft, nfft, lo, hi, slot_capacity=K, device=x_sensors.device, scale=scale,
                     n_tapers=sens.n_tapers)
    _lib.check(_lib.lib().cs_project_ring(src._h, sens._h, ctypes.c_void_p(Md.data_ptr()), 0, K,
                                          _stream_ptr(None)))
    src._keep = (sens, Md)
    slots = torch.arange(K, dtype=torch.int32, device=x_sensors.device)
    out = src.pair_metrics(slots, metrics, 0, src.n_bins, per_bin=per_bin, band=band)
    return out, src


class OverlapAddFilter:
    """Streaming causal FIR on the device (preprocess.py:109-136): each block is
    convolved with the taps continuing from the previous block's last samples, so
    the concatenated output equals ``np.convolve(signal, taps)[:len(signal)]``."""

    def __init__(self, fir):
        taps = fir.taps if hasattr(fir, "taps") else fir
        self.taps = _dev(taps).flatten().contiguous()
        self._hist = None
        self._n_channels = None

    def process(self, block):
        b = _dev(block)
        if b.dim() == 1:
            b = b[None]
        b = b.contiguous()
        C, S = b.shape
        H = self.taps.numel() - 1
        if self._n_channels is None:
            self._n_channels = C
            self._hist = torch.zeros((C, max(H, 1)), dtype=torch.float64, device=b.device)
        elif C != self._n_channels:
            raise ParameterError(f"channel count changed mid-stream: {self._n_channels} -> {C}")
        y = torch.empty_like(b)
        new_hist = torch.empty_like(self._hist)
        _lib.check(_lib.lib().cs_fir_apply(ctypes.c_void_p(self.taps.data_ptr()), int(H + 1),
                                           ctypes.c_void_p(b.data_ptr()), C, S,
                                           ctypes.c_void_p(self._hist.data_ptr()),
                                           ctypes.c_void_p(new_hist.data_ptr()), ctypes.c_void_p(y.data_ptr()),
                                           _stream_ptr(None)))
        self._hist = new_hist
        return y


def filter_offline(fir, data):
    """One-shot causal convolution truncated to the input length (preprocess.py:139-142)."""
    return OverlapAddFilter(fir).process(data)
