"""Upstream of the spectra: source projection and FIR filtering.

* Inverse projection (reference inverse.py:147-154: source data = M @ sensor
  data, then the spectral path on the sources).  Demean, taper and the DFT are
  linear per channel, so the source spectra equal M times the sensor spectra:
  ``source_connectivity`` runs K1 on the C sensors and projects the HBM spectrum
  ring, a [K L nb, C] x [C, N_src] complex GEMM (cuBLAS, fp64) instead of
  projecting K x T samples and transforming N_src >> C channels.
* Overlap-add FIR (reference preprocess.py:109-142): streaming FFT convolution
  with the block tail carried over (cuFFT, fp64), equal to the causal convolution
  truncated to the input length.
"""
from __future__ import annotations

import numpy as np
import torch

from .core import EpochMatrix, ParameterError
from .plan import SEVEN, DevicePlan, pow2_scale


def _dev(a, dtype=torch.float64):
    from .spectral import _device
    t = a if isinstance(a, torch.Tensor) else torch.as_tensor(np.asarray(a, dtype=np.float64))
    return t.to(device=_device(), dtype=dtype)


def apply_inverse(op, epoch: EpochMatrix) -> EpochMatrix:
    """Project a sensor-space epoch to source space on the device (inverse.py:147-154);
    ``op`` is an operator with ``.M`` [n_sources, n_sensors] or the matrix itself."""
    M = op.M if hasattr(op, "M") else op
    M = _dev(M)
    if epoch.n_channels != M.shape[1]:
        raise ParameterError(f"operator expects {M.shape[1]} sensors, got {epoch.n_channels}")
    return EpochMatrix(data=M @ _dev(epoch.data), sfreq=epoch.sfreq, t0_offset=epoch.t0_offset,
                       trial_index=epoch.trial_index)


def source_connectivity(x_sensors: torch.Tensor, M, nfft: int, lo: int, hi: int, metrics=SEVEN, taper=None,
                        per_bin=True, band=True, mode: str = "fixed"):
    """Connectivity between the N_src sources of ``M @ x`` for sensor trials
    x [K, C, T] (device), computed as K1 on the sensors + a spectral projection
    of the ring + the fused pair kernels on the sources.  Returns
    (outputs, source_plan) like ``compute_connectivity``."""
    K, C, T = x_sensors.shape
    Md = _dev(M)
    if Md.dim() != 2 or Md.shape[1] != C:
        raise ParameterError(f"operator must be [n_sources, {C}], got {tuple(Md.shape)}")
    N = Md.shape[0]
    sens = DevicePlan(C, T, nfft, lo, hi, taper=taper, slot_capacity=K, device=x_sensors.device,
                      scale=pow2_scale(float(x_sensors.abs().amax()), min(T, nfft)), welch=(mode == "welch"))
    sens.spectra(x_sensors, 0)
    Xs = sens.ring()[0][:K]                                   # [K, L, nb, C] complex128
    Lt, nb = Xs.shape[1], Xs.shape[2]
    Xsrc = (Xs.reshape(K * Lt * nb, C) @ Md.T.to(torch.complex128)).reshape(K, Lt, nb, N)  # ZGEMM
    amax = float(Xsrc.abs().amax())
    scale = 2.0 ** -int(np.ceil(np.log2(amax))) if amax > 0 else 1.0
    src = DevicePlan(N, nfft, nfft, lo, hi, slot_capacity=K, device=x_sensors.device, scale=scale, n_tapers=Lt)
    r64, r32 = src.ring()
    r64[:K].copy_(Xsrc)
    r32[:K].copy_((Xsrc * scale).to(torch.complex64))
    slots = torch.arange(K, dtype=torch.int32, device=x_sensors.device)
    out = src.pair_metrics(slots, metrics, 0, src.n_bins, per_bin=per_bin, band=band)
    return out, src


class OverlapAddFilter:
    """Streaming causal FIR on the device (preprocess.py:109-136): each block is
    FFT-convolved with the taps and the previous block's tail is added, so the
    concatenated output equals ``np.convolve(signal, taps)[:len(signal)]``."""

    def __init__(self, fir):
        taps = fir.taps if hasattr(fir, "taps") else fir
        self.taps = _dev(taps).flatten()
        self._tail = None
        self._n_channels = None

    def process(self, block):
        b = _dev(block)
        if b.dim() == 1:
            b = b[None]
        C, S = b.shape
        if self._n_channels is None:
            self._n_channels = C
            self._tail = torch.zeros((C, self.taps.numel() - 1), dtype=torch.float64, device=b.device)
        elif C != self._n_channels:
            raise ParameterError(f"channel count changed mid-stream: {self._n_channels} -> {C}")
        Lt = self._tail.shape[1]
        n = S + Lt
        nf = 1 << max(1, (n - 1).bit_length())
        full = torch.fft.irfft(torch.fft.rfft(b, nf, dim=1) * torch.fft.rfft(self.taps, nf)[None], nf, dim=1)[:, :n]
        if Lt:
            full[:, :Lt] += self._tail
            self._tail = full[:, S:].clone()
        return full[:, :S]


def filter_offline(fir, data):
    """One-shot causal convolution truncated to the input length (preprocess.py:139-142)."""
    return OverlapAddFilter(fir).process(data)
