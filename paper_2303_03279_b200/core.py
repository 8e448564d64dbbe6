"""Domain types of the reference's public API (connstream.core, core.py:17-160),
restated so the drop-in keeps the same names, argument meaning and errors.

``ConnectivityNetwork`` keeps its weights on the device and materialises the
O(P) host arrays (edge_i, edge_j, weights) only on access -- at 10k nodes the
reference's eager host arrays alone are 3 x 420 MB (core.py:141-152).
"""
from __future__ import annotations

from dataclasses import dataclass, field
from enum import Enum

import numpy as np


class ParameterError(ValueError):
    """Invalid argument (core.py:17)."""


class DegenerateTrialCountError(ParameterError):
    """Metric requested with too few accumulated trials (core.py:21)."""


class MetricId(str, Enum):
    COR = "COR"
    XCOR = "XCOR"
    COHY = "COHY"
    COH = "COH"
    IMAGCOHY = "IMAGCOHY"
    PLV = "PLV"
    PLI = "PLI"
    USPLI = "USPLI"
    WPLI = "WPLI"
    DSWPLI = "DSWPLI"

    @classmethod
    def parse(cls, name: str) -> "MetricId":
        key = str(name).strip().upper()
        if key not in cls.__members__:
            raise ParameterError(f"unknown metric {name!r}")
        return cls[key]

    @property
    def is_spectral(self) -> bool:
        return self not in (MetricId.COR, MetricId.XCOR)


SIGNED_METRICS = frozenset({MetricId.COR, MetricId.IMAGCOHY, MetricId.USPLI})


@dataclass(frozen=True)
class FrequencyBand:
    """Inclusive bin range [lo_bin, hi_bin] and the Hz width of a bin (core.py:53-76)."""

    lo_bin: int
    hi_bin: int
    bin_hz: float

    def __post_init__(self):
        if self.lo_bin < 0 or self.hi_bin < self.lo_bin:
            raise ParameterError(f"invalid band bins [{self.lo_bin}, {self.hi_bin}]")

    @property
    def n_bins(self) -> int:
        return self.hi_bin - self.lo_bin + 1

    @property
    def lo_hz(self) -> float:
        return self.lo_bin * self.bin_hz

    @property
    def hi_hz(self) -> float:
        return self.hi_bin * self.bin_hz

    @classmethod
    def from_hz(cls, lo_hz: float, hi_hz: float, sfreq: float, nfft: int) -> "FrequencyBand":
        """Nearest-bin rule (SURVEY.md conventions item 10)."""
        bin_hz = sfreq / nfft
        return cls(int(round(lo_hz / bin_hz)), int(round(hi_hz / bin_hz)), bin_hz)


@dataclass(frozen=True)
class EpochMatrix:
    """One trial, channels x samples (core.py:79-108).  ``data`` may be a numpy
    array (cast to float64 as in the reference) or a torch tensor already on
    the device (kept as is: float32 or float64)."""

    data: object
    sfreq: float
    t0_offset: float = 0.0
    trial_index: int = 0

    def __post_init__(self):
        d = self.data
        try:
            import torch
            is_t = isinstance(d, torch.Tensor)
        except ImportError:  # pragma: no cover
            is_t = False
        if is_t:
            if d.dim() != 2:
                raise ParameterError("epoch data must be 2-D (channels x samples)")
            shape = tuple(d.shape)
        else:
            d = np.asarray(d, dtype=np.float64)
            object.__setattr__(self, "data", d)
            if d.ndim != 2:
                raise ParameterError("epoch data must be 2-D (channels x samples)")
            shape = d.shape
        if shape[0] < 1 or shape[1] < 2:
            raise ParameterError(f"epoch too small: {shape}")
        if self.sfreq <= 0:
            raise ParameterError("sfreq must be positive")
        if self.trial_index < 0:
            raise ParameterError("trial_index must be non-negative")
        finite = bool(d.isfinite().all()) if is_t else bool(np.all(np.isfinite(d)))
        if not finite:
            raise ParameterError("epoch contains non-finite values")

    @property
    def n_channels(self) -> int:
        return int(self.data.shape[0])

    @property
    def n_samples(self) -> int:
        return int(self.data.shape[1])


def default_positions(n_nodes: int) -> np.ndarray:
    return np.zeros((n_nodes, 3))


def _triu(n: int):
    return np.triu_indices(n, k=1)


class ConnectivityNetwork:
    """Undirected all-to-all network over i < j (core.py:119-160).

    ``weights`` / ``complex_weights`` may be given as device tensors; the host
    numpy views (float64 / complex128) and the edge index arrays are built on
    first access.
    """

    def __init__(self, metric, band, n_trials, node_ids, positions, weights, edge_i=None, edge_j=None,
                 complex_weights=None, lags=None, normalized=False, warnings=()):
        if n_trials < 1:
            raise ParameterError("n_trials must be >= 1")
        self.metric = metric
        self.band = band
        self.n_trials = int(n_trials)
        self.node_ids = tuple(node_ids)
        self.positions = np.asarray(positions, dtype=np.float64).reshape(-1, 3)
        self._w = weights
        self._cw = complex_weights
        self._ei, self._ej = edge_i, edge_j
        self.lags = lags
        self.normalized = normalized
        self.warnings = tuple(warnings)
        self._check_finite()

    def _check_finite(self):
        w = self._w
        try:
            import torch
            if isinstance(w, torch.Tensor):
                if not bool(torch.isfinite(w).all()):
                    raise ParameterError("edge weights must be finite")
                return
        except ImportError:  # pragma: no cover
            pass
        if not np.all(np.isfinite(np.asarray(w))):
            raise ParameterError("edge weights must be finite")

    @staticmethod
    def _host(v, dtype):
        if v is None:
            return None
        try:
            import torch
            if isinstance(v, torch.Tensor):
                v = v.detach().cpu().numpy()
        except ImportError:  # pragma: no cover
            pass
        return np.asarray(v).astype(dtype, copy=False)

    @property
    def weights(self) -> np.ndarray:
        if not isinstance(self._w, np.ndarray) or self._w.dtype != np.float64:
            self._w = self._host(self._w, np.float64)
        return self._w

    @property
    def weights_device(self):
        return self._w

    @property
    def complex_weights(self):
        if self._cw is None:
            return None
        if not isinstance(self._cw, np.ndarray):
            self._cw = self._host(self._cw, np.complex128)
        return self._cw

    @property
    def edge_i(self) -> np.ndarray:
        if self._ei is None:
            self._ei, self._ej = (a.astype(np.int64) for a in _triu(self.n_nodes))
        return self._ei

    @property
    def edge_j(self) -> np.ndarray:
        if self._ej is None:
            self._ei, self._ej = (a.astype(np.int64) for a in _triu(self.n_nodes))
        return self._ej

    @property
    def n_nodes(self) -> int:
        return len(self.node_ids)

    @property
    def n_edges(self) -> int:
        return int(self._w.shape[0])


def band_average(per_bin_weights, band: FrequencyBand):
    """Mean over the inclusive bin range of ``band`` (core.py:208-215); accepts
    [P, nb] numpy arrays (reference layout) or torch tensors."""
    n_bins = per_bin_weights.shape[1]
    if band.hi_bin >= n_bins:
        raise ParameterError(f"band [{band.lo_bin}, {band.hi_bin}] exceeds {n_bins} bins")
    return per_bin_weights[:, band.lo_bin:band.hi_bin + 1].mean(axis=1) if isinstance(per_bin_weights, np.ndarray) \
        else per_bin_weights[:, band.lo_bin:band.hi_bin + 1].mean(dim=1)
