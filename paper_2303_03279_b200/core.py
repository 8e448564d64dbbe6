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
        if is_t and d.is_cuda:
            # device samples: the finiteness flag stays on the device (no host sync per
            # trial); it is checked by validate(), which the engine calls once per finalize
            object.__setattr__(self, "_finite_dev", d.isfinite().all())
            return
        finite = bool(d.isfinite().all()) if is_t else bool(np.all(np.isfinite(d)))
        if not finite:
            raise ParameterError("epoch contains non-finite values")

    def validate(self) -> None:
        """Raise ParameterError if the samples are not finite (core.py:97-100);
        synchronises only for device samples whose check is still pending."""
        f = self.__dict__.get("_finite_dev")
        if f is not None:
            ok = bool(f)
            object.__setattr__(self, "_finite_dev", None)
            if not ok:
                raise ParameterError("epoch contains non-finite values")

    @property
    def n_channels(self) -> int:
        return int(self.data.shape[0])

    @property
    def n_samples(self) -> int:
        return int(self.data.shape[1])


@dataclass(frozen=True)
class XCorEdgeValue:
    """Peak of the normalised cross-correlation and the lag where it occurs (core.py:111-116)."""

    peak_value: float
    peak_lag: int


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

    def __init__(self, metric, band, n_trials, node_ids, positions, edge_i=None, edge_j=None, weights=None,
                 complex_weights=None, lags=None, normalized=False, warnings=(), pairs=None):
        """Fields in the reference dataclass's order (core.py:130-141), so positional
        construction by reference callers keeps working.  edge_i / edge_j may be
        omitted: then the edges are all i < j pairs, or ``pairs`` -- optional device
        int64 pair indices (triu order) when they are a subset thresholded on the device."""
        if weights is None:
            raise ParameterError("weights are required")
        if n_trials < 1:
            raise ParameterError("n_trials must be >= 1")
        if edge_i is not None or edge_j is not None:
            if edge_i is None or edge_j is None:
                raise ParameterError("edge_i and edge_j go together")
            edge_i = np.asarray(edge_i, dtype=np.int64)
            edge_j = np.asarray(edge_j, dtype=np.int64)
            if np.any(edge_i >= edge_j):
                raise ParameterError("edges must satisfy i < j")
        self._pairs = pairs
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
                # device weights come from the pair kernels, finite by construction for
                # finite (validated) epochs: checked on host access, not with a sync here
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
            if not np.all(np.isfinite(self._w)):
                raise ParameterError("edge weights must be finite")
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

    def _edges(self):
        if self._ei is None:
            if self._pairs is None:
                self._ei, self._ej = (a.astype(np.int64) for a in _triu(self.n_nodes))
            else:
                p = self._host(self._pairs, np.int64)
                self._ei, self._ej = pair_to_ij(p, self.n_nodes)
        return self._ei, self._ej

    @property
    def edge_i(self) -> np.ndarray:
        return self._edges()[0]

    @property
    def edge_j(self) -> np.ndarray:
        return self._edges()[1]

    def _replace(self, **kw):
        d = dict(metric=self.metric, band=self.band, n_trials=self.n_trials, node_ids=self.node_ids,
                 positions=self.positions, weights=self._w, edge_i=self._ei, edge_j=self._ej,
                 complex_weights=self._cw, lags=self.lags, normalized=self.normalized, warnings=self.warnings,
                 pairs=self._pairs)
        d.update(kw)
        ei, ej = d.pop("edge_i"), d.pop("edge_j")
        net = ConnectivityNetwork(**d)
        net._ei, net._ej = ei, ej        # subsets of validated edges: no second i < j pass
        return net

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


def pair_to_ij(p: np.ndarray, n: int):
    """(i, j) of upper-triangle pair indices p (inverse of spectral.py:119-122)."""
    p = np.asarray(p, dtype=np.int64)
    i = np.floor((2 * n - 1 - np.sqrt((2.0 * n - 1) ** 2 - 8.0 * p)) / 2).astype(np.int64)
    i = np.clip(i, 0, max(n - 2, 0))
    start = i * (n - 1) - i * (i - 1) // 2
    fix = start > p                      # guard the float sqrt at row boundaries
    i[fix] -= 1
    start = i * (n - 1) - i * (i - 1) // 2
    nxt = (i + 1) * (n - 1) - (i + 1) * i // 2
    fix = (nxt <= p) & (i + 1 < n - 1)
    i[fix] += 1
    start = i * (n - 1) - i * (i - 1) // 2
    return i, p - start + i + 1


def _is_device(t) -> bool:
    try:
        import torch
        return isinstance(t, torch.Tensor) and t.is_cuda
    except ImportError:  # pragma: no cover
        return False


def normalize_network(net: ConnectivityNetwork) -> ConnectivityNetwork:
    """Scale all edge weights by the maximum |weight| (core.py:168-181); an
    all-zero network is returned unchanged apart from the flag.  Device weights
    are normalised on the device (cs_net_normalize)."""
    if net.n_edges < 1:
        raise ParameterError("cannot normalize a network without edges")
    if _is_device(net.weights_device):
        import ctypes
        import torch
        from . import _lib
        w = net.weights_device.to(torch.float32).clone()
        cw = net._cw.to(torch.complex64).clone() if _is_device(net._cw) else None
        with torch.cuda.device(w.device):
            _lib.check(_lib.lib().cs_net_normalize(ctypes.c_void_p(w.data_ptr()),
                                                   ctypes.c_void_p(cw.data_ptr()) if cw is not None else None,
                                                   int(w.numel()),
                                                   ctypes.c_void_p(torch.cuda.current_stream().cuda_stream)))
        return net._replace(weights=w, complex_weights=cw if cw is not None else net._cw, normalized=True)
    wmax = float(np.max(np.abs(net.weights)))
    if wmax == 0.0:
        return net._replace(normalized=True)
    cw = net.complex_weights / wmax if net.complex_weights is not None else None
    return net._replace(weights=net.weights / wmax, complex_weights=cw, normalized=True)


def threshold_network(net: ConnectivityNetwork, keep_fraction: float) -> ConnectivityNetwork:
    """Keep the ceil(keep_fraction * n_edges) strongest edges by |weight|, ties
    broken by ascending (i, j) (core.py:184-205).  Device weights are selected on
    the device (cs_net_threshold: radix select + ordered compaction)."""
    import math
    if not (0.0 < keep_fraction <= 1.0):
        raise ParameterError(f"keep_fraction must be in (0, 1], got {keep_fraction}")
    n_keep = math.ceil(keep_fraction * net.n_edges)
    if _is_device(net.weights_device):
        import ctypes
        import torch
        from . import _lib
        w = net.weights_device.to(torch.float32).contiguous()
        idx = torch.empty(n_keep, dtype=torch.int64, device=w.device)
        with torch.cuda.device(w.device):
            _lib.check(_lib.lib().cs_net_threshold(ctypes.c_void_p(w.data_ptr()), int(w.numel()), int(n_keep),
                                                   ctypes.c_void_p(idx.data_ptr()),
                                                   ctypes.c_void_p(torch.cuda.current_stream().cuda_stream)))
        pairs = idx if net._pairs is None else net._pairs[idx]
        cw = net._cw[idx] if _is_device(net._cw) else (net.complex_weights[idx.cpu().numpy()]
                                                      if net._cw is not None else None)
        lags = None if net.lags is None else np.asarray(net.lags)[idx.cpu().numpy()]
        return net._replace(weights=w[idx], complex_weights=cw, lags=lags, edge_i=None, edge_j=None, pairs=pairs)
    order = np.lexsort((net.edge_j, net.edge_i, -np.abs(net.weights)))   # last key is primary
    kept = np.sort(order[:n_keep])
    return net._replace(weights=net.weights[kept], edge_i=net.edge_i[kept], edge_j=net.edge_j[kept],
                        complex_weights=net.complex_weights[kept] if net.complex_weights is not None else None,
                        lags=np.asarray(net.lags)[kept] if net.lags is not None else None, pairs=None)


def serialize_network(net: ConnectivityNetwork) -> bytes:
    """Canonical UTF-8 JSON (core.py:218-243): fixed key order, so
    re-serialisation is byte-identical."""
    import json
    cw = net.complex_weights
    lags = net.lags
    ei, ej, w = net.edge_i, net.edge_j, net.weights
    obj = {
        "metric": net.metric.value,
        "band": {"lo_bin": net.band.lo_bin, "hi_bin": net.band.hi_bin, "bin_hz": net.band.bin_hz},
        "n_trials": net.n_trials,
        "normalized": net.normalized,
        "nodes": [{"id": int(nid), "pos": [float(x) for x in pos]} for nid, pos in zip(net.node_ids, net.positions)],
        "edges": [{"i": int(ei[k]), "j": int(ej[k]), "w": float(w[k]),
                   "w_im": float(cw[k].imag) if cw is not None else None,
                   "lag": int(lags[k]) if lags is not None else None} for k in range(net.n_edges)],
    }
    return json.dumps(obj, separators=(",", ":")).encode("utf-8")


def deserialize_network(raw: bytes) -> ConnectivityNetwork:
    """Inverse of serialize_network (core.py:246-273).  The wire format carries
    (|c|, Im c) for complex metrics, so the real part comes back as
    sqrt(|c|^2 - Im^2) (sign lost, as in the reference); re-serialisation is
    byte-identical."""
    import json
    obj = json.loads(raw.decode("utf-8"))
    b = obj["band"]
    band = FrequencyBand(b["lo_bin"], b["hi_bin"], b["bin_hz"])
    node_ids = tuple(n["id"] for n in obj["nodes"])
    positions = np.array([n["pos"] for n in obj["nodes"]], dtype=np.float64).reshape(-1, 3)
    edges = obj["edges"]
    ei = np.fromiter((e["i"] for e in edges), dtype=np.int64, count=len(edges))
    ej = np.fromiter((e["j"] for e in edges), dtype=np.int64, count=len(edges))
    w = np.fromiter((e["w"] for e in edges), dtype=np.float64, count=len(edges))
    cw = lags = None
    if any(e["w_im"] is not None for e in edges):
        im = np.array([e["w_im"] or 0.0 for e in edges], dtype=np.float64)
        cw = np.sqrt(np.maximum(w * w - im * im, 0.0)) + 1j * im
    if any(e["lag"] is not None for e in edges):
        lags = np.array([e["lag"] or 0 for e in edges], dtype=np.int64)
    return ConnectivityNetwork(MetricId.parse(obj["metric"]), band, obj["n_trials"], node_ids, positions, ei, ej, w,
                               complex_weights=cw, lags=lags, normalized=obj["normalized"])
