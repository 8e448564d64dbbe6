"""Device plan: the HBM spectrum ring plus the fused pair kernels (csconn C ABI).

This is the B200-native replacement of the reference's per-trial fold
(spectral.py:204-261) and finalisers (metrics.py:32-134): one plan owns the
spectrum cache of ``slot_capacity`` trials (fp64 + scaled fp32 copies) and runs
K1 (taper + DFT) and the pair kernels over any list of cached trial slots.
"""
from __future__ import annotations

import ctypes
import math

import numpy as np
import torch

from . import _lib
from .core import ParameterError

METRIC_BITS = {"COHY": 0, "COH": 1, "IMAGCOHY": 2, "PLV": 3, "PLI": 4, "USPLI": 5, "WPLI": 6, "DSWPLI": 7}
SEVEN = ("COH", "IMAGCOHY", "PLV", "PLI", "USPLI", "WPLI", "DSWPLI")


def _stream_ptr(stream: torch.cuda.Stream | None) -> ctypes.c_void_p:
    s = stream if stream is not None else torch.cuda.current_stream()
    return ctypes.c_void_p(s.cuda_stream)


def make_taper(taper, n_eff: int):
    """None/'boxcar' -> rectangular (the reference), 'hann' -> np.hanning(n_eff),
    ('dpss', NW, L) -> scipy.signal.windows.dpss(n_eff, NW, Kmax=L), or an explicit
    [L, n_eff] / [n_eff] array (SURVEY.md conventions item 11)."""
    if taper is None or (isinstance(taper, str) and taper.lower() in ("boxcar", "rect", "none")):
        return None
    if isinstance(taper, str) and taper.lower() == "hann":
        return np.hanning(n_eff)[None, :]
    if isinstance(taper, tuple) and taper and str(taper[0]).lower() == "dpss":
        from scipy.signal import windows
        return np.atleast_2d(windows.dpss(n_eff, float(taper[1]), Kmax=int(taper[2])))
    arr = np.atleast_2d(np.asarray(taper, dtype=np.float64))
    if arr.shape[1] != n_eff:
        raise ParameterError(f"taper length {arr.shape[1]} != {n_eff}")
    return arr


def pow2_scale(max_abs: float, n_eff: int) -> float:
    """Power-of-two scale bringing spectra to O(1) in the fp32 copy (metrics are
    invariant to it; it only protects the fp32 range)."""
    if not (max_abs > 0.0) or not math.isfinite(max_abs):
        return 1.0
    e = -round(math.log2(max_abs * math.sqrt(n_eff)))
    e = max(-100, min(100, e))
    return float(2.0 ** e)


class DevicePlan:
    """Owns a csconn plan: spectrum ring of ``slot_capacity`` trials for bins
    [lo, hi] of an nfft-point one-sided spectrum."""

    def __init__(self, n_nodes: int, n_samples: int, nfft: int, lo: int, hi: int, taper=None,
                 slot_capacity: int = 1, device=None, scale: float = 1.0, welch: bool = False,
                 n_tapers: int | None = None):
        """welch: segment mode (spectral.py:100-111, 264-283) -- trials of
        n_samples >= 2 nfft become n_samples // nfft demeaned nfft segments on the
        taper axis.  n_tapers (no taper given): a rectangular ring with that many
        taper slots, filled by put_spectra(..., taper=l) (mixed welch trials)."""
        if not torch.cuda.is_available():
            raise RuntimeError("paper_2303_03279_b200 needs a CUDA device (B200); there is no CPU fallback")
        dev = torch.device(device) if device is not None else torch.device("cuda")
        if dev.index is None:
            dev = torch.device("cuda", torch.cuda.current_device())
        self.device = dev
        self.n_nodes, self.n_samples, self.nfft = int(n_nodes), int(n_samples), int(nfft)
        self.lo, self.hi = int(lo), int(hi)
        self.n_bins = self.hi - self.lo + 1
        self.welch = bool(welch) and self.n_samples >= 2 * self.nfft
        if welch and taper is not None:
            raise ParameterError("welch mode takes no taper")
        self.n_eff = self.nfft if self.welch else min(self.n_samples, self.nfft)
        tap = make_taper(taper, self.n_eff)
        if tap is None and n_tapers is not None and int(n_tapers) > 1:
            tap = np.ones((int(n_tapers), self.n_eff))  # rectangular taper slots
        self.n_tapers = (self.n_samples // self.nfft if self.welch else 1) if tap is None else tap.shape[0]
        self.slot_capacity = int(slot_capacity)
        self.scale = float(scale)
        L = _lib.lib()
        h = ctypes.c_void_p()
        tptr = None
        if tap is not None:
            self._taper = np.ascontiguousarray(tap, dtype=np.float64)
            tptr = self._taper.ctypes.data_as(ctypes.POINTER(ctypes.c_double))
        with torch.cuda.device(self.device):
            _lib.check(L.cs_plan_create(ctypes.byref(h), self.device.index, self.n_nodes, self.n_samples,
                                        self.nfft, self.lo, self.hi, 1 if tap is None else self.n_tapers, tptr,
                                        self.slot_capacity, self.scale, _lib.CS_PLAN_WELCH if welch else 0))
        self._h = h
        self.profiling = False

    def __del__(self):
        h = getattr(self, "_h", None)
        if h is not None and h.value:
            try:
                _lib.lib().cs_plan_destroy(h)
            except Exception:
                pass
            self._h = None

    @property
    def n_pairs(self) -> int:
        return self.n_nodes * (self.n_nodes - 1) // 2

    # -- K1 ---------------------------------------------------------------
    def spectra(self, x: torch.Tensor, slot0: int = 0, stream=None) -> None:
        """x: device [k, N, T] (float32/float64; inner dim contiguous)."""
        if x.device != self.device:
            raise ParameterError("input must live on the plan's device")
        if x.dim() != 3 or x.shape[1] != self.n_nodes or x.shape[2] < 1:
            raise ParameterError(f"expected [k, {self.n_nodes}, T] samples, got {tuple(x.shape)}")
        if x.shape[2] != self.n_samples:
            raise ParameterError(f"plan expects {self.n_samples} samples per trial, got {x.shape[2]}")
        if x.stride(2) != 1:
            x = x.contiguous()
        if x.dtype == torch.float64:
            dt = _lib.CS_F64
        elif x.dtype == torch.float32:
            dt = _lib.CS_F32
        else:
            raise ParameterError(f"unsupported sample dtype {x.dtype}")
        self._last_x = x  # keep alive until the launch is ordered
        _lib.check(_lib.lib().cs_spectra(self._h, ctypes.c_void_p(x.data_ptr()), dt, x.stride(0), x.stride(1),
                                         int(slot0), int(x.shape[0]), _stream_ptr(stream)))

    def spectra_nodes(self, x: torch.Tensor, node0: int, slot0: int = 0, stream=None) -> None:
        """K1 for the node range [node0, node0 + x.shape[1]) only (multi-GPU: a rank's
        node block, csconn cs_spectra_nodes); x: device [k, n, T]."""
        if x.device != self.device:
            raise ParameterError("input must live on the plan's device")
        if x.dim() != 3 or x.shape[2] != self.n_samples or node0 < 0 or node0 + x.shape[1] > self.n_nodes:
            raise ParameterError(f"expected [k, n <= {self.n_nodes - node0}, {self.n_samples}] samples, "
                                 f"got {tuple(x.shape)}")
        if x.stride(2) != 1:
            x = x.contiguous()
        dt = {torch.float64: _lib.CS_F64, torch.float32: _lib.CS_F32}.get(x.dtype)
        if dt is None:
            raise ParameterError(f"unsupported sample dtype {x.dtype}")
        self._last_x = x
        _lib.check(_lib.lib().cs_spectra_nodes(self._h, ctypes.c_void_p(x.data_ptr()), dt, x.stride(0),
                                               x.stride(1), int(node0), int(x.shape[1]), int(slot0),
                                               int(x.shape[0]), _stream_ptr(stream)))

    # -- pair kernels -------------------------------------------------------
    def alloc_outputs(self, metrics, n_bins: int, per_bin=True, band=True, pair_count=None):
        P = self.n_pairs if pair_count is None else int(pair_count)
        out = {}
        for m in metrics:
            cplx = m == "COHY"
            dt = torch.complex64 if cplx else torch.float32
            out[m] = {"bins": torch.empty((n_bins, P), dtype=dt, device=self.device) if per_bin else None,
                      "band": torch.empty((P,), dtype=dt, device=self.device) if band else None}
        return out

    def pair_metrics(self, slots: torch.Tensor, metrics=SEVEN, bin_lo: int = 0, n_bins: int | None = None,
                     outputs=None, per_bin=True, band=True, row_tiles=(0, -1), pair_base: int = 0,
                     pair_count: int | None = None, stream=None, reuse_prep: bool = False):
        """reuse_prep: keep the node statistics and packed operands of the previous call
        (same slots tensor, bins and metrics; cs_pair_metrics_ex CS_PM_REUSE_PREP)."""
        if n_bins is None:
            n_bins = self.n_bins - bin_lo
        metrics = tuple(m.upper() for m in metrics)
        for m in metrics:
            if m not in METRIC_BITS:
                raise ParameterError(f"{m} is not a spectral metric")
        if slots.dtype != torch.int32 or slots.device != self.device:
            slots = slots.to(device=self.device, dtype=torch.int32)
        if outputs is None:
            outputs = self.alloc_outputs(metrics, n_bins, per_bin, band, pair_count)
        desc = _lib.CsOutputs()
        mask = 0
        for m in metrics:
            bit = METRIC_BITS[m]
            mask |= 1 << bit
            o = outputs[m]
            desc.bins[bit] = o["bins"].data_ptr() if o.get("bins") is not None else None
            desc.band[bit] = o["band"].data_ptr() if o.get("band") is not None else None
        desc.pair_base = int(pair_base)
        desc.pair_stride = int(self.n_pairs if pair_count is None else pair_count)
        self._last_slots = slots
        _lib.check(_lib.lib().cs_pair_metrics_ex(self._h, ctypes.c_void_p(slots.data_ptr()), int(slots.numel()),
                                                 mask, int(bin_lo), int(n_bins), int(row_tiles[0]),
                                                 int(row_tiles[1]), ctypes.byref(desc),
                                                 _lib.CS_PM_REUSE_PREP if reuse_prep else 0, _stream_ptr(stream)))
        return outputs

    def pair_sums(self, slots: torch.Tensor, bin_lo: int = 0, n_bins: int | None = None, stream=None) -> dict:
        """The reference's running sums over the trials in ``slots`` (cs_pair_sums):
        csd / plv complex128 [nbb, P], pli int32 [nbb, P], abs_im float64 [nbb, P],
        psd float64 [nbb, N] (bin-major; the reference layout is the transpose)."""
        if n_bins is None:
            n_bins = self.n_bins - bin_lo
        if slots.dtype != torch.int32 or slots.device != self.device:
            slots = slots.to(device=self.device, dtype=torch.int32)
        P = self.n_pairs
        o = {"csd": torch.empty((n_bins, P), dtype=torch.complex128, device=self.device),
             "plv": torch.empty((n_bins, P), dtype=torch.complex128, device=self.device),
             "pli": torch.empty((n_bins, P), dtype=torch.int32, device=self.device),
             "abs_im": torch.empty((n_bins, P), dtype=torch.float64, device=self.device),
             "psd": torch.empty((n_bins, self.n_nodes), dtype=torch.float64, device=self.device)}
        d = _lib.CsSums(o["csd"].data_ptr(), o["plv"].data_ptr(), o["pli"].data_ptr(), o["abs_im"].data_ptr(),
                        o["psd"].data_ptr(), 0, P)
        self._last_slots = slots
        _lib.check(_lib.lib().cs_pair_sums(self._h, ctypes.c_void_p(slots.data_ptr()), int(slots.numel()),
                                           int(bin_lo), int(n_bins), ctypes.byref(d), _stream_ptr(stream)))
        return o

    def fallback_count(self, stream=None) -> int:
        n = ctypes.c_int64()
        _lib.check(_lib.lib().cs_last_fallback_count(self._h, _stream_ptr(stream), ctypes.byref(n)))
        return int(n.value)

    def guard_stats(self, stream=None) -> dict:
        """Exact-sign guard of the last pair_metrics call: entries recomputed in fp64 and
        the overflow records used when the work list was full (none is ever dropped)."""
        n, r = ctypes.c_int64(), ctypes.c_int64()
        _lib.check(_lib.lib().cs_last_guard_stats(self._h, _stream_ptr(stream), ctypes.byref(n), ctypes.byref(r)))
        return {"flagged": int(n.value), "records": int(r.value),
                "imag_handoff": bool(_lib.lib().cs_last_imag_handoff(self._h))}

    def get_spectra(self, slots: torch.Tensor, bin_lo: int = 0, n_bins: int | None = None, stream=None):
        if n_bins is None:
            n_bins = self.n_bins - bin_lo
        slots = slots.to(device=self.device, dtype=torch.int32)
        dst = torch.empty((slots.numel(), self.n_nodes, n_bins), dtype=torch.complex128, device=self.device)
        _lib.check(_lib.lib().cs_get_spectra(self._h, ctypes.c_void_p(slots.data_ptr()), int(slots.numel()),
                                             int(bin_lo), int(n_bins), ctypes.c_void_p(dst.data_ptr()),
                                             _stream_ptr(stream)))
        return dst

    # -- instrumentation --------------------------------------------------------
    def set_profiling(self, on: bool = True) -> None:
        _lib.check(_lib.lib().cs_plan_set_profiling(self._h, int(bool(on))))
        self.profiling = bool(on)

    def profile(self) -> dict:
        """{phase: (total_ms, count)} since the last read (synchronises)."""
        buf = ctypes.create_string_buffer(4096)
        _lib.check(_lib.lib().cs_profile_read(self._h, buf, 4096))
        out = {}
        for rec in buf.value.decode().split(";"):
            if rec:
                name, ms, n = rec.split(":")
                out[name] = (float(ms), int(n))
        return out

    def launch_count(self) -> int:
        return int(_lib.lib().cs_launch_count(self._h))

    def ring(self):
        """(X64, X32) spectrum-ring views as torch tensors [slot, L, nb, N] complex."""
        x64, x32, n = ctypes.c_void_p(), ctypes.c_void_p(), ctypes.c_int64()
        _lib.check(_lib.lib().cs_ring_view(self._h, ctypes.byref(x64), ctypes.byref(x32), ctypes.byref(n)))
        shape = (self.slot_capacity, self.n_tapers, self.n_bins, self.n_nodes)
        return (_wrap(x64.value, shape, torch.complex128, self.device, self),
                _wrap(x32.value, shape, torch.complex64, self.device, self))

    def put_spectra(self, spectra: torch.Tensor, slot0: int, bin_lo: int = 0, stream=None, taper: int = 0,
                    weight: float = 1.0) -> None:
        """Upload complex128 spectra [n, N, nbins] (trial_spectra layout) into taper
        slot ``taper`` of slots slot0.., multiplied by ``weight``."""
        spectra = spectra.to(device=self.device, dtype=torch.complex128).contiguous()
        if spectra.dim() != 3 or spectra.shape[1] != self.n_nodes:
            raise ParameterError(f"spectra must be [n, {self.n_nodes}, bins], got {tuple(spectra.shape)}")
        self._last_put = spectra
        _lib.check(_lib.lib().cs_put_taper_spectra(self._h, ctypes.c_void_p(spectra.data_ptr()),
                                                   int(spectra.shape[0]), int(bin_lo), int(spectra.shape[2]),
                                                   int(slot0), int(taper), float(weight), _stream_ptr(stream)))

    @property
    def k1_kind(self) -> str:
        """The K1 kernel this plan runs: dft_fp64 | dft_tensor | fft4 | fft_radix2."""
        return ("dft_fp64", "dft_tensor", "fft4", "fft_radix2")[_lib.lib().cs_plan_k1_kind(self._h)]

    def fft_call_count(self) -> int:
        return int(_lib.lib().cs_fft_call_count(self._h))

    def reset_fft_call_count(self) -> None:
        _lib.lib().cs_reset_fft_call_count(self._h)


class _DevBuf:
    """__cuda_array_interface__ shim exposing a plan-owned device buffer to torch."""

    def __init__(self, ptr, shape, typestr, owner):
        self._owner = owner
        self.__cuda_array_interface__ = {"shape": shape, "typestr": typestr, "data": (ptr, False),
                                         "version": 3, "strides": None}


def _wrap(ptr, shape, dtype, device, owner):
    typestr = {torch.complex128: "<c16", torch.complex64: "<c8"}[dtype]
    with torch.cuda.device(device):
        return torch.as_tensor(_DevBuf(ptr, shape, typestr, owner), device=device)


def probe_peaks(device_index: int = 0):
    """(FP32 FMA-pipe lane ops/s, FP64 DFMA/s) measured live on this device."""
    a, b = ctypes.c_double(), ctypes.c_double()
    _lib.check(_lib.lib().cs_probe_peaks(int(device_index), ctypes.byref(a), ctypes.byref(b)))
    return a.value, b.value


def bind_host_to_gpu_numa(device_index: int = 0):
    """Pin this process to the CPU cores local to the GPU's PCIe root (sysfs
    local_cpulist), so pinned host buffers allocated afterwards land on the GPU's
    NUMA node and host<->device copies do not cross the inter-socket link.
    Returns (numa_node, n_cpus) or None when the topology is not visible."""
    import os
    try:
        pr = torch.cuda.get_device_properties(device_index)
        bdf = f"{pr.pci_domain_id:04x}:{pr.pci_bus_id:02x}:{pr.pci_device_id:02x}.0"
        base = f"/sys/bus/pci/devices/{bdf}"
        with open(f"{base}/local_cpulist") as f:
            spec = f.read().strip()
        cpus = set()
        for part in spec.split(","):
            if "-" in part:
                a, b = part.split("-")
                cpus.update(range(int(a), int(b) + 1))
            elif part:
                cpus.add(int(part))
        cpus &= os.sched_getaffinity(0)
        if not cpus:
            return None
        os.sched_setaffinity(0, cpus)
        try:
            with open(f"{base}/numa_node") as f:
                node = int(f.read().strip())
        except OSError:
            node = -1
        return node, len(cpus)
    except (OSError, AttributeError, ValueError):
        return None


def copy_ceilings(nbytes_h2d: int, nbytes_d2h: int, device=None, reps: int = 3) -> dict:
    """Measured pinned-host <-> device copy rates (GB/s, best of ``reps``) for buffers of
    the given sizes on this box: the ceiling an end-to-end step that moves those
    bytes cannot beat."""
    dev = torch.device(device) if device is not None else torch.device("cuda")
    out = {}
    for name, nb, h2d in (("h2d_gbs", nbytes_h2d, True), ("d2h_gbs", nbytes_d2h, False)):
        n = max(1, int(nb) // 4)
        h = torch.empty(n, dtype=torch.float32).pin_memory()
        d = torch.empty(n, dtype=torch.float32, device=dev)
        best = 0.0
        for _ in range(reps):
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record()
            (d.copy_(h, non_blocking=True) if h2d else h.copy_(d, non_blocking=True))
            e1.record()
            e1.synchronize()
            best = max(best, n * 4 / (e0.elapsed_time(e1) * 1e-3) / 1e9)
        out[name] = best
        del h, d
    # both directions at once (a pipelined step uploads and downloads concurrently)
    nh, nd = max(1, int(nbytes_h2d) // 4), max(1, int(nbytes_d2h) // 4)
    hh, dh = torch.empty(nh, dtype=torch.float32).pin_memory(), torch.empty(nh, dtype=torch.float32, device=dev)
    hd, dd = torch.empty(nd, dtype=torch.float32).pin_memory(), torch.empty(nd, dtype=torch.float32, device=dev)
    s1, s2 = torch.cuda.Stream(dev), torch.cuda.Stream(dev)
    best = float("inf")
    for _ in range(reps):
        torch.cuda.synchronize(dev)
        e0, e1, e2 = (torch.cuda.Event(enable_timing=True) for _ in range(3))
        e0.record()
        s1.wait_event(e0)
        s2.wait_event(e0)
        with torch.cuda.stream(s1):
            dh.copy_(hh, non_blocking=True)
            e1.record(s1)
        with torch.cuda.stream(s2):
            hd.copy_(dd, non_blocking=True)
            e2.record(s2)
        torch.cuda.synchronize(dev)
        best = min(best, max(e0.elapsed_time(e1), e0.elapsed_time(e2)))
    out["bidir_ms"] = best
    return out


def row_tile_range(n_nodes: int, n_shards: int, shard: int):
    L = _lib.lib()
    rb, re = ctypes.c_int(), ctypes.c_int()
    p0, p1 = ctypes.c_int64(), ctypes.c_int64()
    _lib.check(L.cs_row_tile_range(n_nodes, n_shards, shard, ctypes.byref(rb), ctypes.byref(re),
                                   ctypes.byref(p0), ctypes.byref(p1)))
    return (rb.value, re.value), (p0.value, p1.value)


def compute_connectivity(x: torch.Tensor, nfft: int, lo: int, hi: int, metrics=SEVEN, taper=None,
                         per_bin=True, band=True, plan: DevicePlan | None = None, stream=None, mode: str = "fixed"):
    """Batch path: all trials of x [K, N, T] (device) -> per-bin [nb, P] and band
    [P] outputs for ``metrics`` over the inclusive bins [lo, hi].  mode="welch":
    the reference's segment mode (spectral.py:264-283)."""
    if mode not in ("fixed", "welch"):
        raise ParameterError(f"unknown spectral mode {mode!r}")
    K, N, T = x.shape
    if plan is None:
        scale = pow2_scale(float(x.abs().amax()), min(T, nfft))
        plan = DevicePlan(N, T, nfft, lo, hi, taper=taper, slot_capacity=K, device=x.device, scale=scale,
                          welch=(mode == "welch"))
    plan.spectra(x, 0, stream=stream)
    slots = torch.arange(K, dtype=torch.int32, device=x.device)
    out = plan.pair_metrics(slots, metrics, 0, plan.n_bins, per_bin=per_bin, band=band, stream=stream)
    return out, plan


class HostPipeline:
    """Host-in / host-out batch path with the copies overlapped (the e2e call).

    ``run(xh)`` takes pinned host samples [K, N, T] and returns the band means of
    ``metrics`` as pinned host arrays [P] (pair order of ``np.triu_indices(N, 1)``),
    the layout of ``ConnectivityNetwork.weights`` (reference core.py:132-152).
    Inside one call the upload is split into trial chunks so K1 starts on the
    first chunk while the rest is in flight, and the pair kernels run over row-tile
    chunks so each chunk's download overlaps the next chunk's kernels.  ``submit``
    enqueues without waiting: the upload of call s+1 then overlaps the pair
    kernels and download of call s (three streams, event-ordered; the spectrum
    ring and outputs are reused, so every ordering hazard is an event wait).
    """

    def __init__(self, n_nodes: int, n_samples: int, nfft: int, lo: int, hi: int, n_trials: int,
                 metrics=SEVEN, taper=None, scale: float = 1.0, device=None, dtype=torch.float32,
                 in_chunks: int = 10, row_chunks: int = 8):
        self.plan = DevicePlan(n_nodes, n_samples, nfft, lo, hi, taper=taper, slot_capacity=n_trials,
                               device=device, scale=scale)
        dev = self.plan.device
        self.K = int(n_trials)
        self.metrics = tuple(m.upper() for m in metrics)
        # two device staging buffers: call s+1 uploads into the other one while call s's K1
        # reads its own, so the PCIe link stays busy from one call to the next
        self.xds = [torch.empty((self.K, n_nodes, n_samples), dtype=dtype, device=dev) for _ in range(2)]
        self.xd = self.xds[0]
        self._calls = 0
        self.slots = torch.arange(self.K, dtype=torch.int32, device=dev)
        P = self.plan.n_pairs
        self.out = {m: torch.empty((P,), dtype=torch.complex64 if m == "COHY" else torch.float32, device=dev)
                    for m in self.metrics}
        bounds = np.linspace(0, self.K, min(in_chunks, self.K) + 1).round().astype(int)
        self.k_chunks = [(int(a), int(b)) for a, b in zip(bounds[:-1], bounds[1:]) if b > a]
        self.r_chunks = []
        n_r = max(1, min(row_chunks, (n_nodes + 63) // 64))
        for r in range(n_r):
            rt, pr = row_tile_range(n_nodes, n_r, r)
            if pr[1] > pr[0]:
                self.r_chunks.append((rt, pr))
        with torch.cuda.device(dev):
            self.s_in, self.s_comp, self.s_out = torch.cuda.Stream(), torch.cuda.Stream(), torch.cuda.Stream()
            self.ev_in = [torch.cuda.Event() for _ in self.k_chunks]
            self.ev_k1s = [torch.cuda.Event() for _ in range(2)]
            self.ev_rows = [torch.cuda.Event() for _ in self.r_chunks]
            self.ev_out = torch.cuda.Event()
        self._armed = False  # ev_out recorded at least once

    def alloc_host(self):
        return {m: torch.empty(t.shape, dtype=t.dtype).pin_memory() for m, t in self.out.items()}

    @property
    def h2d_bytes(self) -> int:
        return self.xd.numel() * self.xd.element_size()

    def submit(self, xh: torch.Tensor, host_out: dict) -> torch.cuda.Event:
        """Enqueue one call; returns the event that completes its download."""
        if tuple(xh.shape) != tuple(self.xd.shape) or xh.dtype != self.xd.dtype:
            raise ParameterError(f"expected host samples {tuple(self.xd.shape)} {self.xd.dtype}")
        p = self.plan
        h = self._calls % 2
        xd, ev_k1 = self.xds[h], self.ev_k1s[h]
        if self._calls >= 2:
            self.s_in.wait_event(ev_k1)           # call s-2's K1 has consumed this buffer
        for (k0, k1), ev in zip(self.k_chunks, self.ev_in):
            with torch.cuda.stream(self.s_in):
                xd[k0:k1].copy_(xh[k0:k1], non_blocking=True)
            ev.record(self.s_in)
        for (k0, k1), ev in zip(self.k_chunks, self.ev_in):
            self.s_comp.wait_event(ev)
            p.spectra(xd[k0:k1], k0, stream=self.s_comp)
        ev_k1.record(self.s_comp)
        self._calls += 1
        if self._armed:
            self.s_comp.wait_event(self.ev_out)   # the previous call's download has read the outputs
        for q, (((rb, re), (p0, p1)), ev) in enumerate(zip(self.r_chunks, self.ev_rows)):
            view = {m: {"bins": None, "band": t[p0:p1]} for m, t in self.out.items()}
            # node statistics and operand packing once per step, not once per row chunk
            p.pair_metrics(self.slots, self.metrics, 0, p.n_bins, outputs=view, per_bin=False, band=True,
                           row_tiles=(rb, re), pair_base=p0, pair_count=p1 - p0, stream=self.s_comp,
                           reuse_prep=q > 0)
            ev.record(self.s_comp)
        for ((rb, re), (p0, p1)), ev in zip(self.r_chunks, self.ev_rows):
            self.s_out.wait_event(ev)
            with torch.cuda.stream(self.s_out):
                for m, t in self.out.items():
                    host_out[m][p0:p1].copy_(t[p0:p1], non_blocking=True)
        self.ev_out.record(self.s_out)
        self._armed = True
        return self.ev_out

    def run(self, xh: torch.Tensor, host_out: dict | None = None) -> dict:
        host_out = host_out if host_out is not None else self.alloc_host()
        self.submit(xh, host_out).synchronize()
        return host_out


class WindowGraph:
    """The online sliding-window update (``ConnectivityEngine.update_and_finalize``
    every ``n_new`` trials over the last ``window``; pipeline.py:304-309,
    metrics.py:450-460) replayed from CUDA graphs.

    The plan's ring holds exactly ``window`` slots: update u writes its ``n_new``
    trials over the ones that just left the window, and recomputes the metrics
    over the window's slots.  The (slot0, slot list) pattern repeats every
    ``window / gcd(window, n_new)`` updates, so one graph per phase and buffer is
    captured on first use (K1 on a staging buffer + the pair kernels into an
    output set) and replayed afterwards: an update is one staging copy and one
    graph launch instead of a dozen launches from Python.

    Staging buffers and output sets are double-buffered, so ``submit`` (host
    samples in, host band results out) overlaps update u+1's upload and update
    u-1's download with update u's kernels on separate copy streams.
    """

    def __init__(self, plan: DevicePlan, n_new: int, metrics=SEVEN, bin_lo: int = 0, n_bins: int | None = None,
                 per_bin=True, band=True, dtype=torch.float32, buffers: int = 2):
        self.plan = plan
        self.window = plan.slot_capacity
        self.n_new = int(n_new)
        if not 1 <= self.n_new <= self.window:
            raise ParameterError(f"n_new must be in [1, {self.window}], got {n_new}")
        self.metrics = tuple(m.upper() for m in metrics)
        self.bin_lo = int(bin_lo)
        self.n_bins = plan.n_bins - self.bin_lo if n_bins is None else int(n_bins)
        self.nbuf = max(1, int(buffers))
        self._outs = [plan.alloc_outputs(self.metrics, self.n_bins, per_bin, band) for _ in range(self.nbuf)]
        self._stage = [torch.empty((self.n_new, plan.n_nodes, plan.n_samples), dtype=dtype, device=plan.device)
                       for _ in range(self.nbuf)]
        self.n_phases = self.window // math.gcd(self.window, self.n_new)
        self._slots = [torch.tensor([(u * self.n_new + k) % self.window for k in range(self.window)],
                                    dtype=torch.int32, device=plan.device) for u in range(self.n_phases)]
        self._graphs: dict[tuple, torch.cuda.CUDAGraph] = {}
        self._kernels_per_update = 0
        self.updates = 0
        self._cur = 0
        with torch.cuda.device(plan.device):
            self._h2d, self._d2h = torch.cuda.Stream(), torch.cuda.Stream()
            self._ev_in = [torch.cuda.Event() for _ in range(self.nbuf)]
            self._ev_used = [torch.cuda.Event() for _ in range(self.nbuf)]   # graph done reading stage / writing outs
            self._ev_out = [torch.cuda.Event() for _ in range(self.nbuf)]    # download of outs done
            for e in self._ev_used + self._ev_out:
                e.record()

    @property
    def outputs(self) -> dict:
        """Output set of the latest update."""
        return self._outs[self._cur]

    @property
    def staging(self) -> torch.Tensor:
        return self._stage[0]

    def prime(self, x: torch.Tensor) -> dict:
        """Fill the ring with the first ``window`` trials [window, N, T] and compute
        the first window's metrics (not graphed)."""
        if x.shape[0] != self.window:
            raise ParameterError(f"prime needs {self.window} trials, got {x.shape[0]}")
        self.plan.spectra(x.to(self.plan.device, non_blocking=True), 0)
        self.plan.pair_metrics(self._slots[0], self.metrics, self.bin_lo, self.n_bins, outputs=self._outs[0])
        self._ev_used[0].record()
        self._cur = 0
        self.updates = 1
        return self._outs[0]

    def _body(self, u: int, b: int) -> None:
        slot0 = ((u - 1) * self.n_new) % self.window
        self.plan.spectra(self._stage[b], slot0)
        self.plan.pair_metrics(self._slots[u % self.n_phases], self.metrics, self.bin_lo, self.n_bins,
                               outputs=self._outs[b])

    def _run(self, u: int, b: int) -> None:
        key = (u % self.n_phases, b)
        g = self._graphs.get(key)
        if g is None:
            l0 = self.plan.launch_count()
            self._body(u, b)  # eager once per key: lazy allocations happen outside capture
            self._kernels_per_update = self.plan.launch_count() - l0
            torch.cuda.current_stream().synchronize()
            prof = self.plan.profiling
            if prof:  # per-phase timing events are not captured
                self.plan.set_profiling(False)
            g = torch.cuda.CUDAGraph()
            try:
                with torch.cuda.graph(g):
                    self._body(u, b)
            finally:
                if prof:
                    self.plan.set_profiling(True)
            self._graphs[key] = g
        g.replay()

    def submit(self, x_new: torch.Tensor, host_out: dict | None = None):
        """Append ``n_new`` trials [n_new, N, T] (pinned host or device memory) and
        enqueue the window update; with ``host_out`` ({metric: pinned float32 [P]})
        the band results are downloaded into it.  Returns the CUDA event that marks
        the results (host or device) complete.  Nothing synchronises the host, so
        consecutive submits pipeline upload, kernels and download."""
        if self.updates == 0:
            raise ParameterError("prime() the first window first")
        if tuple(x_new.shape) != tuple(self._stage[0].shape):
            raise ParameterError(f"expected {tuple(self._stage[0].shape)} new samples, got {tuple(x_new.shape)}")
        u = self.updates
        b = u % self.nbuf
        cs = torch.cuda.current_stream(self.plan.device)
        self._h2d.wait_event(self._ev_used[b])        # the graph that last read stage b is done
        if x_new.is_cuda:
            self._h2d.wait_stream(cs)                 # device input: ordered after its producer
        with torch.cuda.stream(self._h2d):
            self._stage[b].copy_(x_new, non_blocking=True)
            self._ev_in[b].record()
        cs.wait_event(self._ev_in[b])
        cs.wait_event(self._ev_out[b])                # output set b has been downloaded
        self._run(u, b)
        self._ev_used[b].record(cs)
        self._cur = b
        self.updates += 1
        if host_out is None:
            return self._ev_used[b]
        self._d2h.wait_event(self._ev_used[b])
        with torch.cuda.stream(self._d2h):
            for m, h in host_out.items():
                h.copy_(self._outs[b][m]["band"], non_blocking=True)
            self._ev_out[b].record()
        return self._ev_out[b]

    def update(self, x_new: torch.Tensor) -> dict:
        """Append ``n_new`` trials [n_new, N, T] (host or device) and return the
        outputs of the new window (device buffers, stream-ordered on the current
        stream; reused ``buffers`` updates later)."""
        self.submit(x_new)
        return self._outs[self._cur]

    def graph_kernels(self) -> int:
        """Kernels one replay launches (the plan's launch counter over one eager update)."""
        return self._kernels_per_update


class IncrementalWindow:
    """The online sliding window (``update_and_finalize`` every ``n_new`` trials over
    the last ``window``; pipeline.py:304-309, metrics.py:450-460) with the running sums
    moved by the changed trials only (csconn ``cs_window_*``, csrc/window.cu).

    The reference's ``rebuild_last`` re-folds all ``window`` trials per update; the
    fold sums are additive over trials, so each update adds the ``n_new`` trials that
    entered and subtracts the ``n_new`` that left: O(n_new) work per (pair, bin)
    instead of O(window).  A (pair, bin) with a trial inside the fp32 exact-sign error
    bound anywhere in the window is recomputed over the whole window in fp64 (the batch
    path's fallback), and the sums are rebuilt from scratch every ``resync_every``
    updates so fp32 rounding cannot drift.  The plan's ring needs ``window + n_new``
    slots (new trials must not overwrite the ones still to be subtracted).  One CUDA
    graph per (ring phase, buffer) -- K1 on the staging buffer, the sums update, the
    fallback, the band means -- is captured on first use and replayed after; staging
    buffers and output sets are double-buffered so ``submit`` overlaps the next
    window's upload and the previous window's download with the kernels.
    """

    def __init__(self, plan: DevicePlan, window: int, n_new: int, metrics=("PLV", "WPLI"), bin_lo: int = 0,
                 n_bins: int | None = None, dtype=torch.float32, resync_every: int = 256, buffers: int = 2):
        self.plan = plan
        self.window, self.n_new = int(window), int(n_new)
        if not 1 <= self.n_new <= self.window:
            raise ParameterError(f"n_new must be in [1, {self.window}], got {n_new}")
        if plan.slot_capacity < self.window + self.n_new:
            raise ParameterError(f"the plan needs window + n_new = {self.window + self.n_new} slots, "
                                 f"has {plan.slot_capacity}")
        self.cap = plan.slot_capacity
        self.metrics = tuple(m.upper() for m in metrics)
        self.bin_lo = int(bin_lo)
        self.n_bins = plan.n_bins - self.bin_lo if n_bins is None else int(n_bins)
        mask = 0
        for m in self.metrics:
            if m not in METRIC_BITS:
                raise ParameterError(f"{m} is not a spectral metric")
            mask |= 1 << METRIC_BITS[m]
        h = ctypes.c_void_p()
        _lib.check(_lib.lib().cs_window_create(ctypes.byref(h), plan._h, mask, self.bin_lo, self.n_bins))
        self._h = h
        self.nbuf = max(1, int(buffers))
        self._outs, self._descs = [], []
        for _ in range(self.nbuf):
            o = plan.alloc_outputs(self.metrics, self.n_bins, per_bin=True, band=True)
            d = _lib.CsOutputs()
            for m in self.metrics:
                d.bins[METRIC_BITS[m]] = o[m]["bins"].data_ptr()
                d.band[METRIC_BITS[m]] = o[m]["band"].data_ptr()
            d.pair_base = 0
            d.pair_stride = plan.n_pairs
            self._outs.append(o)
            self._descs.append(d)
        self._stage = [torch.empty((self.n_new, plan.n_nodes, plan.n_samples), dtype=dtype, device=plan.device)
                       for _ in range(self.nbuf)]
        self.n_phases = self.cap // math.gcd(self.cap, self.n_new)
        dev = plan.device
        # phase u (window starts at trial u n_new mod cap): changed slots (entering, then leaving)
        # and the window's slots
        self._changed, self._win = [], []
        for u in range(self.n_phases):
            first = (u * self.n_new) % self.cap
            new = [(first + self.window - self.n_new + q) % self.cap for q in range(self.n_new)]
            old = [(first - self.n_new + q) % self.cap for q in range(self.n_new)]
            self._changed.append(torch.tensor(new + old, dtype=torch.int32, device=dev))
            self._win.append(torch.tensor([(first + k) % self.cap for k in range(self.window)], dtype=torch.int32,
                                          device=dev))
        self._graphs: dict[tuple, torch.cuda.CUDAGraph] = {}
        self._kernels_per_update = 0
        self.resync_every = max(1, int(resync_every))
        self.updates = 0
        self._cur = 0
        with torch.cuda.device(dev):
            self._h2d, self._d2h = torch.cuda.Stream(), torch.cuda.Stream()
            self._ev_in = [torch.cuda.Event() for _ in range(self.nbuf)]
            self._ev_used = [torch.cuda.Event() for _ in range(self.nbuf)]
            self._ev_out = [torch.cuda.Event() for _ in range(self.nbuf)]
            for e in self._ev_used + self._ev_out:
                e.record()

    def __del__(self):
        h = getattr(self, "_h", None)
        if h is not None and h.value:
            try:
                _lib.lib().cs_window_destroy(h)
            except Exception:
                pass
            self._h = None

    @property
    def outputs(self) -> dict:
        """Output set of the latest update."""
        return self._outs[self._cur]

    @property
    def staging(self) -> torch.Tensor:
        return self._stage[0]

    def _update_call(self, changed, n_add, n_sub, win, b):
        _lib.check(_lib.lib().cs_window_update(self._h, ctypes.c_void_p(changed.data_ptr()), int(n_add), int(n_sub),
                                               ctypes.c_void_p(win.data_ptr()), self.window,
                                               ctypes.byref(self._descs[b]), _stream_ptr(None)))

    def _resync(self, u: int, b: int) -> None:
        """Sums of the window of phase u from scratch (reset + add every window trial)."""
        _lib.check(_lib.lib().cs_window_reset(self._h, _stream_ptr(None)))
        self._update_call(self._win[u], self.window, 0, self._win[u], b)

    def prime(self, x: torch.Tensor) -> dict:
        """The first ``window`` trials [window, N, T]: K1 into slots 0.., sums from scratch."""
        if x.shape[0] != self.window:
            raise ParameterError(f"prime needs {self.window} trials, got {x.shape[0]}")
        self.plan.spectra(x.to(self.plan.device, non_blocking=True), 0)
        self._resync(0, 0)
        self._ev_used[0].record()
        self._cur = 0
        self.updates = 1
        return self._outs[0]

    def _body(self, u: int, b: int) -> None:
        self.plan.spectra(self._stage[b], (u * self.n_new + self.window - self.n_new) % self.cap)
        self._update_call(self._changed[u], self.n_new, self.n_new, self._win[u], b)

    def _run(self, u: int, b: int) -> None:
        if self.updates % self.resync_every == 0:   # fp32 rounding of the running sums stays bounded
            self.plan.spectra(self._stage[b], (u * self.n_new + self.window - self.n_new) % self.cap)
            self._resync(u, b)
            return
        key = (u, b)
        g = self._graphs.get(key)
        if g is not None:
            g.replay()
            return
        l0 = self.plan.launch_count()
        self._body(u, b)  # eager once per key (this update's sums move here)
        self._kernels_per_update = self.plan.launch_count() - l0
        torch.cuda.current_stream().synchronize()
        prof = self.plan.profiling
        if prof:
            self.plan.set_profiling(False)
        g = torch.cuda.CUDAGraph()
        try:
            with torch.cuda.graph(g):  # capture only: the eager call above applied this update
                self._body(u, b)
        finally:
            if prof:
                self.plan.set_profiling(True)
        self._graphs[key] = g

    def submit(self, x_new: torch.Tensor, host_out: dict | None = None):
        """Append ``n_new`` trials [n_new, N, T] (pinned host or device memory) and enqueue
        the window update; with ``host_out`` ({metric: pinned float32 [P]}) the band means
        are downloaded into it.  Returns the CUDA event marking the results complete;
        nothing synchronises the host."""
        if self.updates == 0:
            raise ParameterError("prime() the first window first")
        if tuple(x_new.shape) != tuple(self._stage[0].shape):
            raise ParameterError(f"expected {tuple(self._stage[0].shape)} new samples, got {tuple(x_new.shape)}")
        u = self.updates % self.n_phases
        b = self.updates % self.nbuf
        cs = torch.cuda.current_stream(self.plan.device)
        self._h2d.wait_event(self._ev_used[b])        # the update that last read stage b is done
        if x_new.is_cuda:
            self._h2d.wait_stream(cs)
        with torch.cuda.stream(self._h2d):
            self._stage[b].copy_(x_new, non_blocking=True)
            self._ev_in[b].record()
        cs.wait_event(self._ev_in[b])
        cs.wait_event(self._ev_out[b])                # output set b has been downloaded
        self._run(u, b)
        self._ev_used[b].record(cs)
        self._cur = b
        self.updates += 1
        if host_out is None:
            return self._ev_used[b]
        self._d2h.wait_event(self._ev_used[b])
        with torch.cuda.stream(self._d2h):
            for m, h in host_out.items():
                h.copy_(self._outs[b][m]["band"], non_blocking=True)
            self._ev_out[b].record()
        return self._ev_out[b]

    def update(self, x_new: torch.Tensor) -> dict:
        """Append ``n_new`` trials [n_new, N, T] (host or device) and return the new
        window's outputs (device buffers, stream-ordered; reused ``buffers`` updates later)."""
        self.submit(x_new)
        return self._outs[self._cur]

    def graph_kernels(self) -> int:
        return self._kernels_per_update
