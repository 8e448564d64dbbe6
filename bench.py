#!/usr/bin/env python3
"""Benchmark of the all-to-all spectral connectivity path (BASELINE.json metric:
edge*freq*trial updates/s).

    python bench.py [--gpus N] [--steps K] [--warmup W] [--config 5] [--impl ours|reference]

A step = one pass of the hot path over one batch: K1 (demean + taper + DFT of
every node x trial) and the fused pair kernels (all 7 metrics, per-bin and
band-averaged outputs) for the configured workload.  Default workload: config 5
(N=10242, K=100, T=1000, Hann, 6 bins), the config BASELINE.json scales over
1/2/4/8 GPUs.  Inputs (4.1 GB) exceed the 126 MB L2, so no explicit flush.

N > 1 (torchrun): rank r owns node block r for K1 and pushes that block of its
fp32 spectrum ring into every peer's ring over NVLink peer memory (CUDA IPC +
copy engines; the path's one exchange step), then computes the pair row-tiles
of its balanced shard (strong scaling; results stay sharded; the fp64 fallback
reads remote nodes' fp64 spectra from their owner by P2P loads).  Timing: CUDA events on the launching stream, barrier + synchronize
on both sides, max over ranks.

--impl reference times the reference's CPU path (the oracle port of
connstream, oracle/) on a bounded node subset of the same workload.
"""
from __future__ import annotations

import argparse
import json
import math
import os
import statistics
import subprocess
import sys
import threading
import time
from pathlib import Path

ROOT = Path(__file__).resolve().parent
sys.path.insert(0, str(ROOT))

import numpy as np  # noqa: E402
import torch  # noqa: E402


def _peaks():
    p = ROOT / "MEASURED_PEAKS.json"
    if p.exists():
        d = json.loads(p.read_text())
        return d, "measured"
    return {"hbm_gbs": 6650.0, "bf16_tflops": 1590.0, "bf16_tflops_sustained": 1400.0}, "fallback"


def _ncu_traffic(cfg: int, kernel, ws: int):
    """dram bytes per launch of ``kernel`` at config ``cfg`` from the committed ncu capture
    (profiles/ncu_traffic.json, written from an `ncu --set full` run of this bench)."""
    p = ROOT / "profiles" / "ncu_traffic.json"
    if kernel is None or ws != 1 or not p.exists():
        return None
    for e in json.loads(p.read_text()).get("entries", []):
        if e.get("config") == cfg and kernel.startswith(e.get("kernel", "?")):
            return e
    return None


class ClockSampler:
    """SM clock + throttle reasons sampled during the timed region: NVML polled every
    5 ms from a thread (so timed regions of a few tens of ms still get samples), or
    `nvidia-smi -lms 50` when NVML is unavailable."""

    Q = ("clocks.sm,clocks.max.sm,clocks_event_reasons.active,clocks_event_reasons.hw_slowdown,"
         "clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,"
         "clocks_event_reasons.sw_power_cap")
    NAMES = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]

    def __init__(self, gpu_index: int):
        self.idx = gpu_index
        self.proc = None
        self.lines = []
        self.samples = []        # NVML: (sm_mhz, reasons bitmask)
        self.nv = None

    def _nvml_handle(self):
        import pynvml
        pynvml.nvmlInit()
        try:   # the CUDA ordinal need not be the NVML index: match by PCI bus id
            pr = torch.cuda.get_device_properties(self.idx)
            bus = f"{pr.pci_domain_id:08X}:{pr.pci_bus_id:02X}:{pr.pci_device_id:02X}.0"
            return pynvml, pynvml.nvmlDeviceGetHandleByPciBusId(bus)
        except Exception:
            return pynvml, pynvml.nvmlDeviceGetHandleByIndex(self.idx)

    def __enter__(self):
        try:
            nv, h = self._nvml_handle()
            self.nv, self.h = nv, h
            self.max_mhz = float(nv.nvmlDeviceGetMaxClockInfo(h, nv.NVML_CLOCK_SM))
            self.bits = {"hw_slowdown": nv.nvmlClocksThrottleReasonHwSlowdown,
                         "hw_thermal_slowdown": nv.nvmlClocksThrottleReasonHwThermalSlowdown,
                         "sw_thermal_slowdown": nv.nvmlClocksThrottleReasonSwThermalSlowdown,
                         "sw_power_cap": nv.nvmlClocksThrottleReasonSwPowerCap}
            self.stop = threading.Event()
            self._t = threading.Thread(target=self._poll, daemon=True)
            self._t.start()
            return self
        except Exception:
            self.nv = None
        try:
            self.proc = subprocess.Popen(["nvidia-smi", "-i", str(self.idx), f"--query-gpu={self.Q}",
                                          "--format=csv,noheader,nounits", "-lms", "50"],
                                         stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            self._t = threading.Thread(target=self._read, daemon=True)
            self._t.start()
            # nvidia-smi takes a moment to start: wait for its first sample and drop it, so
            # the kept samples fall inside the timed region that starts after __enter__
            t0 = time.time()
            while not self.lines and time.time() - t0 < 3.0 and self.proc.poll() is None:
                time.sleep(0.01)
            self.lines.clear()
        except OSError:
            self.proc = None
        return self

    def _poll(self):
        nv, h = self.nv, self.h
        while not self.stop.is_set():
            try:
                self.samples.append((float(nv.nvmlDeviceGetClockInfo(h, nv.NVML_CLOCK_SM)),
                                     int(nv.nvmlDeviceGetCurrentClocksEventReasons(h))))
            except Exception:
                return
            self.stop.wait(0.005)

    def _read(self):
        for line in self.proc.stdout:
            self.lines.append(line.strip())

    def __exit__(self, *a):
        if self.nv is not None:
            self.stop.set()
            self._t.join(timeout=1.0)
        if self.proc is not None:
            self.proc.terminate()
            try:
                self.proc.wait(timeout=5)
            except subprocess.TimeoutExpired:
                self.proc.kill()

    def summary(self):
        sm, mx, reasons = [], None, set()
        if self.nv is not None:
            for mhz, r in self.samples:
                sm.append(mhz)
                reasons.update(n for n, bit in self.bits.items() if r & bit)
            mx = self.max_mhz
        for ln in self.lines:
            f = [x.strip() for x in ln.split(",")]
            if len(f) < 7:
                continue
            try:
                sm.append(float(f[0]))
                mx = float(f[1])
            except ValueError:
                continue
            for n, v in zip(self.NAMES, f[3:7]):
                if v.lower().startswith("active"):
                    reasons.add(n)
        if not sm:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["no samples"]}
        return {"sm_mhz": statistics.median(sm), "sm_max_mhz": mx, "reasons": sorted(reasons),
                "samples": len(sm), "source": "nvml 5 ms" if self.nv is not None else "nvidia-smi 50 ms"}


def dist_setup():
    ws = int(os.environ.get("WORLD_SIZE", "1"))
    if ws > 1:
        os.environ.setdefault("MASTER_ADDR", "127.0.0.1")
        import torch.distributed as dist
        lr = int(os.environ.get("LOCAL_RANK", "0"))
        # BENCH_DEVICE_OF_RANK=0 + BENCH_BACKEND=gloo: a host-side smoke test of the N > 1
        # path with every rank on one GPU (collectives staged through host memory, so no
        # kernel of one rank waits on another's); timings from such a run are not scaling
        dev_idx = int(os.environ.get("BENCH_DEVICE_OF_RANK", lr))
        torch.cuda.set_device(dev_idx)
        backend = os.environ.get("BENCH_BACKEND", "nccl")
        if backend == "nccl":
            dist.init_process_group("nccl", device_id=torch.device("cuda", dev_idx))
        else:
            dist.init_process_group(backend)
        return dist, dist.get_rank(), ws, dev_idx
    torch.cuda.set_device(0)
    return None, 0, 1, 0


CPU_NODES = 512  # node subset of the CPU legs (the reference arm and cpu_baseline use the same sample)


def metric_name(c) -> str:
    """The metric string both arms print (the driver divides the two values only when
    metric, unit and direction agree)."""
    if c.cfg == 4:
        return "edge*freq*trial updates/s per online window (config 4, PLV + WPLI)"
    return f"edge*freq*trial updates/s (config {c.cfg}, {len(c.metrics)} metrics)"


def cpu_baseline(c, n_sub: int, threads: int):
    """The reference's CPU path (oracle port, oracle/) on a node subset of the
    workload: per-trial spectra through a thread pool (as compute_metric does,
    metrics.py:542-547) and the single-threaded fold + 7 finalizers."""
    import oracle as O
    from concurrent.futures import ThreadPoolExecutor
    from paper_2303_03279_b200 import synth
    from paper_2303_03279_b200.plan import make_taper
    dev = "cuda" if torch.cuda.is_available() else "cpu"
    x = synth.generate(c, dev, nodes=slice(0, n_sub)).double().cpu().numpy()
    tap = make_taper(c.taper, min(c.T, c.nfft))
    t0 = time.perf_counter()
    with ThreadPoolExecutor(max_workers=threads) as pool:
        if tap is not None and tap.shape[0] > 1:
            specs = list(pool.map(lambda e: np.stack([O.trial_spectra(e, c.nfft, tp)[:, c.lo:c.hi + 1]
                                                      for tp in tap]), x))
        else:
            tp = None if tap is None else tap[0]
            specs = list(pool.map(lambda e: O.trial_spectra(e, c.nfft, tp)[:, c.lo:c.hi + 1], x))
    t1 = time.perf_counter()
    acc = O.Sums(n_sub, c.n_bins)
    for s in specs:
        if s.ndim == 3:
            O.accumulate_multitaper(acc, s)
        else:
            O.accumulate(acc, s)
    t2 = time.perf_counter()
    for m in c.metrics:
        O.band_reduce(m, O.BINS[m](acc))
    t3 = time.perf_counter()
    upd = n_sub * (n_sub - 1) // 2 * c.n_bins * c.K
    return {"updates": upd, "s": t3 - t0, "fft_s": t1 - t0, "fold_s": t2 - t1, "finalize_s": t3 - t2}


def run_reference(args, c, rank):
    if rank != 0:
        return
    threads = os.cpu_count() or 1
    n_sub = min(args.cpu_nodes or CPU_NODES, c.N)  # cfg5: ~3 s per step, the whole run stays within minutes
    samples = []
    for i in range(args.warmup + args.steps):
        r = cpu_baseline(c, n_sub, threads)
        if i >= args.warmup:
            samples.append(r)
    s = statistics.mean(r["s"] for r in samples)
    val = samples[0]["updates"] / s
    line = {
        "impl": "reference", "metric": metric_name(c), "value": val,
        "unit": "updates/s", "n_gpus": args.gpus, "steps": args.steps, "warmup": args.warmup,
        "ms_per_step": s * 1e3, "higher_is_better": True, "scaling": "strong", "vs_baseline": None,
        "dtype": "f64", "data": "synthetic (seeded; SURVEY.md 8(d) signal model)",
        "config": {"workload": f"cfg{c.cfg}: {c.name}", "sample_nodes": n_sub},
        "cpu_baseline": {"value": val, "unit": "updates/s", "cores": threads, "kind": "port",
                         "sample": f"node subset N'={n_sub} of cfg{c.cfg} (all K={c.K} trials, {c.n_bins} bins); "
                                   "FFT in a thread pool, fold single-threaded as in the reference",
                         "breakdown_s": {k: statistics.mean(r[k] for r in samples) for k in ("fft_s", "fold_s", "finalize_s")}},
        "e2e": {"value": val, "unit": "updates/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)


def run_window(args, c, dist, rank, ws, lr):
    """Config 4: online sliding window.  A stream of 1045 trials, window w =
    trials [5w, 5w + 50): per window K1 runs on the 5 new trials only (cached
    spectra of the other 45 are reused from the HBM ring) and PLV and WPLI are
    produced over the window's 50 trials -- the work the reference's
    rebuild_last(50) performs (metrics.py:450-460, pipeline.py:304-309), counted
    as P nb 50 updates per window.  The timed path is the incremental window
    (plan.IncrementalWindow, csrc/window.cu): the running sums move by the 5
    entering and 5 leaving trials, risky (pair, bin) entries are recomputed over
    the window in fp64, one CUDA-graph replay per window.  The full re-fold of
    every window (plan.WindowGraph, the reference's semantics executed literally)
    is timed beside it as ``full_recompute``.  Replicas only at N > 1."""
    from paper_2303_03279_b200 import synth
    from paper_2303_03279_b200.plan import DevicePlan, IncrementalWindow, WindowGraph, pow2_scale, probe_peaks
    dev = torch.device("cuda", lr)
    win, new = 50, 5
    W = min(synth.CFG4_WINDOWS, max(args.warmup, 11) + args.steps + 1)  # windows of the stream
    n_trials = new * (W - 1) + win
    x = synth.generate(c, dev, trials=range(n_trials))            # [n_trials, N, T] resident in HBM
    scale = pow2_scale(float(x.abs().amax()), min(c.T, c.nfft))

    def barrier():
        if dist is not None:
            dist.barrier()
        torch.cuda.synchronize()

    def max_over_ranks(v: float) -> float:
        if dist is None:
            return v
        t = torch.tensor([v], dtype=torch.float64, device=dev if dist.get_backend() == "nccl" else "cpu")
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        return float(t)

    def new_trials(w):  # trials [5w + 45, 5w + 50) of window w (cycling over the generated stream)
        w = 1 + (w - 1) % (W - 1)
        return x[new * w + win - new: new * w + win]

    def time_windows(runner, warm):
        for w in range(1, 1 + warm):
            runner.update(new_trials(w))
        barrier()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        with ClockSampler(lr) as clk:
            barrier()
            e0.record()
            for w in range(1 + warm, 1 + warm + args.steps):
                runner.update(new_trials(w))
            e1.record()
            barrier()
        return max_over_ranks(e0.elapsed_time(e1) / args.steps), clk.summary()

    # the timed online path: incremental sums
    plan_i = DevicePlan(c.N, c.T, c.nfft, c.lo, c.hi, taper=c.taper, slot_capacity=win + new, device=dev, scale=scale)
    iw = IncrementalWindow(plan_i, win, new, c.metrics)
    iw.prime(x[0:win])
    warm_i = max(args.warmup, 2 * iw.n_phases)          # every (phase, buffer) graph captured
    ms, clk = time_windows(iw, warm_i)
    launches = iw.graph_kernels() * args.steps
    # e2e: each window's 5 new trials from pinned host memory, band results back to the host
    n_e2e = min(args.steps, 500)
    xh = x[: new * (W - 1) + win].cpu().pin_memory()
    hb = {m: torch.empty(c.n_pairs, dtype=torch.float32).pin_memory() for m in c.metrics}
    barrier()
    f0, f1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    f0.record()
    for w in range(1 + warm_i, 1 + warm_i + n_e2e):   # back to back: upload / kernels / download overlap
        wi = 1 + (w - 1) % (W - 1)
        ev = iw.submit(xh[new * wi + win - new: new * wi + win], hb)
    torch.cuda.current_stream().wait_event(ev)
    f1.record()
    barrier()
    e2e_ms = max_over_ranks(f0.elapsed_time(f1) / n_e2e)
    # per-kernel breakdown from an eager profiled pass (graphs are not profiled per kernel)
    plan_i.set_profiling(True)
    plan_i.profile()
    n_prof = min(args.steps, 10)
    for w in range(1, 1 + n_prof):
        iw._body(iw.updates % iw.n_phases, 0)
        iw.updates += 1
    prof = plan_i.profile()
    plan_i.set_profiling(False)
    per = {k: v[0] / max(v[1], 1) for k, v in prof.items()}
    del iw, plan_i

    # the full re-fold of every window, for comparison
    plan_f = DevicePlan(c.N, c.T, c.nfft, c.lo, c.hi, taper=c.taper, slot_capacity=win, device=dev, scale=scale)
    wg = WindowGraph(plan_f, new, c.metrics, 0, c.n_bins)
    wg.prime(x[0:win])
    ms_full, _ = time_windows(wg, max(args.warmup, 2 * wg.n_phases))
    del wg, plan_f

    upd = c.n_pairs * c.n_bins * win
    fp32_ops, fp64_fma = probe_peaks(lr)
    line = {"metric": metric_name(c),
            "value": ws * upd / (ms * 1e-3),
            "unit": "updates/s", "ms_per_window": ms, "n_gpus": ws, "steps": args.steps, "warmup": args.warmup,
            "ms_per_step": ms, "higher_is_better": True, "scaling": "weak" if ws > 1 else "strong",
            "vs_baseline": None, "dtype": "f32", "data": "synthetic (seeded; SURVEY.md 8(d) cfg4 pink noise + planted 20 Hz)",
            "config": {"workload": f"cfg{c.cfg}: {c.name}", "N": c.N, "window": win, "new_trials_per_window": new,
                       "bins": [c.lo, c.hi], "metrics": list(c.metrics), "parallelism": f"replicas x{ws}",
                       "updates_per_window": upd,
                       "path": "incremental window sums (+5 entering, -5 leaving trials; fp64 re-fold of risky "
                               "entries), one CUDA-graph replay per window"},
            "full_recompute": {"ms_per_window": ms_full, "updates_per_s": ws * upd / (ms_full * 1e-3),
                               "path": "WindowGraph: the pair kernels re-fold all 50 trials every window"},
            "breakdown": {k: {"ms_per_launch": round(v, 4), "launches": prof[k][1]} for k, v in per.items()},
            "breakdown_note": "eager profiled pass over the same windows; the timed region replays CUDA graphs",
            "gpu_launches": launches, "clocks": clk,
            "e2e": {"value": ws * upd / (e2e_ms * 1e-3), "unit": "updates/s", "ms_per_window": e2e_ms,
                    "windows": n_e2e,
                    "h2d_bytes_per_step": int(new * c.N * c.T * 4) * ws,
                    "d2h_bytes_per_step": int(sum(v.numel() * 4 for v in hb.values())) * ws,
                    "path": "IncrementalWindow.submit(pinned host trials, pinned host band buffers): H2D into a "
                            "double-buffered staging buffer, graph replay, band results D2H, on three streams "
                            "so consecutive windows overlap"},
            "peaks": {"fp32_lane_ops_per_s": fp32_ops, "fp64_dfma_per_s": fp64_fma}}
    if rank == 0:
        print(json.dumps(line), flush=True)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=None,
                    help="timed steps (default 50; cfg1/2/4: 4000/1000/3000 so the timed region is ~0.5 s)")
    ap.add_argument("--warmup", type=int, default=5)
    ap.add_argument("--config", type=int, default=5)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--metrics", default=None, help="comma list (default: the config's metrics)")
    ap.add_argument("--cpu-nodes", type=int, default=None,
                    help=f"node subset of the CPU legs (default {CPU_NODES}, both arms)")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--e2e-steps", type=int, default=10)
    ap.add_argument("--no-per-metric", action="store_true", help="skip the one-metric-at-a-time runs")
    args = ap.parse_args()
    if args.steps is None:  # timed regions of >= ~0.5 s, so nvidia-smi samples the clocks in them
        args.steps = {1: 4000, 2: 1000, 4: 3000}.get(args.config, 50) if args.impl == "ours" else 50

    from paper_2303_03279_b200 import synth
    c = synth.CONFIGS[args.config]
    if args.impl == "reference":
        rank = int(os.environ.get("RANK", "0"))
        run_reference(args, c, rank)
        return

    from paper_2303_03279_b200.plan import DevicePlan, pow2_scale, probe_peaks
    dist, rank, ws, lr = dist_setup()
    if c.cfg == 4:
        run_window(args, c, dist, rank, ws, lr)
        return
    dev = torch.device("cuda", lr)
    metrics = tuple(args.metrics.split(",")) if args.metrics else c.metrics

    # ---- node block for K1, pair shard for the pair kernels ----
    from paper_2303_03279_b200.shard import RingExchange, node_block, shard_plan
    n0, n1, nloc = node_block(c.N, ws, rank)
    (rb, re), (p0, p1) = shard_plan(c.N, ws, rank)
    x = synth.generate(c, dev, nodes=slice(n0, n1))
    amax = x.abs().amax()
    if dist is not None:
        dist.all_reduce(amax, op=dist.ReduceOp.MAX)
    scale = pow2_scale(float(amax), min(c.T, c.nfft))
    # N > 1: the ring holds two steps (slots [0, K) and [K, 2K) alternate), so a step's K1
    # and push never overwrite slots a peer's fallback of the previous step may still read
    full = DevicePlan(c.N, c.T, c.nfft, c.lo, c.hi, taper=c.taper, slot_capacity=c.K * (2 if ws > 1 else 1),
                      device=dev, scale=scale)
    ex = RingExchange(full, dist) if ws > 1 else None
    slot_sets = [torch.arange(h * c.K, (h + 1) * c.K, dtype=torch.int32, device=dev) for h in range(2 if ws > 1 else 1)]
    outs = full.alloc_outputs(metrics, c.n_bins, per_bin=True, band=True, pair_count=p1 - p0)
    n_step = [0]

    def exchange(h):
        """K1 on this rank's node block, then the ring exchange (the path's one exchange step):
        push the block into every peer's ring, wait for this rank's pushes, host barrier."""
        if ex is None:
            full.spectra(x, 0)
            return
        ex.spectra(x, h * c.K)
        ex.push(h * c.K, c.K)
        torch.cuda.current_stream().synchronize()
        dist.barrier()

    def step():
        h = n_step[0] % len(slot_sets)
        n_step[0] += 1
        exchange(h)
        full.pair_metrics(slot_sets[h], metrics, 0, c.n_bins, outputs=outs, row_tiles=(rb, re), pair_base=p0,
                          pair_count=p1 - p0)

    def barrier():
        if dist is not None:
            dist.barrier()
        torch.cuda.synchronize()

    for _ in range(args.warmup):
        step()
    barrier()
    n_fallback = full.fallback_count()
    full.set_profiling(True)
    full.profile()
    launches0 = full.launch_count()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    with ClockSampler(lr) as clk:
        barrier()
        e0.record()
        for _ in range(args.steps):
            step()
        e1.record()
        barrier()
    ms = e0.elapsed_time(e1)
    prof = full.profile()
    launches = full.launch_count() - launches0
    ms_t = torch.tensor([ms], device=dev)
    if dist is not None:
        dist.all_reduce(ms_t, op=dist.ReduceOp.MAX)
    ms_max = float(ms_t)
    ms_step = ms_max / args.steps
    value = c.updates / (ms_step * 1e-3)

    # ---- roofline of the dominant kernel ----
    peaks, peak_kind = _peaks()
    fp32_ops, fp64_fma = probe_peaks(lr)
    per = {k: v[0] / max(v[1], 1) for k, v in prof.items()}  # ms per launch
    dom = max(per, key=per.get)
    lag_ms = per.get("pairs_lag", 0.0)
    spec_key = "spectra"
    roof = roof_k3 = roof_k1 = None
    if lag_ms > 0:
        # algorithmic FP32-pipe work per update (trial): t = sum over L tapers of FMUL+FFMA (2L),
        # sum t (1), sum |t| (1); multitaper PLV (not separable) adds Re of the
        # taper-mean CSD (2L), |CSD|^2 (2) and the phasor accumulation (2)
        P_loc = p1 - p0
        upd = P_loc * c.n_bins * c.K
        L_k3 = 1 if not isinstance(c.taper, tuple) else c.taper[2]
        plv_k3 = L_k3 > 1 and "PLV" in metrics
        # IMAGCOHY hand-off (cs_last_imag_handoff): sum t comes from the tensor-core D_im
        handoff = full.guard_stats()["imag_handoff"]
        w_upd = 2 * L_k3 + (1 if handoff else 2) + ((2 * L_k3 + 4) if plv_k3 else 0)
        ach = w_upd * upd / (lag_ms * 1e-3)
        roof_k3 = {"kernel": "k_pairs_lag", "bound": "fp32", "achieved": ach / 1e12, "peak": fp32_ops / 1e12,
                "unit": "T FP32-pipe lane-ops/s", "frac": ach / fp32_ops, "traffic": None,
                "peak_source": "measured live on this GPU by cs_probe_peaks (dependent FFMA chains)",
                "work_per_update": (f"{w_upd} FP32 lane-ops: t over {L_k3} taper(s) {2 * L_k3}, "
                                    + ("sum |t| 1 (sum t: IMAGCOHY hand-off from k_pairs_tc)" if handoff
                                       else "sum t 1, sum |t| 1")
                                    + (f", multitaper PLV {2 * L_k3 + 4}" if plv_k3 else ""))}
        # the same kernel on SURVEY.md 8(d)'s own basis: FP32 instructions per update (t = FMUL +
        # FFMA per taper, sum of signs, sum |Im|, sum Im unless handed over) at the nominal
        # 148 x 128 x 1.965 GHz = 3.72e13 instr/s, or the output bytes at HBM, whichever is longer
        if not plv_k3:
            n_instr = 2 * L_k3 + 2 + (0 if handoff else 1)
            t_issue = n_instr * upd / 3.72e13
            t_out = 16.0 * P_loc * (c.n_bins + 1) / (peaks["hbm_gbs"] * 1e9)
            roof_k3["survey_8d"] = {"instr_per_update": n_instr, "bound_ms": max(t_issue, t_out) * 1e3,
                                    "frac": max(t_issue, t_out) / (lag_ms * 1e-3)}
    if per.get(spec_key, 0.0) > 0:
        k1_ms = per[spec_key]
        L_ = 1 if not isinstance(c.taper, tuple) else c.taper[2]
        kind = full.k1_kind
        if kind.startswith("fft"):   # 5 M log2 M + 16 M fp64 flops per signal-taper, M = nfft / 2 (2 flops per DFMA)
            M_ = c.nfft // 2
            fma = c.K * nloc * L_ * (5 * M_ * math.log2(M_) + 16 * M_) / 2
            work = "fp64 FMA-equivalents of a 5 M log2 M + 16 M real-input FFT"
        else:                        # direct DFT: 2 FMA per sample and plan bin
            fma = c.K * nloc * L_ * min(c.T, c.nfft) * c.n_bins * 2
            work = "2 fp64 FMA per sample and plan bin"
        bytes_ = c.K * nloc * c.T * x.element_size() + c.K * nloc * L_ * c.n_bins * 24
        roof_k1 = {"kernel": "k_spectra", "k1_kind": kind, "bound": "fp64", "achieved": fma / (k1_ms * 1e-3) / 1e12,
                "peak": fp64_fma / 1e12, "unit": "T FP64 FMA/s", "frac": fma / (k1_ms * 1e-3) / fp64_fma,
                "traffic": None, "hbm_frac": bytes_ / (k1_ms * 1e-3) / (peaks["hbm_gbs"] * 1e9),
                "work": work}
    roof = roof_k3 if dom.endswith("pairs_lag") else (roof_k1 if dom.endswith("spectra") else None)
    # dram traffic per launch from the committed ncu --set full capture (same config)
    for rf in (roof_k1, roof_k3):
        if rf is not None:
            tr = _ncu_traffic(c.cfg, rf["kernel"], ws)
            rf["traffic"] = tr["bytes_per_launch"] if tr else None
            if tr:
                rf["traffic_source"] = tr["source"]
    # K2 (tensor cores): SURVEY 8(d) roofline = max(3 x flops / bf16 (burst), output bytes / HBM)
    roof_k2 = None
    tc_ms = per.get("pairs_tc", 0.0)
    if tc_ms > 0:
        L = 1 if not isinstance(c.taper, tuple) else c.taper[2]
        P_loc = p1 - p0
        flops = 8.0 * c.K * L * P_loc * c.n_bins + (8.0 * c.K * P_loc * c.n_bins if ("PLV" in metrics and L == 1) else 0.0)
        n_out = sum(m in metrics for m in ("COH", "IMAGCOHY", "PLV", "COHY"))
        out_bytes = 4.0 * n_out * P_loc * (c.n_bins + 1)
        # burst peak: the timed region runs at the maximum SM clock (the clocks line shows it)
        t_tc = 3.0 * flops / (peaks["bf16_tflops"] * 1e12)
        t_hbm = out_bytes / (peaks["hbm_gbs"] * 1e9)
        bound = "tensor" if t_tc >= t_hbm else "hbm"
        roof_k2 = {"kernel": "k_pairs_tc", "bound": bound,
                   "achieved": (3.0 * flops / (tc_ms * 1e-3) / 1e12) if bound == "tensor" else out_bytes / (tc_ms * 1e-3) / 1e9,
                   "peak": peaks["bf16_tflops"] if bound == "tensor" else peaks["hbm_gbs"],
                   "unit": "TFLOP/s (bf16x3-equivalent)" if bound == "tensor" else "GB/s",
                   "frac": max(t_tc, t_hbm) / (tc_ms * 1e-3),
                   "raw_tflops": flops / (tc_ms * 1e-3) / 1e12, "ms": tc_ms,
                   "note": "fp16 hi/lo split = 3 products per real product; frac = roofline time / measured time"}
    if roof_k2 is not None:
        tr = _ncu_traffic(c.cfg, "k_pairs_tc", ws)
        roof_k2["traffic"] = tr["bytes_per_launch"] if tr else None
        if tr:
            roof_k2["traffic_source"] = tr["source"]
    if roof is None and dom.endswith("pairs_tc"):
        roof = roof_k2
    breakdown = {k: {"ms_per_launch": round(v[0] / max(v[1], 1), 4), "launches": v[1]} for k, v in prof.items()}

    # ---- network post-processing on the device over the COH band weights ----
    post = None
    if "COH" in metrics and ws == 1:
        import ctypes as _ct
        from paper_2303_03279_b200 import _lib as L_
        wband = outs["COH"]["band"]
        wcopy = wband.clone()
        P_all = wband.numel()
        keep = int(np.ceil(0.05 * P_all))
        idx = torch.empty(keep, dtype=torch.int64, device=dev)
        sp = _ct.c_void_p(torch.cuda.current_stream().cuda_stream)
        for _ in range(2):
            L_.check(L_.lib().cs_net_normalize(_ct.c_void_p(wcopy.data_ptr()), None, P_all, sp))
            L_.check(L_.lib().cs_net_threshold(_ct.c_void_p(wcopy.data_ptr()), P_all, keep, _ct.c_void_p(idx.data_ptr()), sp))
        torch.cuda.synchronize()
        tn, tt = [], []
        for _ in range(5):
            a, b, c2 = (torch.cuda.Event(enable_timing=True) for _ in range(3))
            a.record()
            L_.check(L_.lib().cs_net_normalize(_ct.c_void_p(wcopy.data_ptr()), None, P_all, sp))
            b.record()
            L_.check(L_.lib().cs_net_threshold(_ct.c_void_p(wcopy.data_ptr()), P_all, keep, _ct.c_void_p(idx.data_ptr()), sp))
            c2.record()
            torch.cuda.synchronize()
            tn.append(a.elapsed_time(b))
            tt.append(b.elapsed_time(c2))
        post = {"edges": P_all, "keep_fraction": 0.05, "normalize_ms": float(np.median(tn)),
                "threshold_ms": float(np.median(tt)),
                "threshold_gbs": 5 * 4.0 * P_all / (float(np.median(tt)) * 1e-3) / 1e9,
                "note": "device normalize (max |w| + scale) and top-k threshold (4 radix passes + count + ordered compaction) on the cfg5 COH band weights"}
        del wcopy, idx

    # ---- per metric: each metric alone with K1 + only the kernel it needs ----
    per_metric = None
    if not args.no_per_metric and len(metrics) > 1:
        full.set_profiling(False)
        per_metric = {}
        n_pm = max(3, min(args.steps, 10))
        for m in metrics:
            om = full.alloc_outputs((m,), c.n_bins, per_bin=True, band=True, pair_count=p1 - p0)

            def step_m():
                h = n_step[0] % len(slot_sets)
                n_step[0] += 1
                exchange(h)
                full.pair_metrics(slot_sets[h], (m,), 0, c.n_bins, outputs=om, row_tiles=(rb, re), pair_base=p0,
                                  pair_count=p1 - p0)
            for _ in range(2):
                step_m()
            barrier()
            e0.record()
            for _ in range(n_pm):
                step_m()
            e1.record()
            barrier()
            tm = torch.tensor([e0.elapsed_time(e1) / n_pm], device=dev)
            if dist is not None:
                dist.all_reduce(tm, op=dist.ReduceOp.MAX)
            per_metric[m] = {"updates_per_s": c.updates / (float(tm) * 1e-3), "ms_per_step": float(tm)}
            del om

    line = {
        "metric": metric_name(c) if tuple(metrics) == tuple(c.metrics) else
        f"edge*freq*trial updates/s (config {c.cfg}, {len(metrics)} metrics)",
        "value": value, "unit": "updates/s", "n_gpus": ws, "steps": args.steps, "warmup": args.warmup,
        "ms_per_step": ms_step, "higher_is_better": True, "scaling": "strong", "vs_baseline": None,
        "dtype": "f32", "data": "synthetic (seeded; SURVEY.md 8(d) signal model, no public dataset)",
        "config": {"workload": f"cfg{c.cfg}: {c.name}", "N": c.N, "K": c.K, "T": c.T, "nfft": c.nfft,
                   "bins": [c.lo, c.hi], "taper": str(c.taper), "metrics": list(metrics),
                   "outputs": "per-bin [nb,P] + band-mean [P] per metric", "parallelism": f"pair-row-tiles x{ws}",
                   "l2": "inputs 4.1 GB > 126 MB L2 (no flush needed)" if c.cfg == 5 else "inputs > L2" ,
                   "updates_per_step": c.updates},
        "roofline": roof, "roofline_k1": roof_k1, "roofline_k2": roof_k2, "roofline_k3": roof_k3,
        "per_metric": per_metric, "post_processing": post,
        "breakdown": breakdown, "fp64_fallback_entries": n_fallback,
        "gpu_launches": launches, "clocks": clk.summary(),
        "peaks": {"fp32_lane_ops_per_s": fp32_ops, "fp64_dfma_per_s": fp64_fma, "hbm_gbs": peaks["hbm_gbs"],
                  "hbm_source": peak_kind},
    }

    # ---- e2e through the public API with host buffers ----
    if not args.no_e2e and ws == 1:
        # HostPipeline.submit: pinned host samples -> H2D (trial chunks, overlapping K1) ->
        # pair kernels (row chunks, each downloaded while the next runs) -> pinned host band
        # means; consecutive steps are enqueued back to back, so step s+1's upload overlaps
        # step s's pair kernels and download.  Every step's copies are inside the timed region.
        from paper_2303_03279_b200.plan import HostPipeline, bind_host_to_gpu_numa, copy_ceilings
        del outs
        torch.cuda.empty_cache()
        aff0 = os.sched_getaffinity(0)
        numa = bind_host_to_gpu_numa(lr)   # pinned buffers below land on the GPU's NUMA node
        hp = HostPipeline(c.N, c.T, c.nfft, c.lo, c.hi, c.K, metrics=metrics, taper=c.taper, scale=scale,
                          device=dev, dtype=x.dtype)
        xh = x.cpu().pin_memory()
        hb = hp.alloc_host()
        hp.run(xh, hb)  # warm-up (tile lists, operand buffers)
        torch.cuda.synchronize()
        e0.record(hp.s_in)
        for _ in range(args.e2e_steps):
            done = hp.submit(xh, hb)
        torch.cuda.current_stream().wait_event(done)
        e1.record()
        torch.cuda.synchronize()
        t_ms = e0.elapsed_time(e1) / args.e2e_steps
        d2h = sum(v.numel() * v.element_size() for v in hb.values())
        del xh, hb
        ceil = copy_ceilings(hp.h2d_bytes, d2h, dev)
        copy_ms = max(hp.h2d_bytes / (ceil["h2d_gbs"] * 1e9), d2h / (ceil["d2h_gbs"] * 1e9), ceil["bidir_ms"] * 1e-3) * 1e3
        line["e2e"] = {"value": c.updates / (t_ms * 1e-3), "unit": "updates/s",
                       "h2d_bytes_per_step": hp.h2d_bytes,
                       "d2h_bytes_per_step": d2h,
                       "ms_per_step": t_ms, "steps": args.e2e_steps,
                       "h2d_ceiling_gbs": ceil["h2d_gbs"], "d2h_ceiling_gbs": ceil["d2h_gbs"],
                       "bidir_copy_ms": ceil["bidir_ms"],
                       "copy_bound_ms": copy_ms, "frac_of_copy_bound": copy_ms / t_ms,
                       "numa": None if numa is None else {"node": numa[0], "cpus": numa[1]},
                       "path": "HostPipeline.submit: pinned host samples -> H2D in trial chunks (overlapping K1) -> "
                               "pair kernels over row-tile chunks -> band means D2H per chunk; steps enqueued "
                               "back to back (step s+1 upload overlaps step s kernels + download)"}
        os.sched_setaffinity(0, aff0)   # the CPU baseline below uses every host core again
    elif not args.no_e2e:
        # N > 1: every rank uploads its node block, runs K1, pushes it into the peers' rings,
        # runs its pair rows and downloads its band means; uploads and downloads run on copy
        # streams so step s+1's upload overlaps step s's kernels and download (event-ordered)
        xh = x.cpu().pin_memory()
        hb = {m: torch.empty(p1 - p0, dtype=torch.float32).pin_memory() for m in metrics}
        xd = torch.empty_like(x)
        s_in, s_out = torch.cuda.Stream(dev), torch.cuda.Stream(dev)
        ev_in, ev_k1, ev_pm, ev_out = (torch.cuda.Event() for _ in range(4))
        cur = torch.cuda.current_stream(dev)
        for ev in (ev_k1, ev_out):
            ev.record(cur)

        def e2e_step():
            h = n_step[0] % len(slot_sets)
            n_step[0] += 1
            s_in.wait_event(ev_k1)                 # the previous K1 has consumed xd
            with torch.cuda.stream(s_in):
                xd.copy_(xh, non_blocking=True)
                ev_in.record(s_in)
            cur.wait_event(ev_in)
            ex.spectra(xd, h * c.K)
            ev_k1.record(cur)
            ex.push(h * c.K, c.K)
            cur.synchronize()
            dist.barrier()
            cur.wait_event(ev_out)                 # the previous download has read the outputs
            o = full.pair_metrics(slot_sets[h], metrics, 0, c.n_bins, per_bin=False, band=True,
                                  row_tiles=(rb, re), pair_base=p0, pair_count=p1 - p0)
            ev_pm.record(cur)
            s_out.wait_event(ev_pm)
            with torch.cuda.stream(s_out):
                for m in metrics:
                    hb[m].copy_(o[m]["band"], non_blocking=True)
                ev_out.record(s_out)
        e2e_step()
        barrier()
        full.set_profiling(False)
        barrier()
        e0.record()
        for _ in range(args.e2e_steps):
            e2e_step()
        cur.wait_event(ev_out)
        e1.record()
        barrier()
        t = torch.tensor([e0.elapsed_time(e1) / args.e2e_steps], device=dev)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        line["e2e"] = {"value": c.updates / (float(t) * 1e-3), "unit": "updates/s",
                       "h2d_bytes_per_step": xh.numel() * xh.element_size() * ws,
                       "d2h_bytes_per_step": sum(v.numel() * 4 for v in hb.values()) * ws,
                       "ms_per_step": float(t), "steps": args.e2e_steps,
                       "path": "per rank: pinned host node block -> H2D (copy stream) -> K1 -> ring push to the "
                               "peers + barrier -> pair rows -> band means D2H (copy stream); steps back to back"}

    # ---- CPU baseline (rank 0, N=1 only) ----
    if rank == 0 and ws == 1 and not args.no_cpu_baseline:
        n_cpu = min(args.cpu_nodes or CPU_NODES, c.N)
        n_thr = os.cpu_count() or 1
        r = cpu_baseline(c, n_cpu, n_thr)
        # cores = the threads the run used (the FFT pool); the fold itself is single-threaded
        line["cpu_baseline"] = {"value": r["updates"] / r["s"], "unit": "updates/s", "cores": n_thr, "kind": "port",
                                "sample": f"node subset N'={n_cpu} of cfg{c.cfg}, all K={c.K}, {c.n_bins} bins, "
                                          f"{len(c.metrics)} finalizers; fold single-threaded as in the reference "
                                          f"(FFT pool of {os.cpu_count()} threads)",
                                "breakdown_s": {k: r[k] for k in ("fft_s", "fold_s", "finalize_s")}}
    if rank == 0:
        print(json.dumps(line), flush=True)
    if dist is not None:
        dist.destroy_process_group()


if __name__ == "__main__":
    main()
