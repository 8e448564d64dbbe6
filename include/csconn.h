/*
 * csconn.h -- C ABI of the B200-native all-to-all spectral connectivity path.
 *
 * Drop-in boundary for the reference package `connstream` (arXiv 2303.03279
 * restated in Python; /root/reference/pkg/src/connstream).  The reference has
 * no FFI: its "operator API" is the Python namespace (src/__init__.py:3-15).
 * The Python shim `paper_2303_03279_b200` keeps those names and calls this
 * library through ctypes with raw device pointers.
 *
 * Entry point  <->  reference interface it replaces
 *   cs_plan_create / cs_plan_destroy
 *        SpectrumSet(n_channels, nfft) allocation      spectral.py:125-154
 *        TrialCache (storage mode spectrum cache)       metrics.py:267-282
 *   cs_spectra
 *        trial_spectra / fft_real (+ taper extension)  spectral.py:49-97
 *   cs_pair_metrics
 *        accumulate_spectra + _fold_csd                 spectral.py:204-261
 *        *_bins finalizers                              metrics.py:32-98
 *        finalize_spectral band average                 metrics.py:115-134,
 *                                                       core.py:208-215
 *   cs_pair_sums
 *        SpectrumSet running sums (csd/plv/pli/abs_im)  spectral.py:125-201
 *   cs_row_tile_range / cs_pair_range
 *        pair_index / pair_row_slice (triu row-major)   spectral.py:114-122
 *   cs_last_error
 *        ParameterError / DegenerateTrialCountError     core.py:17-22
 *
 * Conventions: pair p <-> (i<j), row-major upper
 * triangle; per-bin outputs are bin-major [n_bins][pair_stride] fp32 (the
 * reference's [P, nb] is the transposed view); band outputs are [pair_stride].
 * All calls are asynchronous on the caller's cudaStream_t; a plan is
 * single-owner (not thread safe), mirroring spectral.py:250-251.
 */
#ifndef CSCONN_H
#define CSCONN_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

/* status codes (the Python shim maps them to the reference's exceptions) */
#define CS_OK 0
#define CS_EPARAM 1      /* ParameterError                         */
#define CS_EDEGENERATE 2 /* DegenerateTrialCountError              */
#define CS_ECUDA 3       /* CUDA runtime / launch failure          */
#define CS_ENOMEM 4      /* device allocation failed               */

/* input sample types for cs_spectra */
#define CS_F32 0
#define CS_F64 1

/* metric bits (MetricId order of core.py:25-35, spectral metrics only) */
#define CS_COHY (1u << 0)
#define CS_COH (1u << 1)
#define CS_IMAGCOHY (1u << 2)
#define CS_PLV (1u << 3)
#define CS_PLI (1u << 4)
#define CS_USPLI (1u << 5)
#define CS_WPLI (1u << 6)
#define CS_DSWPLI (1u << 7)
#define CS_NUM_METRICS 8

/* cs_plan_create flags */
#define CS_PLAN_WELCH (1u << 0) /* welch mode (spectral.py:100-111, 264-283): a trial of
                                   n_samples >= 2 nfft is cut into n_samples / nfft
                                   non-overlapping nfft segments, each demeaned and
                                   transformed; its CSD / PSD is the mean over segments
                                   before the nonlinear terms.  The segments occupy the
                                   plan's taper axis (n_tapers must be 1, tapers NULL).
                                   Shorter trials fall back to fixed mode. */

typedef struct cs_plan cs_plan;

/* Output descriptor for cs_pair_metrics.  bins[m]: [nbb][pair_stride] fp32
 * (COHY: complex64 interleaved, [nbb][pair_stride][2]); band[m]: [pair_stride]
 * fp32 band mean (COHY: complex64 mean, the weight is its modulus).  NULL
 * pointers are not written.  Output element for global pair p lives at
 * index (p - pair_base). */
typedef struct cs_outputs {
  void* bins[CS_NUM_METRICS];
  void* band[CS_NUM_METRICS];
  int64_t pair_base;
  int64_t pair_stride;
} cs_outputs;

/* Running sums (SpectrumSet layout of spectral.py:136-141, restricted to the
 * requested bins, bin-major [nbb][pair_stride]), fp64 like the reference.  Any
 * pointer may be NULL. */
typedef struct cs_sums {
  double* csd;     /* complex128 [nbb][pair_stride][2]: sum_k CSD_k (Im flushed)   */
  double* plv;     /* complex128 [nbb][pair_stride][2]: sum_k CSD_k / |CSD_k|       */
  int32_t* pli;    /* [nbb][pair_stride]: sum_k sign(Im CSD_k) (integer-valued)    */
  double* abs_im;  /* [nbb][pair_stride]: sum_k |Im CSD_k|                         */
  double* psd;     /* [nbb][n_nodes]: sum_k |X_k|^2                                */
  int64_t pair_base;
  int64_t pair_stride;
} cs_sums;

/*
 * Create a plan for n_nodes channels, trials of n_samples samples, FFT length
 * nfft and the inclusive bin range [lo_bin, hi_bin] kept in the HBM spectrum
 * cache.  tapers: host fp64 [n_tapers][min(n_samples, nfft)] or NULL for the
 * reference's rectangular window (n_tapers must then be 1).  slot_capacity:
 * number of trial slots in the spectrum ring.  spectrum_scale: power of two
 * applied to the fp32 copy of the spectra (0 -> 1.0); every metric is
 * invariant to it.  flags: CS_PLAN_WELCH or 0 (reference: SpectrumSet(...) +
 * accumulate_epoch(mode) of spectral.py:125-141, 264-286).
 */
int cs_plan_create(cs_plan** plan, int device, int n_nodes, int n_samples, int nfft,
                   int lo_bin, int hi_bin, int n_tapers, const double* tapers,
                   int slot_capacity, double spectrum_scale, unsigned flags);
int cs_plan_destroy(cs_plan* plan);

/* K1: demean + taper + one-sided DFT of k_count trials x n_nodes channels.
 * x_dev: device samples, element (k, n, t) at x[k*trial_stride + n*node_stride + t].
 * Trial k lands in slot (slot0 + k) mod slot_capacity.  Increments the plan's
 * FFT counter by k_count*n_nodes*n_tapers (spectral.py:18-30). */
int cs_spectra(cs_plan* plan, const void* x_dev, int dtype, int64_t trial_stride,
               int64_t node_stride, int slot0, int k_count, void* stream);

/* Fused pair kernels over the trials in slots_dev[0..n_slots) and the plan-local
 * bins [bin_lo, bin_lo + n_bins): metric finalisation in the epilogue, per-bin
 * and band-mean outputs.  Row tiles [row_tile_begin, row_tile_end) of the
 * upper-triangular 64-node tiling are computed (0, -1 = all). */
int cs_pair_metrics(cs_plan* plan, const int* slots_dev, int n_slots, unsigned metric_mask,
                    int bin_lo, int n_bins, int row_tile_begin, int row_tile_end,
                    const cs_outputs* out, void* stream);

/* cs_pair_metrics with flags.  CS_PM_REUSE_PREP: the node statistics and packed
 * operands of the previous call on this plan (same slots pointer, trial count,
 * bins and metric mask -- checked) are reused, so a caller that splits one
 * step into row-tile chunks (e.g. to overlap each chunk's download) pays the
 * per-call preparation once; the slots' contents must not have changed. */
#define CS_PM_REUSE_PREP 1u
int cs_pair_metrics_ex(cs_plan* plan, const int* slots_dev, int n_slots, unsigned metric_mask,
                       int bin_lo, int n_bins, int row_tile_begin, int row_tile_end,
                       const cs_outputs* out, unsigned flags, void* stream);

/* SpectrumSet-compatible running sums over the same trial / bin selection, from
 * the fp64 ring with the reference's arithmetic (spectral.py:204-241: per-trial
 * CSD = sum over tapers / welch segments, Im flush at 1e-13 |Re|, unit phasor
 * where |CSD| > DBL_MIN, sign(0) = 0) for pairs [pair_base, pair_base +
 * pair_stride).  An accessor (SpectrumSet.csd_sum etc.), not the metric path. */
int cs_pair_sums(cs_plan* plan, const int* slots_dev, int n_slots, int bin_lo, int n_bins,
                 const cs_sums* out, void* stream);

/* Copy spectra of n_slots slots (plan-local bins [bin_lo, bin_lo+n_bins), taper 0)
 * as complex128 [n_slots][n_nodes][n_bins] into dst_dev (trial_spectra layout). */
int cs_get_spectra(cs_plan* plan, const int* slots_dev, int n_slots, int bin_lo, int n_bins,
                   void* dst_dev, void* stream);

/* Upload externally computed spectra (complex128 [n][n_nodes][n_bins], the
 * trial_spectra layout) into slots slot0.. of a single-taper plan: the drop-in
 * for accumulate_spectra(acc, spectra) (spectral.py:244-261). */
int cs_put_spectra(cs_plan* plan, const void* src_dev, int n, int bin_lo, int n_bins, int slot0,
                   void* stream);
/* Same, into taper (or welch segment) index `taper` of each slot; with weight w
 * applied to the stored values (a welch trial of S segments is stored with
 * w = 1/sqrt(S), so that its summed CSD is the segment mean of
 * spectral.py:272-283 even when trials of different S share one ring). */
int cs_put_taper_spectra(cs_plan* plan, const void* src_dev, int n, int bin_lo, int n_bins, int slot0,
                         int taper, double w, void* stream);

/* Network post-processing on the device (core.py:168-205), over band weights
 * w[n] (fp32, pair order of np.triu_indices) and optional complex weights
 * cw[n] (complex64):
 *  cs_net_normalize  divides w (and cw) in place by max |w| (an all-zero network
 *                    is left unchanged; n >= 1 required),
 *  cs_net_threshold  writes the pair indices of the `keep` largest |w|, ties at the
 *                    threshold broken by ascending (i, j), in ascending order into
 *                    out_idx_dev[keep] (keep = ceil(keep_fraction * n)). */
int cs_net_normalize(float* w_dev, void* cw_dev, int64_t n, void* stream);
int cs_net_threshold(const float* w_dev, int64_t n, int64_t keep, int64_t* out_idx_dev, void* stream);

/* Time-domain metrics (metrics.py:140-260) on the fp64 tensor cores, every trial of
 * a call in one launch.  x_dev: fp64 samples [n_trials][n_channels][n_samples].
 *  cs_cor_sums   total[p] += clip(Pearson_k(i, j), -1, 1) over trials k (upper-triangle
 *                pair order); dead (optional, [n_trials][n_channels]) = 1 for a
 *                zero-variance channel (its edges are 0, the reference warns).
 *  cs_xcor_sums  per pair the first maximum over lags [-max_lag, max_lag] of the
 *                overlap-normalised cross-correlation, peak_sum[p] += value and
 *                lag_sum[p] += lag over trials (negative lag: x = channel i leads);
 *                a constant x or y gives (0, 0). */
int cs_cor_sums(const double* x_dev, int n_trials, int n_channels, int n_samples, double* total,
                unsigned char* dead, void* stream);
int cs_xcor_sums(const double* x_dev, int n_trials, int n_channels, int n_samples, int max_lag,
                 double* peak_sum, double* lag_sum, unsigned char* dead, void* stream);

/* Which K1 kernel the plan runs (for rooflines / reports): 0 direct DFT on the
 * FP64 pipe, 1 direct DFT on the fp64 tensor cores, 2 four-step register FFT,
 * 3 radix-2 shared-memory FFT; -1 for a null plan. */
int cs_plan_k1_kind(const cs_plan* plan);

/* Tiling helpers for sharding (multi-GPU): number of 64-node tiles, the row-tile
 * range of shard `shard` of `n_shards` (balanced by tile count) and the
 * contiguous global pair range [pair_begin, pair_end) it covers. */
int cs_num_row_tiles(int n_nodes);
int cs_row_tile_range(int n_nodes, int n_shards, int shard, int* row_tile_begin,
                      int* row_tile_end, int64_t* pair_begin, int64_t* pair_end);

/* Fallback bookkeeping of the last cs_pair_metrics call (device -> host copy;
 * synchronises the stream).  n_flagged: (pair, bin) entries recomputed in fp64
 * (spectral.py:227-239 arithmetic).  The work list never drops an entry: when it
 * is full, flagged entries go to per-(tile, bin, warp) mask records instead
 * (n_records > 0), which the fallback kernel also processes. */
int cs_last_fallback_count(cs_plan* plan, void* stream, int64_t* n_flagged);
int cs_last_guard_stats(cs_plan* plan, void* stream, int64_t* n_flagged, int64_t* n_records);
int64_t cs_fft_call_count(const cs_plan* plan);
void cs_reset_fft_call_count(cs_plan* plan);
/* 1 when the last cs_pair_metrics call took the IMAGCOHY hand-off (the tensor-core
 * kernel's per-bin IMAGCOHY read by the phase-lag kernel in place of its own sum of
 * Im), else 0.  Instrumentation: the bench's work count. */
int cs_last_imag_handoff(const cs_plan* plan);

/* Instrumentation (bench evidence): CUDA events around every kernel phase on
 * the launching stream; cs_profile_read returns "name:total_ms:count;..." and
 * clears the records.  cs_launch_count: kernels launched by the plan so far. */
int cs_plan_set_profiling(cs_plan* plan, int on);
int cs_profile_read(cs_plan* plan, char* buf, int len);
int64_t cs_launch_count(const cs_plan* plan);

/* Device pointers of the spectrum ring (fp64 and fp32 copies, [slot][L][nb][N]
 * complex) and its element count: used to all-gather node blocks across GPUs. */
int cs_ring_view(cs_plan* plan, void** x64, void** x32, int64_t* n_elems);

/* ---- incremental online window (window.cu; pipeline.py:304-309, metrics.py:450-460) ----
 * The reference re-folds the whole window per update (rebuild_last); every fold sum is
 * additive over trials, so a cs_window keeps per-(pair, bin) running sums (fp32 / int32)
 * for the metric families of its mask and moves them by the changed trials only:
 * changed_slots = n_add new ring slots then n_sub leaving ones.  Per trial the
 * exact-sign guard is |Im| <= g |X_i||X_j| (a count that moves with the window); a
 * (pair, bin) with a risky trial in the window is recomputed over window_slots[0..K) in
 * fp64 by the fallback.  Outputs (all pairs, pair_base 0): per-bin values and band
 * means by metric bit (either may be NULL).  COHY and multitaper plans are not incremental.
 * cs_window_reset zeroes the sums (resynchronise: reset + one update adding the window). */
typedef struct cs_window cs_window;
int cs_window_create(cs_window** w, cs_plan* plan, unsigned metric_mask, int bin_lo, int n_bins);
int cs_window_destroy(cs_window* w);
int cs_window_reset(cs_window* w, void* stream);
int cs_window_update(cs_window* w, const int* changed_slots_dev, int n_add, int n_sub,
                     const int* window_slots_dev, int K, const cs_outputs* out, void* stream);

/* ---- upstream of the spectra (upstream.cu; fp64, hand-written DMMA GEMM / FIR) ----
 *  cs_apply_inverse  y[n_src][T] = M[n_src][n_sens] x[n_sens][T]   (inverse.py:147-154)
 *  cs_project_ring   the source plan's rings (fp64 + scaled fp32) for slots slot0 ..
 *                    slot0 + k_count - 1 = M[dst N][src N] times the sensor plan's
 *                    fp64 spectra (same slots / tapers / bins): source connectivity
 *                    without transforming the source time series
 *  cs_fir_apply      streaming causal FIR of a block x[C][S] (preprocess.py:109-142):
 *                    y = (taps * [hist, x])[:S]; hist / hist_out [C][n_taps - 1]
 *                    (the previous / new last input samples; distinct buffers) */
int cs_apply_inverse(const double* M_dev, int n_src, int n_sens, const double* x_dev, int n_samples,
                     double* y_dev, void* stream);
int cs_project_ring(cs_plan* dst_plan, const cs_plan* src_plan, const double* M_dev, int slot0, int k_count,
                    void* stream);
int cs_fir_apply(const double* taps_dev, int n_taps, const double* x_dev, int n_channels, int n_samples,
                 const double* hist_dev, double* hist_out_dev, double* y_dev, void* stream);

/* ---- multi-GPU: the spectrum ring exchanged over NVLink peer memory (shard.cu) ----
 * Every rank holds a plan over all N nodes; rank r computes K1 for its node block
 * [r*node_block, (r+1)*node_block) with cs_spectra_nodes, then cs_ring_push copies
 * that block of its fp32 ring into every attached peer's ring (strided copy-engine
 * copies, no staging).  The fp64 ring is not exchanged: the exact-sign fallback
 * reads a node's fp64 spectra from the rank owning it (P2P loads).  After the push
 * the caller synchronises the ranks (all pushes into this rank's ring complete)
 * before cs_pair_metrics over its row tiles (cs_row_tile_range).  The reference
 * has no multi-process path; this replaces the NCCL all-gather proposed in
 * SURVEY.md 8(b) (in place, no layout constraint on the ring). */
typedef struct cs_ring_handle {
  unsigned char x64[64];  /* cudaIpcMemHandle_t of the fp64 ring */
  unsigned char x32[64];  /* cudaIpcMemHandle_t of the fp32 ring */
  int32_t n_nodes, slot_capacity, n_tapers, n_bins;  /* geometry, checked on attach */
} cs_ring_handle;
/* K1 for the node range [node0, node0 + n_nodes) only; x_dev holds those nodes. */
int cs_spectra_nodes(cs_plan* plan, const void* x_dev, int dtype, int64_t trial_stride, int64_t node_stride,
                     int node0, int n_nodes, int slot0, int k_count, void* stream);
int cs_ring_export(cs_plan* plan, cs_ring_handle* out);
/* handles[r] of every rank (own included, not opened); node n is owned by rank n / node_block */
int cs_ring_attach(cs_plan* plan, const cs_ring_handle* handles, int n_ranks, int self, int node_block);
/* the same with device pointers of rings in this process (tests, one process driving several plans) */
int cs_ring_attach_ptrs(cs_plan* plan, void* const* x64, void* const* x32, int n_ranks, int self, int node_block);
/* push nodes [node0, node0 + n_nodes) of slots slot0 .. slot0 + k_count - 1 (mod capacity) of the
 * fp32 ring into every attached peer's ring, on stream */
int cs_ring_push(cs_plan* plan, int node0, int n_nodes, int slot0, int k_count, void* stream);

/* Measure this device's FP32 FMA-pipe lane-op rate and FP64 DFMA rate (a few
 * ms of dependent-chain FMA loops; the roofline denominators for K3 and K1). */
int cs_probe_peaks(int device, double* fp32_lane_ops_per_s, double* fp64_fma_per_s);

/* Thread-local message of the last failing call. */
const char* cs_last_error(void);
const char* cs_version(void);

#ifdef __cplusplus
}
#endif
#endif /* CSCONN_H */
