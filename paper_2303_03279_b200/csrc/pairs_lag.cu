// K3: the phase-lag family (PLI, USPLI, WPLI, DSWPLI) plus IMAGCOHY, as a
// register-tiled pair x trial kernel on the FP32/ALU pipes.
//
// Reference: spectral.py:216-241 (_fold_csd: Im flush, sign(Im), |Im| and Im
// sums), metrics.py:49-86 (imagcohy/pli/uspli/wpli/dswpli finalisers),
// metrics.py:115-134 + core.py:208-215 (band mean).
//
// Per (pair i<j, bin b) and trial k the kernel needs t = Im(X_i conj X_j) and
// accumulates sum t, sum |t|, #(t < 0) and min |t| (the exact-sign guard).  Two
// trials are packed per f32x2 register pair, so t costs one FMUL2 + one FFMA2
// per two updates.  A CTA owns a 64 x 64 node tile of the upper triangle and all
// bins of the band; each thread owns 4 x 4 pairs.  Trials are gathered by slot
// index (any window of the HBM spectrum ring) and staged through shared memory
// as float4 (re_a, re_b, im_a, im_b); the J side is stored with Im negated so
// that t = Im_i*Re_j + Re_i*(-Im_j) is a single FFMA2.
//
// Exact-sign guard: with |X| <= M (max over the selected trials), fp32 rounding
// moves t by at most (4 + L) u M_i M_j, so a (pair, bin) whose min_k |t_k| is
// above g*M_i*M_j has the reference's sign(Im) in every trial (and no Im flush,
// spectral.py:227-228).  The rest (about 1e-4 of pair-bins) are appended to a
// work list and recomputed from the fp64 ring by k_lag_fallback.
#include <cuda_fp16.h>

#include <cstdlib>

#include "common.cuh"

namespace cs {

constexpr int kKC = 16;    // k-pairs per pipeline stage (32 trials)
constexpr int kLagStages = 3;

struct LagArgs {
  const float2* X32;
  const double2* X64;
  const float4* PkI;  // [nbb][Kp][N64] (re_a, re_b, im_a, im_b)
  const float4* PkJ;  // [nbb][Kp][N64] (re_a, re_b, -im_a, -im_b)
  int N, N64, nb, L;
  const int* slots;
  int K, Kp;
  int bin_lo, nbb;
  const float* psd;  // [nbb][N]
  const float* mag;  // [nbb][N]
  int real0, real1;  // plan-local bins whose spectra are exactly real (or -1)
  int nt, row_begin;
  int64_t pair_base, pair_stride;
  float* bins[5];    // IMAGCOHY, PLI, USPLI, WPLI, DSWPLI : [nbb][pair_stride]
  float* band[5];
  float* plv_bins;   // multitaper only: PLV of the taper-mean CSD (not separable -> CUDA cores)
  float* plv_band;
  float g;           // guard factor
  float scale2;      // plan scale^2 (fp64 fallback -> fp32 units)
  int4* flags;
  int4* recs;        // guard overflow records (pairs_lag1.cu guard_push), or null
  int* counters;
  int flag_cap;
  double2* const* x64_of;  // sharded plan: fp64 ring of the rank owning node n / node_block (else null)
  int node_block;
  const float* imag_in;    // hand-off: IMAGCOHY per bin from the tensor-core kernel (else null)
  float imag_tau;
  float4* nf;              // [nbb][N64] node factors of the phase-lag epilogue (k_lag_prep)
  const float* nscale;     // [nbb][N] fp16 operand scale of the tensor-core pass (k_tc_prep)
};

// Trial-pair packing of the selected trials (k = 2 kp, 2 kp + 1) into the layouts the
// pair kernel stages with cp.async.  Odd K: the last pair's second trial is a
// phantom with I side (0, M_i 2^-10) and J side (M_j 2^-10, 0), i.e. t = M_i M_j 2^-20
// > g M_i M_j: it never trips the exact-sign guard, adds no negative sign, and its
// contribution to sum t and sum |t| is removed exactly in the epilogue.
constexpr float kPhantom = 9.765625e-4f;  // 2^-10
__global__ void k_lag_prep(const float2* __restrict__ X32, const int* __restrict__ slots, int K, int Kp,
                           int N, int N64, int nb, int L, int bin_lo, const float* __restrict__ mag,
                           const float* __restrict__ psd, const float* __restrict__ nscale, int real0, int real1,
                           float4* __restrict__ PkI, float4* __restrict__ PkJ, float4* __restrict__ nf) {
  // layout [bl][kp][l][n]: taper l of trial pair kp
  const int n = blockIdx.x * blockDim.x + threadIdx.x;
  const int bl = blockIdx.z;
  if (n >= N64) return;
  if (blockIdx.y == 0) {
    // per-node epilogue factors {M', 1/sqrt(psd) / s, 1/sqrt(psd), M' 2^-10}; M' = 0 on
    // exactly-real bins (all Im exactly 0: dead pairs), s = the fp16 operand scale of the
    // tensor-core pass (a power of two: the division is exact), zeros past N
    float4 f = make_float4(0.f, 0.f, 0.f, 0.f);
    if (n < N) {
      const int b = bin_lo + bl;
      const float m = (b == real0 || b == real1) ? 0.f : mag[(int64_t)bl * N + n];
      const float pw = psd[(int64_t)bl * N + n];
      float rp = 0.f;
      if (pw > 0.f) asm("rsqrt.approx.ftz.f32 %0, %1;" : "=f"(rp) : "f"(pw));
      const float s = nscale ? nscale[(int64_t)bl * N + n] : 1.f;
      f = make_float4(m, (pw > 0.f && s > 0.f) ? rp / s : 0.f, rp, m * kPhantom);
    }
    nf[(int64_t)bl * N64 + n] = f;
  }
  for (int y = blockIdx.y; y < Kp * L; y += gridDim.y) {  // grid.y <= 65535 (very long sessions)
  const int kp = y / L, l = y % L;
  float2 va = make_float2(0.f, 0.f), vb = make_float2(0.f, 0.f);
  float2 wb = make_float2(0.f, 0.f);  // J-side value of trial b (phantom differs)
  if (n < N) {
    const int b = bin_lo + bl;
    va = X32[(((int64_t)slots[2 * kp] * L + l) * nb + b) * N + n];
    if (2 * kp + 1 < K) {
      vb = X32[(((int64_t)slots[2 * kp + 1] * L + l) * nb + b) * N + n];
      wb = make_float2(vb.x, -vb.y);
    } else if (l == 0) {  // phantom lives in taper 0 only: t = M_i M_j 2^-20, re = 0
      const float m = mag[(int64_t)bl * N + n] * kPhantom;
      vb = make_float2(0.f, m);
      wb = make_float2(m, -0.f);
    }
  }
  const int64_t o = (((int64_t)bl * Kp + kp) * L + l) * N64 + n;
  PkI[o] = make_float4(va.x, vb.x, va.y, vb.y);
  PkJ[o] = make_float4(va.x, wb.x, -va.y, wb.y);
  }
}

// fp64 recomputation of one flagged (pair, bin) entry by an 8-lane group, lanes over
// trials; reference arithmetic of spectral.py:204-241 in complex128.
__device__ __forceinline__ void fallback_entry(const LagArgs& a, int i, int j, int bl, int lane, bool live) {
  const int64_t slot_stride = (int64_t)a.L * a.nb * a.N;
  const int b = a.bin_lo + bl;
  double s_im = 0.0, s_abs = 0.0;
  int s_sign = 0;
  // a sharded plan reads each node's fp64 spectra from the rank that computed them
  // (P2P loads over NVLink); otherwise from this plan's ring
  const double2* Xi = a.x64_of ? a.x64_of[i / a.node_block] : a.X64;
  const double2* Xj = a.x64_of ? a.x64_of[j / a.node_block] : a.X64;
  const int64_t po = pair_of(i, j, a.N) - a.pair_base;
#pragma unroll 4
  for (int k = lane; k < (live ? a.K : 0); k += 8) {  // unrolled: the trials' loads are independent
    const int slot = a.slots[k];
    double re = 0.0, im = 0.0;
    for (int l = 0; l < a.L; ++l) {
      const double2 xi = Xi[slot * slot_stride + ((int64_t)l * a.nb + b) * a.N + i];
      const double2 xj = Xj[slot * slot_stride + ((int64_t)l * a.nb + b) * a.N + j];
      // (xi.x + i xi.y) * (xj.x - i xj.y)
      re += xi.x * xj.x + xi.y * xj.y;
      im += xi.y * xj.x - xi.x * xj.y;
    }
    if (fabs(im) <= 1e-13 * fabs(re)) im = 0.0;  // spectral.py:227-228
    s_im += im;
    s_abs += fabs(im);
    s_sign += (im > 0.0) - (im < 0.0);
  }
#pragma unroll
  for (int o = 4; o > 0; o >>= 1) {
    s_im += __shfl_xor_sync(0xffffffffu, s_im, o);
    s_abs += __shfl_xor_sync(0xffffffffu, s_abs, o);
    s_sign += __shfl_xor_sync(0xffffffffu, s_sign, o);
  }
  if (lane == 0 && live) {
    float v[5];
    const float psd_i = a.psd[(int64_t)bl * a.N + i], psd_j = a.psd[(int64_t)bl * a.N + j];
    // IMAGCOHY in fp64 then rounded; the ratios are scale invariant
    const double den = sqrt((double)psd_i * (double)psd_j);
    const double imag = den > 0.0 ? s_im * (double)a.scale2 / den : 0.0;
    const double pli = fabs((double)s_sign) / a.K;
    const double wpli = s_abs > 0.0 ? fabs(s_im) / s_abs : 0.0;
    v[0] = (float)imag;
    v[1] = (float)pli;
    v[2] = a.K > 1 ? (float)((a.K * pli * pli - 1.0) / (a.K - 1.0)) : 0.f;
    v[3] = (float)wpli;
    v[4] = (float)(wpli * wpli);
    const float inv = 1.f / (float)a.nbb;
    for (int m = 0; m < 5; ++m) {
      float* bp = a.bins[m] ? a.bins[m] + (int64_t)bl * a.pair_stride + po : nullptr;
      if (bp) *bp = v[m];
      if (a.band[m]) atomicAdd(&a.band[m][po], v[m] * inv);
    }
  }
}

// The fp64 fallback over the guard work list (four entries per warp, so the per-entry
// fp64 finalisation runs four-wide), then over the overflow records of a full list
// (one warp per record, its flagged pairs four at a time; pairs_lag1.cu guard_push).
__global__ void k_lag_fallback(const LagArgs a) {
  const int group = (blockIdx.x * blockDim.x + threadIdx.x) >> 3;
  const int lane = threadIdx.x & 7;
  const int n_groups = (gridDim.x * blockDim.x) >> 3;
  const int count = min(a.counters[0], a.flag_cap);
  for (int w0 = group - (group & 3); w0 < count; w0 += n_groups) {  // warp-uniform trip count
    const int w = w0 + (group & 3);
    int4 f = w < count ? __ldg(&a.flags[w]) : make_int4(-1, -1, 0, 0);
    const bool live = f.x >= 0;  // slots a warp reserved past the capacity are marked empty
    if (!live) f = make_int4(0, 1, 0, 0);
    fallback_entry(a, f.x, f.y, f.z, lane, live);
  }
  if (!a.recs) return;
  const int n_rec = a.counters[2];
  const int warp = (blockIdx.x * blockDim.x + threadIdx.x) >> 5, n_warps = (gridDim.x * blockDim.x) >> 5;
  const int g = (threadIdx.x >> 3) & 3;
  for (int rr = warp; rr < n_rec; rr += n_warps) {
    const int4 h = a.recs[kGuardRecI4 * rr];
    unsigned m[kGuardNP];
#pragma unroll
    for (int w4 = 0; w4 < kGuardNP / 4; ++w4) {
      const int4 v = a.recs[kGuardRecI4 * rr + 1 + w4];
      m[4 * w4] = (unsigned)v.x; m[4 * w4 + 1] = (unsigned)v.y; m[4 * w4 + 2] = (unsigned)v.z; m[4 * w4 + 3] = (unsigned)v.w;
    }
    const int lpr = h.w > 0 ? h.w : 32;  // lanes per tile row of the writer
    int q = 0, pos = 0;  // walk the mask bits (word q, bit pos); group g takes every 4th set bit
    for (;;) {
      int found[4], nf = 0;
      while (nf < 4 && q < kGuardNP) {
        const unsigned rest = m[q] >> pos;
        if (!rest || pos >= 32) { ++q; pos = 0; continue; }
        pos += __ffs(rest) - 1;
        found[nf++] = q * 32 + pos;
        ++pos;
      }
      if (nf == 0) break;
      const bool live = g < nf;
      const int bit = live ? found[g] : 0, qq = bit >> 5, ln = bit & 31;
      const int i = h.x + ln / lpr + kGuardRowStep * (qq / kGuardTC),
                j = h.y + ln % lpr + kGuardColStep * (qq % kGuardTC);
      fallback_entry(a, live ? i : 0, live ? j : 1, h.z, lane, live);
    }
  }
}

// Fallback grid: the flagged count is only known on the device; it scales with the
// pair-bins of the call (~1e-4 of them), so small calls (online windows) launch
// one block per SM instead of 8.
static unsigned fallback_blocks(const LagArgs& a) {
  const int64_t pb = a.pair_stride * (int64_t)a.nbb >> 17;
  return (unsigned)(pb < 148 ? 148 : (pb > 148 * 8 ? 148 * 8 : pb));
}

// the incremental window's fallback (window.cu): the risky (pair, bin) entries over the
// window's slots (per-bin values; band means by atomic adds like the batch path)
void run_window_fallback(Plan& p, const int* slots, int K, int bin_lo, int nbb, const float* psd,
                         float* const* bins5, float* const* band5, int4* recs, cudaStream_t st) {
  LagArgs a{};
  a.X64 = p.X64;
  a.N = p.N; a.nb = p.nb; a.L = p.L;
  a.slots = slots; a.K = K;
  a.bin_lo = bin_lo; a.nbb = nbb;
  a.psd = psd;
  a.pair_base = 0;
  a.pair_stride = (int64_t)p.N * (p.N - 1) / 2;
  for (int q = 0; q < 5; ++q) {
    a.bins[q] = bins5[q];
    a.band[q] = band5[q];
  }
  a.scale2 = p.scale * p.scale;
  a.flags = p.flags; a.recs = recs; a.counters = p.counters; a.flag_cap = p.flag_cap;
  a.x64_of = p.n_ranks > 1 ? p.peer_x64 : nullptr;
  a.node_block = p.node_block;
  PhaseMark ph(p, "lag_fallback", st);
  k_lag_fallback<<<fallback_blocks(a), 256, 0, st>>>(a);
}

bool launch_lag1(const float4* PkI, const float4* PkJ, int N, int N64, int K, int Kp, int bin_lo, int nbb,
                 const float* psd, const float* mag, int real0, int real1, int nt, int row_begin,
                 int64_t pair_base, int64_t pair_stride, float* const* bins, float* const* band, float g,
                 int4* flags, int4* recs, int* counters, int flag_cap, int64_t n_tiles, int nbc,
                 int L, float* plv_bins, float* plv_band, const float* imag_in, float imag_tau, const float4* nf,
                 cudaStream_t st);

bool run_pairs_lag(Plan& p, const LagArgs& a, int64_t n_tiles, cudaStream_t st, bool handoff) {
  cudaMemsetAsync(a.counters, 0, 3 * sizeof(int), st);
  if (!p.reuse_prep) {
    PhaseMark ph(p, "lag_prep", st);
    dim3 grid((a.N64 + 127) / 128, a.Kp * a.L < 65535 ? a.Kp * a.L : 65535, a.nbb);
    k_lag_prep<<<grid, 128, 0, st>>>(p.X32, a.slots, a.K, a.Kp, a.N, a.N64, a.nb, a.L, a.bin_lo, a.mag, a.psd,
                                     a.nscale, a.real0, a.real1, (float4*)a.PkI, (float4*)a.PkJ, a.nf);
  }
  {
    PhaseMark ph(p, "pairs_lag", st);
    // small pair spaces (few tiles, many bins): split the bins over CTAs.  One CTA per
    // SM, so the makespan is waves x (per-CTA fixed cost + bins x per-bin cost); the
    // fixed part (barrier init, band zeroing, first-stage TMA latency, band write-out)
    // measured ~0.25-0.4 of a bin (cfg1/2/4 sweeps), so pick the split minimising
    // waves * (0.4 + bins per CTA).
    int nsm = 148;
    cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, p.device);
    int nbc = 1;
    double best = 1e300;
    for (int c = 1; c <= a.nbb; ++c) {
      const int bpc = (a.nbb + c - 1) / c, chunks = (a.nbb + bpc - 1) / bpc;
      if (chunks != c) continue;  // no empty chunks
      const double waves = (double)((n_tiles * chunks + nsm - 1) / nsm);
      const double cost = waves * (0.4 + bpc);
      if (cost < best) {
        best = cost;
        nbc = c;
      }
    }
    static const int force_nbc = getenv("CSCONN_K3_NBC") ? atoi(getenv("CSCONN_K3_NBC")) : 0;  // sweep override
    if (force_nbc) {
      nbc = force_nbc < 1 ? 1 : (force_nbc > a.nbb ? a.nbb : force_nbc);
      nbc = (a.nbb + ((a.nbb + nbc - 1) / nbc) - 1) / ((a.nbb + nbc - 1) / nbc);
    }
    if (nbc > 1) {
      for (int m = 0; m < 5; ++m)
        if (a.band[m]) cudaMemsetAsync(a.band[m], 0, a.pair_stride * sizeof(float), st);
      if (a.plv_band) cudaMemsetAsync(a.plv_band, 0, a.pair_stride * sizeof(float), st);
    }
    if (!launch_lag1(a.PkI, a.PkJ, a.N, a.N64, a.K, a.Kp, a.bin_lo, a.nbb, a.psd, a.mag, a.real0, a.real1, a.nt,
                     a.row_begin, a.pair_base, a.pair_stride, a.bins, a.band, a.g, a.flags, a.recs, a.counters, a.flag_cap,
                     n_tiles, nbc, a.L, a.plv_bins, a.plv_band, a.imag_in, a.imag_tau, a.nf, st))
      return false;
  }
  {
    PhaseMark ph(p, "lag_fallback", st);
    k_lag_fallback<<<fallback_blocks(a), 256, 0, st>>>(a);
  }
  return true;
}

}  // namespace cs

namespace cs {

// metric-bit -> lag-kernel output slot
static const unsigned kLagBits[5] = {CS_IMAGCOHY, CS_PLI, CS_USPLI, CS_WPLI, CS_DSWPLI};

static const int kLagIdx[5] = {2, 4, 5, 6, 7};

// IMAGCOHY without any sign-based metric: D_im of the tensor-core pass already is
// sum Im(X_i conj X_j) (fp16 hi/lo products, ~1e-6 relative), so the phase-lag
// kernel is not launched for it.  With PLI/USPLI/WPLI/DSWPLI requested the
// phase-lag kernel accumulates sum Im anyway and IMAGCOHY stays there.
// (Not with COHY requested: the near-zero IMAGCOHY entries are zeroed in the
// tensor-core epilogue for the fp64 fallback, which would corrupt COHY's Im.)
static bool imag_on_tensor_cores(unsigned mask) {
  return (mask & CS_IMAGCOHY) && !(mask & (CS_PLI | CS_USPLI | CS_WPLI | CS_DSWPLI | CS_COHY));
}

// The fused call (every phase-lag output plus IMAGCOHY and COH, single taper, no COHY):
// the tensor-core kernel's D_im already is sum Im, so it writes IMAGCOHY and the
// phase-lag kernel reads it for WPLI's numerator instead of accumulating sum Im in its
// trial loop (one FADD2 of four FMA-pipe operations per update).  Entries whose
// per-bin IMAGCOHY comes from the tensor-core kernel (|err| < tau = imag_tau_of); the
// phase-lag kernel forms its band mean, and its guard-flagged entries -- and those whose
// sum |Im| is too small for WPLI's numerator error -- are re-folded in fp64 with IMAGCOHY.
// CSCONN_IMAG_TC=0 turns the hand-off off (A/B).
static bool imag_handoff(const Plan& p, unsigned mask, int K, int nbb, const cs_outputs* out) {
  static const bool off = getenv("CSCONN_IMAG_TC") && getenv("CSCONN_IMAG_TC")[0] == '0';
  if (off || p.L != 1 || (mask & CS_COHY) || !(mask & CS_COH) || (K + 1) / 2 >= 65536) return false;
  if ((uint64_t)nbb * (uint64_t)out->pair_stride + kTile >= (1ull << 32)) return false;  // FULL kernel's 32-bit offsets
  for (int q = 0; q < 5; ++q)
    if (!(mask & kLagBits[q]) || !out->bins[kLagIdx[q]] || !out->band[kLagIdx[q]]) return false;
  return true;
}
static float imag_tau_of(int Kc) { return 1e-5f + 6e-8f * (float)Kc; }  // pairs_tc.cu: D_im error / norm

int run_lag_family(Plan& p, const int* slots, int K, unsigned mask, int bin_lo, int nbb,
                    int rb, int re, const cs_outputs* out, cudaStream_t st) {
  const bool handoff = imag_handoff(p, mask, K, nbb, out);
  if (imag_on_tensor_cores(mask)) mask &= ~(unsigned)CS_IMAGCOHY;
  unsigned any = 0;
  for (int q = 0; q < 5; ++q) any |= mask & kLagBits[q];
  const bool plvk = p.L > 1 && (mask & CS_PLV);
  if (!any && !plvk) return 0;
  if (p.L > 4) {
    cs_set_error("at most 4 tapers are supported, got %d", p.L);
    return -1;
  }
  LagArgs a{};
  a.X32 = p.X32;
  a.X64 = p.X64;
  a.N = p.N; a.nb = p.nb; a.L = p.L;
  a.N64 = (p.N + kTile - 1) / kTile * kTile;
  a.slots = slots; a.K = K;
  a.Kp = (K + 1) / 2;
  {
    const size_t need = (size_t)(2 * nbb * a.Kp * p.L + nbb) * a.N64 * sizeof(float4);
    if (need > p.lag_bytes) {
      if (p.lag_ops) cudaFreeAsync(p.lag_ops, st);
      if (cudaMallocAsync(&p.lag_ops, need, st) != cudaSuccess) {
        p.lag_ops = nullptr;
        p.lag_bytes = 0;
        cs_set_error("device allocation failed (phase-lag operands %zu bytes)", need);
        return -1;
      }
      p.lag_bytes = need;
    }
    a.PkI = (const float4*)p.lag_ops;
    a.PkJ = a.PkI + (size_t)nbb * a.Kp * p.L * a.N64;
    a.nf = (float4*)a.PkJ + (size_t)nbb * a.Kp * p.L * a.N64;
  }
  a.bin_lo = bin_lo; a.nbb = nbb;
  a.psd = p.psd; a.mag = p.mag;
  // exactly-real bins (DC := 0 and the real Nyquist bin of K1's spectra) are resolved in the
  // epilogue without the fp64 fallback; caller spectra (cs_put_spectra) may be complex there,
  // which k_put_spectra records in counters[3] (read here only when caller spectra were put)
  int complex_edge = 0;
  if (p.spectra_put) {
    cudaMemcpyAsync(&complex_edge, p.counters + 3, sizeof(int), cudaMemcpyDeviceToHost, st);
    cudaStreamSynchronize(st);
  }
  a.real0 = complex_edge ? -1 : p.dc_local;
  a.real1 = complex_edge ? -1 : p.nyq_local;
  a.nt = (p.N + kTile - 1) / kTile;
  a.row_begin = rb;
  a.pair_base = out->pair_base;
  a.pair_stride = out->pair_stride;
  for (int q = 0; q < 5; ++q) {
    const bool on = (mask & kLagBits[q]) != 0;
    a.bins[q] = on ? (float*)out->bins[kLagIdx[q]] : nullptr;
    a.band[q] = on ? (float*)out->band[kLagIdx[q]] : nullptr;
  }
  a.plv_bins = plvk ? (float*)out->bins[3] : nullptr;
  a.plv_band = plvk ? (float*)out->band[3] : nullptr;
  // exact-sign guard: t = sum_l FFMA(Im_i, Re_j, FMUL(Re_i, -Im_j)) from fp32-rounded
  // spectra errs by at most (2 + 2L) u sum_l |X_il| |X_jl| <= (2 + 2L) u M_i M_j (two input
  // roundings per product, then one rounding per multiply and per fused add; Cauchy-Schwarz
  // over the tapers), u = 2^-24; 1.25x margin for the fp32 magnitudes M
  a.g = 1.25f * (2.f + 2.f * (float)p.L) * 5.9604645e-8f;
  a.x64_of = p.n_ranks > 1 ? p.peer_x64 : nullptr;
  a.node_block = p.node_block;
  if (const char* gs = getenv("CSCONN_GUARD_G")) a.g *= (float)atof(gs);  // test override (negative control)
  a.scale2 = p.scale * p.scale;
  a.flags = p.flags;
  a.counters = p.counters;
  a.flag_cap = p.flag_cap;
  int64_t n_tiles = 0;
  for (int I = rb; I < re; ++I) n_tiles += a.nt - I;
  // overflow records: at most one per (tile, bin, compute warp) of the call
  const size_t n_rec = (size_t)n_tiles * nbb * kGuardWarps;
  if (n_rec > p.rec_cap) {
    if (p.recs) cudaFreeAsync(p.recs, st);
    if (cudaMallocAsync(&p.recs, n_rec * kGuardRecI4 * sizeof(int4), st) != cudaSuccess) {
      p.recs = nullptr;
      p.rec_cap = 0;
      cs_set_error("device allocation failed (guard records %zu bytes)", n_rec * kGuardRecI4 * sizeof(int4));
      return -1;
    }
    p.rec_cap = n_rec;
  }
  a.recs = p.recs;
  if (handoff) {
    a.imag_in = (const float*)out->bins[2];
    a.imag_tau = imag_tau_of(K * p.L);
  }
  if (!run_pairs_lag(p, a, n_tiles, st, handoff)) return -1;
  return 2;
}

bool run_pairs_tc(Plan& p, const int* slots, int K, int bin_lo, int nbb, int rb, int re, bool do_x, bool do_u,
                  bool do_imag, const cs_outputs* out, const float* nscale, cudaStream_t st, bool handoff);

int run_coh_family(Plan& p, const int* slots, int K, unsigned mask, int bin_lo, int nbb,
                    int rb, int re, const cs_outputs* out, cudaStream_t st) {
  const bool handoff = imag_handoff(p, mask, K, nbb, out);
  p.imag_handoff = handoff;
  const bool do_imag = imag_on_tensor_cores(mask) || handoff;
  const bool do_x = (mask & (CS_COHY | CS_COH)) != 0 || do_imag;
  const bool do_u = (mask & CS_PLV) != 0 && p.L == 1;  // multitaper PLV runs in the lag kernel
  if (!do_x && !do_u) return 0;
  if (!run_pairs_tc(p, slots, K, bin_lo, nbb, rb, re, do_x, do_u, do_imag, out, p.nscale, st, handoff))
    return -1;
  if (do_imag && !handoff && (out->bins[2] || out->band[2])) {  // fp64 values for the near-zero IMAGCOHY entries
    LagArgs a{};
    a.X64 = p.X64;
    a.N = p.N; a.nb = p.nb; a.L = p.L;
    a.slots = slots; a.K = K;
    a.bin_lo = bin_lo; a.nbb = nbb;
    a.psd = p.psd;
    a.pair_base = out->pair_base;
    a.pair_stride = out->pair_stride;
    a.bins[0] = (float*)out->bins[2];
    a.band[0] = (float*)out->band[2];
    a.scale2 = p.scale * p.scale;
    a.flags = p.flags;
    a.counters = p.counters;
    a.flag_cap = p.flag_cap;
    a.x64_of = p.n_ranks > 1 ? p.peer_x64 : nullptr;
    a.node_block = p.node_block;
    PhaseMark ph(p, "lag_fallback", st);
    k_lag_fallback<<<fallback_blocks(a), 256, 0, st>>>(a);
  }
  return 0;  // launches are counted by the phase marks
}

}  // namespace cs
