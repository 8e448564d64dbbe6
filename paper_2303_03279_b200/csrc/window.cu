// Incremental online window (pipeline.py:304-309 + metrics.py:450-460).
//
// The reference re-folds the whole window on every update (rebuild_last: reset +
// re-add the last W cached trials).  Every running sum of the fold is additive over
// trials (spectral.py:216-241: csd_sum, plv_sum, pli_sum, abs_im_sum; psd_sum), so a
// window that moves by n_new trials is the previous window's sums plus the new trials'
// terms minus the leaving trials' terms: O(n_new) instead of O(W) work per (pair, bin).
//
// State per (pair, bin), fp32 / int32, for the requested metric families:
//   S_im = sum Im(X_i conj X_j), S_abs = sum |Im|, S_sign = #(Im < 0)       (phase lag)
//   S_re = sum Re(X_i conj X_j)                                            (COH, with S_im)
//   U_re, U_im = sum of unit phasors X_i conj X_j / |X_i||X_j|               (PLV)
//   risky = number of window trials whose fp32 Im is NOT within its error bound of 0
//           (a (pair, bin) is exact in fp32 when all K are; then no Im is 0 and
//           sum sign = K - 2 #(Im < 0))
// The exact-sign guard is per trial here: a trial is risky when |t| <= g |X_i||X_j| (the
// fp32 error of t is below (4 + L) u |X_i||X_j|), a property of the trial alone, so the
// count moves with the window like the sums.  A (pair, bin) with risky > 0 is recomputed
// over the whole window in fp64 by the batch path's fallback (reference arithmetic incl.
// the 1e-13 Im flush).  Node power sums are per (bin, node).  Band means accumulate by
// atomics (v / nbb per bin), the fallback adding the risky entries' fp64 values.
//
// One CTA of 256 threads per (32 x 32 pair tile, bin): thread = 4 pairs (rows ty + 8 r,
// column tx: a warp is one row segment of 32 consecutive pairs, so every state access
// is coalesced), several CTAs per SM so the state traffic is latency-hidden; the
// changed trials' spectra of the tile's 64 nodes are staged in shared memory, 16
// trials at a time.
#include <type_traits>

#include "common.cuh"
#include "ptx.cuh"

namespace cs {

constexpr int kWinChunk = 16;
constexpr int kWinTile = 32;
constexpr int kWinThreads = 256;
constexpr int kWinPairs = kWinTile * kWinTile / kWinThreads;  // pairs per thread (rows ty + 16 p)
constexpr int kWinRowStep = kWinThreads / 32;

struct WinArgs {
  const float2* X32;
  int N, nb, slot_cap;
  const int* slots;  // [n_add + n_sub]: added trials first
  int n_add, n_sub;
  int bin_lo, nbb;
  int nt;
  float* S_im; float* S_abs; int* S_sign; int* risky;   // [nbb][P] (null when unused)
  float* S_re; float* U_re; float* U_im;
  const float* psd_state;  // [nbb][N] node power sums (the fp32 ring's scaled units)
  int K;                   // trials in the window after the update
  float g;                 // guard factor
  unsigned want;           // metric bits (CS_*)
  float* bins[8];          // per-bin outputs by metric bit, [nbb][P] (or null)
  float* band[8];          // band means by metric bit, [P], zeroed before the launch (or null)
  int4* flags;
  int4* recs;              // overflow records, capacity n_tiles * nbb * 128
  int* counters;
  int flag_cap;
};

// node power sums: psd_state[b][n] += sum_add |X|^2 - sum_sub |X|^2 (one thread per node-bin)
__global__ void k_window_psd(const float2* __restrict__ X32, int N, int nb, const int* __restrict__ slots,
                             int n_add, int n_sub, int bin_lo, int nbb, float* __restrict__ psd_state) {
  const int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (e >= (int64_t)nbb * N) return;
  const int bl = (int)(e / N), n = (int)(e % N), b = bin_lo + bl;
  float s = psd_state[e];
  for (int q = 0; q < n_add + n_sub; ++q) {
    const float2 x = X32[((int64_t)slots[q] * nb + b) * N + n];
    const float p = fmaf(x.x, x.x, x.y * x.y);
    s += q < n_add ? p : -p;
  }
  psd_state[e] = s;
}

template <bool LAG, bool COH, bool PLV>
__global__ void __launch_bounds__(kWinThreads, 4) k_window_update(const WinArgs a) {
  __shared__ float2 xs[kWinChunk][2 * kWinTile];  // the chunk's spectra, tile nodes (i: 0..31, j: 32..63)
  __shared__ float2 us[kWinChunk][2 * kWinTile];  // unit phasors X / |X| (0 for a zero spectrum)
  __shared__ float mg[kWinChunk][2 * kWinTile];   // |X|
  int I, J;
  decode_tile(blockIdx.x, a.nt, 0, I, J);
  const int bl = blockIdx.y, b = a.bin_lo + bl;
  const int iBase = I * kWinTile, jBase = J * kWinTile;
  const int tx = threadIdx.x & 31, ty = threadIdx.x >> 5;
  const int nq = a.n_add + a.n_sub;
  constexpr bool lag = LAG, coh = COH, plv = PLV;
  const bool sgn = a.S_sign != nullptr, absd = a.S_abs != nullptr;  // PLI / USPLI, WPLI / DSWPLI
  const float invK = 1.f / (float)a.K, inv_nb = 1.f / (float)a.nbb;
  const int64_t P = (int64_t)a.N * (a.N - 1) / 2;

  float s_im[kWinPairs], s_abs[kWinPairs], s_re[kWinPairs], u_re[kWinPairs], u_im[kWinPairs];
  int s_sign[kWinPairs], rk[kWinPairs];
  bool ok[kWinPairs];
  int64_t o[kWinPairs];
#pragma unroll
  for (int p = 0; p < kWinPairs; ++p) {
    const int i = iBase + ty + kWinRowStep * p, j = jBase + tx;
    ok[p] = i < j && j < a.N;
    o[p] = ok[p] ? (int64_t)bl * P + pair_of(i, j, a.N) : 0;
    s_im[p] = s_abs[p] = s_re[p] = u_re[p] = u_im[p] = 0.f;
    s_sign[p] = rk[p] = 0;
    if (!ok[p]) continue;
    if (lag || coh) s_im[p] = a.S_im[o[p]];
    if (lag) {
      rk[p] = a.risky[o[p]];
      if (absd) s_abs[p] = a.S_abs[o[p]];
      if (sgn) s_sign[p] = a.S_sign[o[p]];
    }
    if (coh) s_re[p] = a.S_re[o[p]];
    if (plv) { u_re[p] = a.U_re[o[p]]; u_im[p] = a.U_im[o[p]]; }
  }
  for (int q0 = 0; q0 < nq; q0 += kWinChunk) {
    const int nc = min(kWinChunk, nq - q0);
    __syncthreads();
    {  // thread -> one node column of the tile, every fourth trial of the chunk
      const int c = threadIdx.x & (2 * kWinTile - 1);
      const int n = c < kWinTile ? iBase + c : jBase + c - kWinTile;
      const bool nok = n < a.N;
      const float gf = c < kWinTile ? 1.f : a.g;   // |X_i| and g |X_j| (the guard bound)
      for (int q = threadIdx.x / (2 * kWinTile); q < nc; q += kWinThreads / (2 * kWinTile)) {
        const float2 x = nok ? a.X32[((int64_t)a.slots[q0 + q] * a.nb + b) * a.N + n] : make_float2(0.f, 0.f);
        const float m2 = fmaf(x.x, x.x, x.y * x.y);
        const float rr = m2 > 0.f ? rsqrtf(m2) : 0.f;
        xs[q][c] = x;
        us[q][c] = make_float2(x.x * rr, x.y * rr);
        mg[q][c] = gf * m2 * rr;
      }
    }
    __syncthreads();
    // entering trials (+) then leaving trials (-): the sign is a compile-time constant.
    // Counts: #(t < 0) (sign bit; a non-risky entry has no t == 0, so sum sign = K - 2 #neg)
    // and #(trials with |t| > g |X_i||X_j|) (sign bit of |t| - bound), one LEA.HI each.
    auto step = [&](int q, auto sgn) {
      constexpr float sg = decltype(sgn)::value > 0 ? 1.f : -1.f;
      constexpr int isg = decltype(sgn)::value;
      const float2 xj = xs[q][kWinTile + tx];
      const float gmj = mg[q][kWinTile + tx];  // g |X_j|
#pragma unroll
      for (int p = 0; p < kWinPairs; ++p) {
        const int li = ty + kWinRowStep * p;
        const float2 xi = xs[q][li];
        const float t = fmaf(xi.y, xj.x, -xi.x * xj.y);  // Im(X_i conj X_j)
        if (LAG || COH) s_im[p] += sg * t;
        if (LAG) {
          s_abs[p] += sg * fabsf(t);
          s_sign[p] += isg * (int)(__float_as_uint(t) >> 31);                        // negatives
          rk[p] += isg * (int)(__float_as_uint(fmaf(gmj, mg[q][li], -fabsf(t))) >> 31);  // safe trials
        }
        if (COH) s_re[p] += sg * fmaf(xi.x, xj.x, xi.y * xj.y);
        if (PLV) {
          const float2 ui = us[q][li], uj = us[q][kWinTile + tx];
          u_re[p] += sg * fmaf(ui.x, uj.x, ui.y * uj.y);
          u_im[p] += sg * fmaf(ui.y, uj.x, -ui.x * uj.y);
        }
      }
    };
    const int q_add = min(nc, max(0, a.n_add - q0));
    for (int q = 0; q < q_add; ++q) step(q, std::integral_constant<int, 1>{});
    for (int q = q_add; q < nc; ++q) step(q, std::integral_constant<int, -1>{});
  }
  unsigned fl = 0;
#pragma unroll
  for (int p = 0; p < kWinPairs; ++p) {
    if (!ok[p]) continue;
    const int i = iBase + ty + kWinRowStep * p, j = jBase + tx;
    if (lag || coh) a.S_im[o[p]] = s_im[p];
    if (lag) {
      a.risky[o[p]] = rk[p];
      if (absd) a.S_abs[o[p]] = s_abs[p];
      if (sgn) a.S_sign[o[p]] = s_sign[p];
    }
    if (coh) a.S_re[o[p]] = s_re[p];
    if (plv) { a.U_re[o[p]] = u_re[p]; a.U_im[o[p]] = u_im[p]; }
    // ---- the window's metrics (metrics.py:32-86) ----
    // rk counts safe trials, s_sign negative ones (state semantics of this kernel)
    const bool flagged = lag && rk[p] < a.K;  // a risky trial in the window: the fp64 fallback writes

    const int64_t po = o[p] - (int64_t)bl * P;
    auto put = [&](int m, float v) {
      if (a.bins[m]) __stcs(&a.bins[m][o[p]], v);
      if (a.band[m]) atomicAdd(&a.band[m][po], v * inv_nb);
    };
    if (coh) {
      const float den = a.psd_state[(int64_t)bl * a.N + i] * a.psd_state[(int64_t)bl * a.N + j];
      const float rs = den > 0.f ? rsqrtf(den) : 0.f;
      const float cr = s_re[p] * rs, ci = s_im[p] * rs;
      if (a.want & CS_COH) put(1, sqrtf(cr * cr + ci * ci));
      if ((a.want & CS_IMAGCOHY) && !flagged) put(2, ci);
    }
    if (plv) put(3, sqrtf(u_re[p] * u_re[p] + u_im[p] * u_im[p]) * invK);
    if (lag && !flagged) {
      const float pli = fabsf((float)(a.K - 2 * s_sign[p])) * invK;
      const float w = s_abs[p] > 0.f ? fminf(fabsf(s_im[p]) / s_abs[p], 1.f) : 0.f;
      if (a.want & CS_PLI) put(4, pli);
      if (a.want & CS_USPLI) put(5, a.K > 1 ? (a.K * pli * pli - 1.f) / (float)(a.K - 1) : 0.f);
      if (a.want & CS_WPLI) put(6, w);
      if (a.want & CS_DSWPLI) put(7, w * w);
    }
    fl |= (unsigned)flagged << p;
  }
  // rare: full fp64 recompute of these (pair, bin) entries over the window; one list
  // reservation per warp and row segment, a mask record when the list is full
#pragma unroll
  for (int p = 0; p < kWinPairs; ++p) {
    const bool f = (fl >> p) & 1u;
    const unsigned m = __ballot_sync(0xffffffffu, f);
    if (!m) continue;
    const int i = iBase + ty + kWinRowStep * p, j0 = jBase;
    int base = 0;
    if (tx == 0) base = atomicAdd(&a.counters[0], __popc(m));
    base = __shfl_sync(0xffffffffu, base, 0);
    if (base + __popc(m) <= a.flag_cap) {
      if (f) a.flags[base + __popc(m & ((1u << tx) - 1u))] = make_int4(i, j0 + tx, bl, 0);
    } else {
      if (tx < __popc(m) && base + tx < a.flag_cap) a.flags[base + tx] = make_int4(-1, -1, 0, 0);
      if (tx == 0) {  // record (row, column base, bin, mask) in the fallback's format (pairs_lag.cu)
        const int rec = atomicAdd(&a.counters[2], 1);
        a.recs[kGuardRecI4 * rec] = make_int4(i, j0, bl, 32);  // 32 lanes along the row
        a.recs[kGuardRecI4 * rec + 1] = make_int4((int)m, 0, 0, 0);
        for (int w4 = 2; w4 < kGuardRecI4; ++w4) a.recs[kGuardRecI4 * rec + w4] = make_int4(0, 0, 0, 0);
        a.counters[1] = 1;
      }
    }
  }
}

}  // namespace cs

// ---------------------------------------------------------------------------
struct cs_window {
  cs::Plan* plan = nullptr;
  unsigned mask = 0;
  int bin_lo = 0, nbb = 0;
  int64_t P = 0;
  float *S_im = nullptr, *S_abs = nullptr, *S_re = nullptr, *U_re = nullptr, *U_im = nullptr, *psd = nullptr;
  int *S_sign = nullptr, *risky = nullptr;
  int4* recs = nullptr;           // guard overflow records (kGuardRecI4 int4 each)
};

namespace cs {
struct LagArgs;
void run_window_fallback(Plan& p, const int* slots, int K, int bin_lo, int nbb, const float* psd,
                         float* const* bins5, float* const* band5, int4* recs, cudaStream_t st);
}

extern "C" {

int cs_window_create(cs_window** out, cs_plan* plan, unsigned mask, int bin_lo, int nbb) {
  cs::Plan* p = (cs::Plan*)plan;
  if (!out || !p) { cs_set_error("cs_window_create: null argument"); return CS_EPARAM; }
  *out = nullptr;
  if (mask == 0 || (mask >> CS_NUM_METRICS) || (mask & CS_COHY)) {
    cs_set_error("incremental window: metric mask 0x%x (COHY is not supported incrementally)", mask);
    return CS_EPARAM;
  }
  if (p->L != 1) { cs_set_error("incremental window: single-taper plans only"); return CS_EPARAM; }
  if (bin_lo < 0 || nbb < 1 || bin_lo + nbb > p->nb) { cs_set_error("incremental window: bad bins"); return CS_EPARAM; }
  cs_window* w = new cs_window();
  w->plan = p;
  w->mask = mask;
  w->bin_lo = bin_lo;
  w->nbb = nbb;
  w->P = (int64_t)p->N * (p->N - 1) / 2;
  const size_t n = (size_t)nbb * w->P;
  const bool lag = mask & (CS_IMAGCOHY | CS_PLI | CS_USPLI | CS_WPLI | CS_DSWPLI);
  const bool coh = mask & (CS_COH | CS_IMAGCOHY);
  const bool plv = mask & CS_PLV;
  bool ok = true;
  auto al = [&](void** ptr, size_t bytes) { if (ok && cudaMalloc(ptr, bytes) != cudaSuccess) ok = false; };
  if (lag || coh) al((void**)&w->S_im, n * 4);
  if (lag) al((void**)&w->risky, n * 4);
  if (mask & (CS_WPLI | CS_DSWPLI)) al((void**)&w->S_abs, n * 4);
  if (mask & (CS_PLI | CS_USPLI)) al((void**)&w->S_sign, n * 4);
  if (coh) { al((void**)&w->S_re, n * 4); al((void**)&w->psd, (size_t)nbb * p->N * 4); }
  if (plv) { al((void**)&w->U_re, n * 4); al((void**)&w->U_im, n * 4); }
  {  // at most one record per (32 x 32 tile, bin, row)
    const int64_t nt = (p->N + cs::kWinTile - 1) / cs::kWinTile;
    al((void**)&w->recs, (size_t)(nt * (nt + 1) / 2) * nbb * cs::kWinTile * cs::kGuardRecI4 * sizeof(int4));
  }
  if (!ok) {
    cudaGetLastError();
    cs_window_destroy(w);
    cs_set_error("device allocation failed (incremental window state)");
    return CS_ENOMEM;
  }
  *out = w;
  return cs_window_reset(w, nullptr);
}

int cs_window_destroy(cs_window* w) {
  if (!w) return CS_OK;
  cudaFree(w->S_im); cudaFree(w->S_abs); cudaFree(w->S_re); cudaFree(w->U_re); cudaFree(w->U_im);
  cudaFree(w->psd); cudaFree(w->S_sign); cudaFree(w->risky); cudaFree(w->recs);
  delete w;
  return CS_OK;
}

int cs_window_reset(cs_window* w, void* stream) {
  if (!w) return CS_EPARAM;
  cudaStream_t st = (cudaStream_t)stream;
  const size_t n = (size_t)w->nbb * w->P * 4;
  for (void* ptr : {(void*)w->S_im, (void*)w->S_abs, (void*)w->S_re, (void*)w->U_re, (void*)w->U_im,
                    (void*)w->S_sign, (void*)w->risky})
    if (ptr) cudaMemsetAsync(ptr, 0, n, st);
  if (w->psd) cudaMemsetAsync(w->psd, 0, (size_t)w->nbb * w->plan->N * 4, st);
  return cudaPeekAtLastError() == cudaSuccess ? CS_OK : CS_ECUDA;
}

int cs_window_update(cs_window* w, const int* changed_slots, int n_add, int n_sub, const int* window_slots,
                     int K, const cs_outputs* out, void* stream) {
  if (!w || !changed_slots || !window_slots || !out) { cs_set_error("cs_window_update: null argument"); return CS_EPARAM; }
  if (n_add < 0 || n_sub < 0 || K < 1) { cs_set_error("cs_window_update: bad trial counts"); return CS_EDEGENERATE; }
  if ((w->mask & CS_USPLI) && K < 2) { cs_set_error("USPLI needs at least 2 trials"); return CS_EDEGENERATE; }
  if (out->pair_base != 0 || out->pair_stride != w->P) {
    cs_set_error("cs_window_update: outputs must cover all pairs");
    return CS_EPARAM;
  }
  cs::Plan& p = *w->plan;
  if (p.N < 2) return CS_OK;
  cudaStream_t st = (cudaStream_t)stream;
  const bool lag = w->mask & (CS_IMAGCOHY | CS_PLI | CS_USPLI | CS_WPLI | CS_DSWPLI);
  if (w->psd && n_add + n_sub > 0) {
    cs::PhaseMark ph(p, "window_psd", st);
    const int64_t n = (int64_t)w->nbb * p.N;
    cs::k_window_psd<<<(unsigned)((n + 255) / 256), 256, 0, st>>>(p.X32, p.N, p.nb, changed_slots, n_add, n_sub,
                                                                    w->bin_lo, w->nbb, w->psd);
  }
  cs::WinArgs a{};
  a.X32 = p.X32; a.N = p.N; a.nb = p.nb; a.slot_cap = p.slot_cap;
  a.slots = changed_slots; a.n_add = n_add; a.n_sub = n_sub;
  a.bin_lo = w->bin_lo; a.nbb = w->nbb;
  a.nt = (p.N + cs::kWinTile - 1) / cs::kWinTile;
  a.S_im = w->S_im; a.S_abs = w->S_abs; a.S_sign = w->S_sign; a.risky = w->risky;
  a.S_re = w->S_re; a.U_re = w->U_re; a.U_im = w->U_im; a.psd_state = w->psd;
  a.K = K;
  a.g = 1.25f * 4.f * 5.9604645e-8f;  // per trial: 4 u |X_i| |X_j| (pairs_lag.cu), 1.25x margin
  if (const char* gs = getenv("CSCONN_GUARD_G")) a.g *= (float)atof(gs);
  a.want = w->mask;
  for (int m = 0; m < 8; ++m) {
    const bool on = m > 0 && (w->mask & (1u << m));
    a.bins[m] = on ? (float*)out->bins[m] : nullptr;
    a.band[m] = on ? (float*)out->band[m] : nullptr;
    if (a.band[m]) cudaMemsetAsync(a.band[m], 0, w->P * sizeof(float), st);  // atomics add v / nbb
  }
  a.flags = p.flags; a.recs = w->recs; a.counters = p.counters; a.flag_cap = p.flag_cap;
  cudaMemsetAsync(p.counters, 0, 3 * sizeof(int), st);
  {
    cs::PhaseMark ph(p, "window_update", st);
    const int nt = a.nt;
    dim3 grid((unsigned)((int64_t)nt * (nt + 1) / 2), (unsigned)w->nbb);
    const bool coh = w->mask & (CS_COH | CS_IMAGCOHY), plv = w->mask & CS_PLV;
    const int sel = (lag ? 4 : 0) | (coh ? 2 : 0) | (plv ? 1 : 0);
    switch (sel) {  // the metric families as template flags (no per-trial branches)
      case 1: cs::k_window_update<false, false, true><<<grid, cs::kWinThreads, 0, st>>>(a); break;
      case 2: cs::k_window_update<false, true, false><<<grid, cs::kWinThreads, 0, st>>>(a); break;
      case 3: cs::k_window_update<false, true, true><<<grid, cs::kWinThreads, 0, st>>>(a); break;
      case 4: cs::k_window_update<true, false, false><<<grid, cs::kWinThreads, 0, st>>>(a); break;
      case 5: cs::k_window_update<true, false, true><<<grid, cs::kWinThreads, 0, st>>>(a); break;
      case 6: cs::k_window_update<true, true, false><<<grid, cs::kWinThreads, 0, st>>>(a); break;
      default: cs::k_window_update<true, true, true><<<grid, cs::kWinThreads, 0, st>>>(a); break;
    }
  }
  if (lag) {  // exact fp64 values of the risky (pair, bin) entries over the whole window
    float* bins5[5] = {a.bins[2], a.bins[4], a.bins[5], a.bins[6], a.bins[7]};
    float* band5[5] = {a.band[2], a.band[4], a.band[5], a.band[6], a.band[7]};
    cs::run_window_fallback(p, window_slots, K, w->bin_lo, w->nbb, w->psd ? w->psd : p.psd, bins5, band5, w->recs,
                            st);
  }
  return cudaPeekAtLastError() == cudaSuccess ? CS_OK : CS_ECUDA;
}

}  // extern "C"
