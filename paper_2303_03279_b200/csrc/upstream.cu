// Upstream of the spectra: source projection and FIR filtering,
// hand-written on the fp64 tensor cores / CUDA cores.
//
// * k_dgemm: C(m, n) = sum_k A(m, k) B(n, k) with mma.sync m8n8k4 f64 (DMMA), 64 x 64
//   CTA tiles (four warps of 32 x 32, 4 x 4 fragments), k chunks of 32 staged in
//   shared memory (row stride 36 doubles: conflict-free fragment reads).  Operand
//   loaders and the epilogue are template functors, so one engine serves
//   - cs_apply_inverse (inverse.py:147-154): Y = M X, sensor -> source samples;
//   - cs_project_ring: the source spectra as M times the sensor spectra.  Demean,
//     taper and the DFT are linear per channel, so projecting the HBM spectrum ring
//     ([slot][taper][bin] rows x sensors, complex) replaces projecting K x T
//     samples and transforming N_src >> C source channels; the epilogue writes the
//     source plan's fp64 and scaled fp32 rings directly.
// * k_fir: streaming causal FIR (preprocess.py:109-142), direct form in fp64 with the
//   previous block's last n_taps - 1 input samples as history: the concatenated
//   output equals np.convolve(signal, taps)[:len(signal)], as the reference's
//   overlap-add does.
#include "common.cuh"

namespace cs {

constexpr int kGT = 64, kGKC = 32, kGRS = 36, kGThreads = 128;

__device__ __forceinline__ void dmma_f64(double& c0, double& c1, double a, double b) {
  asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};"
               : "+d"(c0), "+d"(c1)
               : "d"(a), "d"(b));
}

// row-major matrix loaders: K_CONTIG: element (r, k) at p[r * ld + k], else p[k * ld + r]
template <bool K_CONTIG>
struct Mat {
  const double* p;
  int64_t ld;
  int rows, K;
  __device__ double operator()(int r, int k) const {
    if (r >= rows || k >= K) return 0.0;
    return K_CONTIG ? p[(int64_t)r * ld + k] : p[(int64_t)k * ld + r];
  }
};
// the spectrum ring as a real matrix: row m = 2 r + part (part 0 = Re, 1 = Im) of ring row
// r (slot, taper, bin), column k = node
struct RingRows {
  const double* x;  // (const double*)X64 + first row's offset
  int64_t ldn;      // nodes per ring row
  int rows, K;
  __device__ double operator()(int m, int k) const {
    if (m >= rows || k >= K) return 0.0;
    return x[((int64_t)(m >> 1) * ldn + k) * 2 + (m & 1)];
  }
};

struct EpiStore {  // C[m * ld + n]
  double* c;
  int64_t ld;
  int M, N;
  __device__ void operator()(int m, int n, double v) const {
    if (m < M && n < N) c[(int64_t)m * ld + n] = v;
  }
};
struct EpiRing {   // destination ring row m >> 1, node n: fp64 and the scaled fp32 copy
  double* x64;
  float* x32;
  int64_t ldn;
  int M, N;
  float scale;
  __device__ void operator()(int m, int n, double v) const {
    if (m >= M || n >= N) return;
    const int64_t o = ((int64_t)(m >> 1) * ldn + n) * 2 + (m & 1);
    x64[o] = v;
    x32[o] = (float)(v * (double)scale);
  }
};

template <class LA, class LB, class EPI>
__global__ void __launch_bounds__(kGThreads) k_dgemm(LA A, LB B, EPI epi, int M, int N, int K) {
  __shared__ __align__(16) double As[kGT * kGRS];
  __shared__ __align__(16) double Bs[kGT * kGRS];
  const int m0 = blockIdx.y * kGT, n0 = blockIdx.x * kGT;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int wm = (warp >> 1) * 32, wn = (warp & 1) * 32;
  double acc[4][4][2];
#pragma unroll
  for (int a = 0; a < 4; ++a)
#pragma unroll
    for (int b = 0; b < 4; ++b) acc[a][b][0] = acc[a][b][1] = 0.0;
  for (int k0 = 0; k0 < K; k0 += kGKC) {
    __syncthreads();
    for (int e = threadIdx.x; e < kGT * kGKC; e += kGThreads) {
      // k fastest for k-contiguous operands (coalesced); the loaders bound-check
      const int r = e / kGKC, k = e % kGKC;
      As[r * kGRS + k] = A(m0 + r, k0 + k);
      Bs[r * kGRS + k] = B(n0 + r, k0 + k);
    }
    __syncthreads();
#pragma unroll
    for (int kk = 0; kk < kGKC; kk += 4) {
      double af[4], bf[4];
#pragma unroll
      for (int a = 0; a < 4; ++a) af[a] = As[(wm + a * 8 + (lane >> 2)) * kGRS + kk + (lane & 3)];
#pragma unroll
      for (int b = 0; b < 4; ++b) bf[b] = Bs[(wn + b * 8 + (lane >> 2)) * kGRS + kk + (lane & 3)];
#pragma unroll
      for (int a = 0; a < 4; ++a)
#pragma unroll
        for (int b = 0; b < 4; ++b) dmma_f64(acc[a][b][0], acc[a][b][1], af[a], bf[b]);
    }
  }
#pragma unroll
  for (int a = 0; a < 4; ++a)
#pragma unroll
    for (int b = 0; b < 4; ++b)
#pragma unroll
      for (int e = 0; e < 2; ++e)
        epi(m0 + wm + a * 8 + (lane >> 2), n0 + wn + b * 8 + 2 * (lane & 3) + e, acc[a][b][e]);
}

template <class LA, class LB, class EPI>
static void launch_dgemm(LA A, LB B, EPI epi, int M, int N, int K, cudaStream_t st) {
  dim3 grid((N + kGT - 1) / kGT, (M + kGT - 1) / kGT);
  k_dgemm<LA, LB, EPI><<<grid, kGThreads, 0, st>>>(A, B, epi, M, N, K);
}

// Streaming causal FIR: y[c][t] = sum_k h[k] xe[c][t - k], xe = [hist (n_taps - 1 samples), x].
constexpr int kFirT = 256, kFirH = 1024;
__global__ void __launch_bounds__(kFirT) k_fir(const double* __restrict__ h, int n_taps,
                                               const double* __restrict__ x, const double* __restrict__ hist,
                                               int S, double* __restrict__ y) {
  __shared__ double xs[kFirT + kFirH];
  __shared__ double hs[kFirH];
  const int c = blockIdx.y, t0 = blockIdx.x * kFirT, t = t0 + threadIdx.x;
  const int H = n_taps - 1;
  const double* xc = x + (int64_t)c * S;
  const double* hc = hist + (int64_t)c * H;
  double acc = 0.0;
  for (int k0 = 0; k0 < n_taps; k0 += kFirH) {  // taps in chunks: xe[t0 - k0 - kh + i]
    const int nk = min(kFirH, n_taps - k0);
    __syncthreads();
    for (int i = threadIdx.x; i < nk; i += kFirT) hs[i] = h[k0 + i];
    // samples t0 - k0 - (nk - 1) .. t0 + kFirT - 1 - k0
    const int base = t0 - k0 - (nk - 1);
    for (int i = threadIdx.x; i < kFirT + nk - 1; i += kFirT) {
      const int tt = base + i;
      xs[i] = tt >= 0 ? (tt < S ? xc[tt] : 0.0) : (tt + H >= 0 ? hc[tt + H] : 0.0);
    }
    __syncthreads();
    if (t < S) {
      // y[t] += sum_{kh < nk} h[k0 + kh] xe[t - k0 - kh];  xe[t - k0 - kh] = xs[threadIdx.x + nk - 1 - kh]
      const double* xp = xs + threadIdx.x + nk - 1;
      for (int kh = 0; kh < nk; ++kh) acc = fma(hs[kh], xp[-kh], acc);
    }
  }
  if (t < S) y[(int64_t)c * S + t] = acc;
}

// the new history: the last n_taps - 1 samples of [hist, x]
__global__ void k_fir_hist(const double* __restrict__ x, const double* __restrict__ hist, int C, int S, int H,
                           double* __restrict__ hist_out) {
  const int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (e >= (int64_t)C * H) return;
  const int c = (int)(e / H), j = (int)(e % H);
  const int tt = S - H + j;
  hist_out[e] = tt >= 0 ? x[(int64_t)c * S + tt] : hist[(int64_t)c * H + tt + H];
}

}  // namespace cs

extern "C" {

int cs_apply_inverse(const double* M, int n_src, int n_sens, const double* x, int n_samples, double* y,
                     void* stream) {
  if (!M || !x || !y || n_src < 1 || n_sens < 1 || n_samples < 1) {
    cs_set_error("cs_apply_inverse: bad argument");
    return CS_EPARAM;
  }
  // Y[n_src][T] = sum_c M[n][c] X[c][t]: A = M (k = sensor contiguous), B(t, c) = X[c][t]
  cs::launch_dgemm(cs::Mat<true>{M, n_sens, n_src, n_sens}, cs::Mat<false>{x, n_samples, n_samples, n_sens},
                   cs::EpiStore{y, n_samples, n_src, n_samples}, n_src, n_samples, n_sens, (cudaStream_t)stream);
  return cudaPeekAtLastError() == cudaSuccess ? CS_OK : CS_ECUDA;
}

int cs_project_ring(cs_plan* dst_plan, const cs_plan* src_plan, const double* M, int slot0, int k_count,
                    void* stream) {
  cs::Plan* d = (cs::Plan*)dst_plan;
  const cs::Plan* s = (const cs::Plan*)src_plan;
  if (!d || !s || !M) { cs_set_error("cs_project_ring: null argument"); return CS_EPARAM; }
  if (d->slot_cap != s->slot_cap || d->L != s->L || d->nb != s->nb) {
    cs_set_error("cs_project_ring: source and sensor rings differ in slots, tapers or bins");
    return CS_EPARAM;
  }
  if (slot0 < 0 || k_count < 0 || k_count > d->slot_cap) { cs_set_error("cs_project_ring: bad slots"); return CS_EPARAM; }
  if (k_count == 0) return CS_OK;
  cudaStream_t st = (cudaStream_t)stream;
  const int64_t rows_per_slot = (int64_t)d->L * d->nb;
  int sl = slot0 % d->slot_cap, left = k_count;
  while (left > 0) {  // slot runs that do not wrap the ring
    const int run = left < d->slot_cap - sl ? left : d->slot_cap - sl;
    const int rows = (int)(2 * run * rows_per_slot);
    const int64_t r0 = sl * rows_per_slot;
    cs::RingRows A{(const double*)(s->X64 + r0 * s->ldn), s->ldn, rows, s->N};
    cs::Mat<true> B{M, s->N, d->N, s->N};
    cs::EpiRing E{(double*)(d->X64 + r0 * d->ldn), (float*)(d->X32 + r0 * d->ldn), d->ldn, rows, d->N, d->scale};
    cs::launch_dgemm(A, B, E, rows, d->N, s->N, st);
    left -= run;
    sl = 0;
  }
  return cudaPeekAtLastError() == cudaSuccess ? CS_OK : CS_ECUDA;
}

int cs_fir_apply(const double* taps, int n_taps, const double* x, int n_channels, int n_samples,
                 const double* hist, double* hist_out, double* y, void* stream) {
  if (!taps || !x || !y || n_taps < 1 || n_channels < 1 || n_samples < 1 || (n_taps > 1 && (!hist || !hist_out))) {
    cs_set_error("cs_fir_apply: bad argument");
    return CS_EPARAM;
  }
  if (n_channels > 65535) { cs_set_error("cs_fir_apply: at most 65535 channels per call"); return CS_EPARAM; }
  cudaStream_t st = (cudaStream_t)stream;
  dim3 grid((n_samples + cs::kFirT - 1) / cs::kFirT, n_channels);
  // (one tap: no history is ever read; x stands in for the pointer)
  cs::k_fir<<<grid, cs::kFirT, 0, st>>>(taps, n_taps, x, n_taps > 1 ? hist : x, n_samples, y);
  if (n_taps > 1) {
    const int64_t n = (int64_t)n_channels * (n_taps - 1);
    cs::k_fir_hist<<<(unsigned)((n + 255) / 256), 256, 0, st>>>(x, hist, n_channels, n_samples, n_taps - 1, hist_out);
  }
  return cudaPeekAtLastError() == cudaSuccess ? CS_OK : CS_ECUDA;
}

}  // extern "C"
