// Time-domain metrics on the fp64 tensor cores: COR and XCOR of
// every channel pair, all trials of a call in one launch.
//
// COR (metrics.py:140-177): per trial the Pearson matrix is the Gram product u u^T of
// the demeaned, unit-norm channels; the clipped upper triangle is added to the pair
// sums (zero-variance channels: u = 0, so their edges are 0 as in the reference).
// XCOR (metrics.py:180-260): per trial and pair the peak over lags tau in
// [-max_lag, max_lag] of sum_t dx[t + tau] dy[t] / sqrt(overlap energy of x *
// energy of y); the first maximum wins (np.argmax), a constant x or y gives (0, 0).
// Both are one kernel over (32 x 32 pair tile, trial): the numerators of a lag are a
// "shifted Gram" of the tile's rows, computed with mma.sync m8n8k4 f64 (DMMA)
// from shared-memory row chunks, four warps on four lags at a time, the
// normalisation / argmax (or clip) fused into the epilogue.  The reference computes
// COR with a numpy matmul and XCOR with one fftconvolve per pair; the direct lag sum
// is its own checker (metrics.py:205-218) and what is computed here, in fp64.
#include "common.cuh"

namespace cs {

constexpr int kTdTile = 32;          // pair tile edge (rows i, columns j)
constexpr int kTdKC = 64;            // samples per staged chunk
constexpr int kTdHalo = 4;           // extra i-row samples: the 4 lags of a batch (one per warp)
constexpr int kTdRS = 72;            // smem row stride in doubles (72 = 8 mod 32 words: conflict-free)
constexpr int kTdThreads = 128;

// One warp per (trial, channel): demean, sum of squares, optional unit norm, prefix
// sums of dx^2 (XCOR overlap energies).  out: [K][C][T]; csq: [K][C][T + 1] or null;
// dead: [K][C] 1 for a zero-variance channel.
template <bool NORM>
__global__ void k_td_prep(const double* __restrict__ x, int K, int C, int T, double* __restrict__ out,
                          double* __restrict__ csq, unsigned char* __restrict__ dead) {
  const int64_t row = (blockIdx.x * (int64_t)blockDim.x + threadIdx.x) >> 5;
  const int lane = threadIdx.x & 31;
  if (row >= (int64_t)K * C) return;
  const double* xr = x + row * T;
  double s = 0.0;
  for (int t = lane; t < T; t += 32) s += xr[t];
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) s += __shfl_xor_sync(0xffffffffu, s, o);
  const double mean = s / (double)T;
  double q = 0.0;
  for (int t = lane; t < T; t += 32) {
    const double d = xr[t] - mean;
    q += d * d;
  }
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) q += __shfl_xor_sync(0xffffffffu, q, o);
  const double norm = sqrt(q);
  const bool z = NORM ? norm == 0.0 : q == 0.0;
  const double inv = (NORM && !z) ? 1.0 / norm : 1.0;
  double* orow = out + row * T;
  double run = 0.0;  // prefix sums of dx^2 in t order (chunks of 32, warp scan)
  if (csq && lane == 0) csq[row * (T + 1)] = 0.0;
  for (int t0 = 0; t0 < T; t0 += 32) {
    const int t = t0 + lane;
    const double d = t < T ? xr[t] - mean : 0.0;
    if (t < T) orow[t] = NORM ? (z ? 0.0 : d * inv) : d;
    if (csq) {
      double v = d * d;
#pragma unroll
      for (int o = 1; o < 32; o <<= 1) {
        const double u = __shfl_up_sync(0xffffffffu, v, o);
        if (lane >= o) v += u;
      }
      if (t < T) csq[row * (T + 1) + t + 1] = run + v;
      run += __shfl_sync(0xffffffffu, v, 31);
    }
  }
  if (lane == 0) dead[row] = z ? 1 : 0;
}

__device__ __forceinline__ void dmma(double& c0, double& c1, double a, double b) {
  asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};"
               : "+d"(c0), "+d"(c1)
               : "d"(a), "d"(b));
}

// XCOR = true: peaks over lags; false: COR (lag 0 only, clipped Gram of the unit rows).
// Grid: x = upper-triangle 32x32 tiles (I <= J), y = trial.  Warp w owns lag tau_b + w of
// each batch and all 32 x 32 pairs of the tile (4 x 4 DMMA fragments).
template <bool XCOR>
__global__ void __launch_bounds__(kTdThreads)
k_td_pairs(const double* __restrict__ D, const double* __restrict__ csq, const unsigned char* __restrict__ dead,
           int C, int T, int max_lag, int nt, double* __restrict__ out0, double* __restrict__ out1) {
  extern __shared__ __align__(16) double td_smem[];
  double* si = td_smem;                                   // i rows, samples t0 + tau_b + [0, KC + halo)
  double* sj = si + kTdTile * kTdRS;                      // j rows, samples t0 + [0, KC)
  double (*bval)[kTdTile * kTdTile] = (double (*)[kTdTile * kTdTile])(sj + kTdTile * kTdRS);
  int (*blag)[kTdTile * kTdTile] = (int (*)[kTdTile * kTdTile])(bval + 4);
  int I, J;
  decode_tile(blockIdx.x, nt, 0, I, J);
  const int k = blockIdx.y;
  const int i0 = I * kTdTile, j0 = J * kTdTile;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const double* Dk = D + (int64_t)k * C * T;
  const int L = XCOR ? max_lag : 0;

  // running maxima per warp in shared memory (registers hold the lag's accumulators);
  // this thread's entries: rows a*8 + (lane>>2), cols b*8 + 2*(lane&3) + {0,1}
  for (int e = lane; e < kTdTile * kTdTile; e += 32) {
    bval[warp][e] = -1.0e308;
    blag[warp][e] = 0;
  }

  for (int tau_b = -L; tau_b <= L; tau_b += 4) {
    const int tau = tau_b + warp;
    const bool lag_on = tau <= L;
    double acc[4][4][2];
#pragma unroll
    for (int a = 0; a < 4; ++a)
#pragma unroll
      for (int b = 0; b < 4; ++b) acc[a][b][0] = acc[a][b][1] = 0.0;
    // t range with an overlap for some lag of the batch: t + tau in [0, T) and t in [0, T)
    const int t_lo = max(0, -(tau_b + 3)), t_hi = min(T, T - tau_b);
    for (int t0 = t_lo; t0 < t_hi; t0 += kTdKC) {
      __syncthreads();
      // stage j rows (t0 .. t0 + KC) and i rows (t0 + tau_b .. + KC + halo), zeros outside [0, T)
      for (int e = threadIdx.x; e < kTdTile * kTdKC; e += kTdThreads) {
        const int r = e / kTdKC, c = e % kTdKC, t = t0 + c, n = j0 + r;
        sj[r * kTdRS + c] = (n < C && t < T) ? Dk[(int64_t)n * T + t] : 0.0;
      }
      for (int e = threadIdx.x; e < kTdTile * (kTdKC + kTdHalo); e += kTdThreads) {
        const int r = e / (kTdKC + kTdHalo), c = e % (kTdKC + kTdHalo), t = t0 + tau_b + c, n = i0 + r;
        si[r * kTdRS + c] = (n < C && t >= 0 && t < T) ? Dk[(int64_t)n * T + t] : 0.0;
      }
      __syncthreads();
      if (lag_on) {
        const int sh = warp;  // this warp's lag offset inside the staged i rows
#pragma unroll 4
        for (int kk = 0; kk < kTdKC; kk += 4) {
          double af[4], bf[4];
#pragma unroll
          for (int a = 0; a < 4; ++a) af[a] = si[(a * 8 + (lane >> 2)) * kTdRS + kk + (lane & 3) + sh];
#pragma unroll
          for (int b = 0; b < 4; ++b) bf[b] = sj[(b * 8 + (lane >> 2)) * kTdRS + kk + (lane & 3)];
#pragma unroll
          for (int a = 0; a < 4; ++a)
#pragma unroll
            for (int b = 0; b < 4; ++b) dmma(acc[a][b][0], acc[a][b][1], af[a], bf[b]);
        }
      }
    }
    if (!lag_on) continue;
    // epilogue of lag tau: COR clip, XCOR normalise + running first maximum
#pragma unroll
    for (int a = 0; a < 4; ++a) {
      const int i = i0 + a * 8 + (lane >> 2);
      double ex = 0.0;
      if (XCOR && i < C) {
        const double* ci = csq + ((int64_t)k * C + i) * (T + 1);
        ex = tau >= 0 ? ci[T] - ci[tau] : ci[T + tau];
      }
#pragma unroll
      for (int b = 0; b < 4; ++b)
#pragma unroll
        for (int e = 0; e < 2; ++e) {
          const int j = j0 + b * 8 + 2 * (lane & 3) + e;
          double v = acc[a][b][e];
          if (XCOR) {
            const double ey = j < C ? csq[((int64_t)k * C + j) * (T + 1) + T] : 0.0;
            const double den = sqrt(ex * ey);
            v = den > 0.0 ? v / den : 0.0;
          }
          const int q = (a * 8 + (lane >> 2)) * kTdTile + b * 8 + 2 * (lane & 3) + e;
          if (v > bval[warp][q]) {  // ascending lags per warp: strict > keeps the first maximum
            bval[warp][q] = v;
            blag[warp][q] = tau;
          }
        }
    }
  }
  // merge the four warps' maxima (larger value, then smaller lag) and accumulate
  __syncthreads();
  for (int e = threadIdx.x; e < kTdTile * kTdTile; e += kTdThreads) {
    const int r = e / kTdTile, c = e % kTdTile, i = i0 + r, j = j0 + c;
    if (!(i < j && j < C)) continue;
    double v = bval[0][e];
    int lg = blag[0][e];
    for (int w = 1; w < 4; ++w)  // (a warp that never had a lag holds -1e308)
      if (bval[w][e] > v || (bval[w][e] == v && blag[w][e] < lg)) {
        v = bval[w][e];
        lg = blag[w][e];
      }
    const int64_t p = pair_of(i, j, C);
    if (XCOR) {
      if (dead[(int64_t)k * C + i] || dead[(int64_t)k * C + j]) {  // metrics.py:203-204
        v = 0.0;
        lg = 0;
      }
      atomicAdd(&out0[p], v);
      atomicAdd(&out1[p], (double)lg);
    } else {
      atomicAdd(&out0[p], fmin(fmax(v, -1.0), 1.0));  // metrics.py:155
    }
  }
}

static int run_td(const double* x, int K, int C, int T, int max_lag, bool xcor, double* out0, double* out1,
                  unsigned char* dead_out, cudaStream_t st) {
  const int64_t rows = (int64_t)K * C;
  double *D = nullptr, *csq = nullptr;
  unsigned char* dead = nullptr;
  if (cudaMallocAsync(&D, rows * T * sizeof(double), st) != cudaSuccess ||
      (xcor && cudaMallocAsync(&csq, rows * (T + 1) * sizeof(double), st) != cudaSuccess) ||
      cudaMallocAsync(&dead, rows, st) != cudaSuccess) {
    cudaGetLastError();
    if (D) cudaFreeAsync(D, st);
    if (csq) cudaFreeAsync(csq, st);
    cs_set_error("device allocation failed (time-domain scratch)");
    return CS_ENOMEM;
  }
  const unsigned pb = (unsigned)((rows * 32 + 255) / 256);
  if (xcor)
    k_td_prep<false><<<pb, 256, 0, st>>>(x, K, C, T, D, csq, dead);
  else
    k_td_prep<true><<<pb, 256, 0, st>>>(x, K, C, T, D, nullptr, dead);
  const int nt = (C + kTdTile - 1) / kTdTile;
  dim3 grid((unsigned)((int64_t)nt * (nt + 1) / 2), (unsigned)K);
  const size_t smem = (size_t)2 * kTdTile * kTdRS * 8 + 4 * kTdTile * kTdTile * (8 + 4);
  if (xcor) {
    CS_SMEM_ONCE(k_td_pairs<true>, smem);
    k_td_pairs<true><<<grid, kTdThreads, smem, st>>>(D, csq, dead, C, T, max_lag, nt, out0, out1);
  } else {
    CS_SMEM_ONCE(k_td_pairs<false>, smem);
    k_td_pairs<false><<<grid, kTdThreads, smem, st>>>(D, nullptr, dead, C, T, 0, nt, out0, nullptr);
  }
  cudaFreeAsync(D, st);
  if (csq) cudaFreeAsync(csq, st);
  // zero-variance flags per (trial, channel): the reference's warnings
  if (dead_out) cudaMemcpyAsync(dead_out, dead, rows, cudaMemcpyDeviceToDevice, st);
  cudaFreeAsync(dead, st);
  return cudaPeekAtLastError() == cudaSuccess ? CS_OK : CS_ECUDA;
}

}  // namespace cs

extern "C" {

int cs_cor_sums(const double* x, int n_trials, int n_channels, int n_samples, double* total,
                unsigned char* dead, void* stream) {
  if (!x || !total || n_trials < 0 || n_channels < 1 || n_samples < 2) {
    cs_set_error("cs_cor_sums: bad argument");
    return CS_EPARAM;
  }
  if (n_trials == 0 || n_channels < 2) return CS_OK;
  if (n_trials > 65535) { cs_set_error("cs_cor_sums: at most 65535 trials per call"); return CS_EPARAM; }
  return cs::run_td(x, n_trials, n_channels, n_samples, 0, false, total, nullptr, dead, (cudaStream_t)stream);
}

int cs_xcor_sums(const double* x, int n_trials, int n_channels, int n_samples, int max_lag, double* peak_sum,
                 double* lag_sum, unsigned char* dead, void* stream) {
  if (!x || !peak_sum || !lag_sum || n_trials < 0 || n_channels < 1 || n_samples < 2) {
    cs_set_error("cs_xcor_sums: bad argument");
    return CS_EPARAM;
  }
  if (max_lag < 0 || max_lag >= n_samples) { cs_set_error("max_lag must be < n_samples"); return CS_EPARAM; }
  if (n_trials == 0 || n_channels < 2) return CS_OK;
  if (n_trials > 65535) { cs_set_error("cs_xcor_sums: at most 65535 trials per call"); return CS_EPARAM; }
  return cs::run_td(x, n_trials, n_channels, n_samples, max_lag, true, peak_sum, lag_sum, dead,
                    (cudaStream_t)stream);
}

}  // extern "C"
