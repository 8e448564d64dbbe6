// Time-domain metrics: the epilogues around library GEMM / FFT.
//
// COR (metrics.py:140-177): per trial the Pearson matrix is one Gram product
// u u^T of the demeaned, normalised channels (a plain GEMM, done by cuBLAS);
// k_cor_accumulate adds the clipped upper triangle to the running pair sums.
// XCOR (metrics.py:180-260): per trial the cross-correlations of all pairs come
// from one FFT per channel and an inverse FFT per pair (cuFFT); k_xcor_peaks
// normalises every lag by sqrt(overlap energy of x * energy of y) and takes the
// first maximum over lags [-max_lag, max_lag], one warp per pair.
#include "common.cuh"

namespace cs {

__global__ void k_cor_accumulate(const double* __restrict__ G, int C, int64_t p0, int64_t np,
                                 double* __restrict__ total) {
  const int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (e >= np) return;
  const int64_t p = p0 + e;
  int64_t i = (int64_t)((2.0 * C - 1.0 - sqrt((2.0 * C - 1.0) * (2.0 * C - 1.0) - 8.0 * (double)p)) / 2.0);
  if (i < 0) i = 0;
  while (i > 0 && pair_of(i, i + 1, C) > p) --i;
  while (i + 1 < C - 1 && pair_of(i + 1, i + 2, C) <= p) ++i;
  const int64_t j = p - pair_of(i, i + 1, C) + i + 1;
  const double g = G[i * C + j];
  total[e] += fmin(fmax(g, -1.0), 1.0);  // metrics.py:155
}

// cc: [npairs][nfft] circular cross-correlation r[tau] = sum_t dx[t + tau] dy[t]
// (negative tau at nfft + tau).  csq: [C][n + 1] prefix sums of dx^2.  ey: [C].
__global__ void k_xcor_peaks(const double* __restrict__ cc, int64_t npairs, int nfft, int n, int max_lag,
                             const int64_t* __restrict__ pi, const int64_t* __restrict__ pj,
                             const double* __restrict__ csq, const unsigned char* __restrict__ xzero,
                             double* __restrict__ peak_sum, double* __restrict__ lag_sum) {
  const int64_t warp = (blockIdx.x * (int64_t)blockDim.x + threadIdx.x) >> 5;
  const int lane = threadIdx.x & 31;
  if (warp >= npairs) return;
  const int64_t a = pi[warp], b = pj[warp];
  const double ey = csq[b * (n + 1) + n];
  double best = -1.0e308;
  int best_lag = 0;
  if (ey == 0.0 || xzero[a]) {  // metrics.py:203-204: (0.0, 0)
    best = 0.0;
  } else {
    const double* cx = csq + a * (n + 1);
    const double* r = cc + warp * (int64_t)nfft;
    for (int t = -max_lag + lane; t <= max_lag; t += 32) {
      const double ex = t >= 0 ? cx[n] - cx[t] : cx[n + t];
      const double den = sqrt(ex * ey);
      const double num = r[t >= 0 ? t : nfft + t];
      const double v = den > 0.0 ? num / den : 0.0;
      if (v > best) {  // lanes see ascending lags: strict > keeps the first maximum
        best = v;
        best_lag = t;
      }
    }
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {  // reduce: larger value, then smaller lag (np.argmax)
      const double ov = __shfl_xor_sync(0xffffffffu, best, o);
      const int ol = __shfl_xor_sync(0xffffffffu, best_lag, o);
      if (ov > best || (ov == best && ol < best_lag)) {
        best = ov;
        best_lag = ol;
      }
    }
  }
  if (lane == 0) {
    peak_sum[warp] += best;
    lag_sum[warp] += (double)best_lag;
  }
}

}  // namespace cs

extern "C" {

int cs_cor_accumulate(const double* G, int n_channels, int64_t pair_base, int64_t n_pairs, double* total,
                      void* stream) {
  if (!G || !total || n_channels < 2 || pair_base < 0 || n_pairs < 0) {
    cs_set_error("cs_cor_accumulate: bad argument");
    return CS_EPARAM;
  }
  if (n_pairs == 0) return CS_OK;
  cs::k_cor_accumulate<<<(unsigned)((n_pairs + 255) / 256), 256, 0, (cudaStream_t)stream>>>(G, n_channels, pair_base,
                                                                                             n_pairs, total);
  return cudaPeekAtLastError() == cudaSuccess ? CS_OK : CS_ECUDA;
}

int cs_xcor_peaks(const double* cc, int64_t n_pairs, int nfft, int n_samples, int max_lag, const int64_t* pi,
                  const int64_t* pj, const double* csq, const unsigned char* xzero, double* peak_sum,
                  double* lag_sum, void* stream) {
  if (!cc || !pi || !pj || !csq || !xzero || !peak_sum || !lag_sum || n_pairs < 0) {
    cs_set_error("cs_xcor_peaks: null argument");
    return CS_EPARAM;
  }
  if (max_lag < 0 || max_lag >= n_samples) { cs_set_error("max_lag must be < n_samples"); return CS_EPARAM; }
  if (nfft < 2 * n_samples - 1) { cs_set_error("nfft %d < 2 n - 1 (circular wrap)", nfft); return CS_EPARAM; }
  if (n_pairs == 0) return CS_OK;
  const int64_t threads = n_pairs * 32;
  cs::k_xcor_peaks<<<(unsigned)((threads + 255) / 256), 256, 0, (cudaStream_t)stream>>>(
      cc, n_pairs, nfft, n_samples, max_lag, pi, pj, csq, xzero, peak_sum, lag_sum);
  return cudaPeekAtLastError() == cudaSuccess ? CS_OK : CS_ECUDA;
}

}  // extern "C"
