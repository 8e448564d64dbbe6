// SpectrumSet running sums (the reference's accumulator state) from the fp64
// spectrum ring: the accessor behind SpectrumSet.csd_sum / plv_sum / pli_sum /
// abs_im_sum / psd_sum.  Not on the metric path (the metric kernels fuse the
// finalisers and never materialise these [P, B] arrays).
//
// Reference: spectral.py:204-213 (trial_csd_psd), :216-241 (_fold_csd: Im flush,
// unit phasor, sign, |Im|), :136-141 (the sums).  One thread per (pair, bin),
// consecutive threads on consecutive j of one row i, so the ring reads of X_j
// are coalesced and X_i is a broadcast.
#include <cfloat>

#include "common.cuh"

namespace cs {

__global__ void k_pair_sums(const double2* __restrict__ X64, const int* __restrict__ slots, int K, int N, int nb,
                            int L, int bin_lo, int nbb, int64_t p0, int64_t np, int64_t stride, double2* __restrict__ csd,
                            double2* __restrict__ plv, int* __restrict__ pli, double* __restrict__ abs_im) {
  const int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  const int bl = blockIdx.y;
  if (e >= np) return;
  // pair index p0 + e -> (i, j)
  const int64_t p = p0 + e;
  int64_t i = (int64_t)((2.0 * N - 1.0 - sqrt((2.0 * N - 1.0) * (2.0 * N - 1.0) - 8.0 * (double)p)) / 2.0);
  if (i < 0) i = 0;
  while (i > 0 && pair_of(i, i + 1, N) > p) --i;
  while (i + 1 < N - 1 && pair_of(i + 1, i + 2, N) <= p) ++i;
  const int64_t j = p - pair_of(i, i + 1, N) + i + 1;
  const int b = bin_lo + bl;
  const int64_t slot_stride = (int64_t)L * nb * N;
  double cr = 0.0, ci = 0.0, ur = 0.0, ui = 0.0, ab = 0.0;
  int sg = 0;
  for (int k = 0; k < K; ++k) {
    const int64_t base = slots[k] * slot_stride + (int64_t)b * N;
    double re = 0.0, im = 0.0;
    for (int l = 0; l < L; ++l) {
      const double2 xi = X64[base + (int64_t)l * nb * N + i];
      const double2 xj = X64[base + (int64_t)l * nb * N + j];
      re += xi.x * xj.x + xi.y * xj.y;  // X_i conj X_j
      im += xi.y * xj.x - xi.x * xj.y;
    }
    if (fabs(im) <= 1e-13 * fabs(re)) im = 0.0;  // spectral.py:227-228
    cr += re;
    ci += im;
    const double mag = hypot(re, im);
    if (mag > DBL_MIN) {  // spectral.py:229-233
      ur += re / mag;
      ui += im / mag;
    }
    sg += (im > 0.0) - (im < 0.0);
    ab += fabs(im);
  }
  const int64_t o = (int64_t)bl * stride + e;
  if (csd) csd[o] = make_double2(cr, ci);
  if (plv) plv[o] = make_double2(ur, ui);
  if (pli) pli[o] = sg;
  if (abs_im) abs_im[o] = ab;
}

__global__ void k_psd_sums(const double2* __restrict__ X64, const int* __restrict__ slots, int K, int N, int nb,
                           int L, int bin_lo, double* __restrict__ psd) {
  const int n = blockIdx.x * blockDim.x + threadIdx.x;
  const int bl = blockIdx.y;
  if (n >= N) return;
  const int b = bin_lo + bl;
  double s = 0.0;
  for (int k = 0; k < K; ++k)
    for (int l = 0; l < L; ++l) {
      const double2 x = X64[((int64_t)slots[k] * L + l) * nb * N + (int64_t)b * N + n];
      s += x.x * x.x + x.y * x.y;
    }
  psd[(int64_t)bl * N + n] = s;
}

void run_pair_sums(const Plan& p, const int* slots, int K, int bin_lo, int nbb, const cs_sums* out,
                   cudaStream_t st) {
  const int64_t P = (int64_t)p.N * (p.N - 1) / 2;
  const int64_t p0 = out->pair_base < 0 ? 0 : out->pair_base;
  int64_t np = out->pair_stride;
  if (p0 + np > P) np = P - p0;
  if (np > 0 && (out->csd || out->plv || out->pli || out->abs_im)) {
    dim3 grid((unsigned)((np + 255) / 256), nbb);
    k_pair_sums<<<grid, 256, 0, st>>>(p.X64, slots, K, p.N, p.nb, p.L, bin_lo, nbb, p0, np, out->pair_stride,
                                      (double2*)out->csd, (double2*)out->plv, out->pli, out->abs_im);
  }
  if (out->psd) {
    dim3 grid((unsigned)((p.N + 255) / 256), nbb);
    k_psd_sums<<<grid, 256, 0, st>>>(p.X64, slots, K, p.N, p.nb, p.L, bin_lo, out->psd);
  }
}

}  // namespace cs
