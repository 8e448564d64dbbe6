// K1: batched demean + taper + one-sided DFT of every node x trial x taper, in
// fp64, writing the HBM spectrum ring (fp64 copy for the exact-sign guard, fp32
// scaled copy for the pair kernels).
//
// Reference: spectral.py:49-62 (_crop_pad_demean: crop to nfft or zero-pad,
// demean over the real samples), spectral.py:82-97 (rfft, DC := 0).  Taper
// extension (SURVEY.md conventions 11): demean, then taper, then zero-pad.
//
// Only the plan's bins [lo, hi] are produced, so the transform is a dense
// [signals x T_eff] x [T_eff x nb] complex contraction: each CTA stages a
// 128-node x 32-sample block (coalesced rows) transposed into shared memory, one
// thread per node accumulates up to NBT bins in fp64 registers, twiddles are
// broadcast from shared memory.  DFMA-bound (B200: 64 DFMA/clk/SM).
#include "common.cuh"

namespace cs {

constexpr int kSpecNodes = 128;   // one thread per node
constexpr int kSpecRowBytes = 128; // staged samples per row per chunk (32 fp32 / 16 fp64)

__device__ __forceinline__ void cp_async16(void* smem, const void* gmem, int src_bytes) {
  const unsigned s = (unsigned)__cvta_generic_to_shared(smem);
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16, %2;\n" ::"r"(s), "l"(gmem), "r"(src_bytes));
}
__device__ __forceinline__ void cp_async4(void* smem, const void* gmem, int src_bytes) {
  const unsigned s = (unsigned)__cvta_generic_to_shared(smem);
  asm volatile("cp.async.ca.shared.global [%0], [%1], 4, %2;\n" ::"r"(s), "l"(gmem), "r"(src_bytes));
}
template <typename T>
__device__ __forceinline__ void cp_async4_any(T* smem, const T* gmem) {  // one element
  const unsigned s = (unsigned)__cvta_generic_to_shared(smem);
  asm volatile("cp.async.ca.shared.global [%0], [%1], %2;\n" ::"r"(s), "l"(gmem), "n"(sizeof(T)));
}
__device__ __forceinline__ void cp_async_commit() { asm volatile("cp.async.commit_group;\n" ::); }
__device__ __forceinline__ void cp_async_wait1() { asm volatile("cp.async.wait_group 1;\n" ::); }
__device__ __forceinline__ void cp_async_wait0() { asm volatile("cp.async.wait_group 0;\n" ::); }

// Single pass over the samples.  With d_t = x_t - c (c = first sample of the row,
// exact in fp64 for fp32 input) the demeaned, tapered DFT is
//   X_b = sum_t (d_t - mean(d)) w_t e_bt = Y_b - mean(d) W_b,  Y_b = sum_t d_t tww_bt,
// W_b = sum_t tww_bt (host, long double), so the mean never needs a second read.
// NS signals per thread share every broadcast twiddle load (NS = 2 for <= 8 bins:
// 24 DFMA per 6 LDS.128 instead of 12).
template <typename Tin, int NBT, int NS>
struct SpecShape {
  static constexpr int ROWS = kSpecNodes * NS;                       // nodes per CTA
  static constexpr int TC = (NS == 1 ? kSpecRowBytes : kSpecRowBytes / 2) / (int)sizeof(Tin);  // samples per chunk
  static constexpr int RS = TC + 16 / (int)sizeof(Tin);             // padded row stride (conflict-free LDS.128)
  static constexpr size_t SMEM = 2 * (size_t)ROWS * RS * sizeof(Tin) + 2 * (size_t)NBT * TC * sizeof(double2);
};

template <typename Tin, int NBT, int NS>
__global__ void __launch_bounds__(kSpecNodes)
k_spectra(const Tin* __restrict__ x, int64_t trial_stride, int64_t node_stride, int N,
          int T_eff, int nb, int L, const double2* __restrict__ tww, const double2* __restrict__ wsum,
          int slot0, int slot_cap, double2* __restrict__ X64, float2* __restrict__ X32, float scale,
          int dc_local, int nyq_local, int vec16, int seg_stride, int ldn) {
  using Sh = SpecShape<Tin, NBT, NS>;
  constexpr int ROWS = Sh::ROWS, TC = Sh::TC, RS = Sh::RS;
  extern __shared__ __align__(16) unsigned char spec_smem[];
  Tin* sx = (Tin*)spec_smem;                                  // [2][ROWS][RS]
  double2* stw = (double2*)(spec_smem + 2 * ROWS * RS * sizeof(Tin));  // [2][NBT][TC]

  const int tid = threadIdx.x;
  const int n0 = blockIdx.x * ROWS;
  const int b0 = blockIdx.y * NBT;
  const int k = blockIdx.z / L;
  const int l = blockIdx.z % L;
  const int nbt = min(NBT, nb - b0);
  const Tin* xk = x + (int64_t)k * trial_stride + (int64_t)l * seg_stride;  // welch: segment l
  const double2* twl = tww + ((int64_t)l * nb + b0) * T_eff;
  const int n_chunk = (T_eff + TC - 1) / TC;

  auto issue = [&](int ch, int buf) {
    const int t0 = ch * TC;
    Tin* dst = sx + buf * ROWS * RS;
    if (vec16) {
      constexpr int EPP = 16 / sizeof(Tin);         // elements per 16-byte piece
      constexpr int PER_ROW = TC / EPP;             // pieces per row
#pragma unroll 4
      for (int q = 0; q < PER_ROW * NS; ++q) {
        const int e = tid + kSpecNodes * q;
        const int row = e / PER_ROW, piece = e % PER_ROW;
        const int n = n0 + row, t = t0 + piece * EPP;
        int bytes = 0;
        if (n < N && t < T_eff) bytes = min(EPP, T_eff - t) * (int)sizeof(Tin);
        const Tin* src = bytes ? xk + (int64_t)n * node_stride + t : xk;
        cp_async16(dst + row * RS + piece * EPP, src, bytes);
      }
    } else {
      for (int q = 0; q < TC * NS; ++q) {
        const int e = tid + kSpecNodes * q;
        const int row = e / TC, col = e % TC;
        const int n = n0 + row, t = t0 + col;
        const bool ok = n < N && t < T_eff;
        const Tin* src = ok ? xk + (int64_t)n * node_stride + t : xk;
        if (sizeof(Tin) == 4) {
          cp_async4(dst + row * RS + col, src, ok ? 4 : 0);
        } else {
          cp_async4(dst + row * RS + col, src, ok ? 4 : 0);
          cp_async4((char*)(dst + row * RS + col) + 4, (const char*)src + 4, ok ? 4 : 0);
        }
      }
    }
    double2* tdst = stw + buf * NBT * TC;
    for (int e = tid; e < NBT * TC; e += kSpecNodes) {
      const int j = e / TC, t = e % TC;
      const bool ok = j < nbt && t0 + t < T_eff;
      cp_async16(tdst + e, ok ? (const void*)(twl + (int64_t)j * T_eff + t0 + t) : (const void*)twl, ok ? 16 : 0);
    }
    cp_async_commit();
  };

  double are[NS][NBT], aim[NS][NBT];
#pragma unroll
  for (int q = 0; q < NS; ++q)
#pragma unroll
    for (int j = 0; j < NBT; ++j) are[q][j] = aim[q][j] = 0.0;
  double c[NS], sum[NS];
#pragma unroll
  for (int q = 0; q < NS; ++q) c[q] = sum[q] = 0.0;

  issue(0, 0);
  for (int ch = 0; ch < n_chunk; ++ch) {
    const int buf = ch & 1;
    if (ch + 1 < n_chunk) {
      issue(ch + 1, buf ^ 1);
      cp_async_wait1();
    } else {
      cp_async_wait0();
    }
    __syncthreads();
    const Tin* rows = sx + buf * ROWS * RS;
    const double2* tw = stw + buf * NBT * TC;
    if (ch == 0) {
#pragma unroll
      for (int q = 0; q < NS; ++q) c[q] = (double)rows[(tid + kSpecNodes * q) * RS];
    }
    const int tn = min(TC, T_eff - ch * TC);
    if (tn == TC) {
      constexpr int VE = 16 / sizeof(Tin);
#pragma unroll 2
      for (int t = 0; t < TC; t += VE) {
        Tin v[NS][VE];
#pragma unroll
        for (int q = 0; q < NS; ++q) *(float4*)v[q] = *(const float4*)(rows + (tid + kSpecNodes * q) * RS + t);
#pragma unroll
        for (int u = 0; u < VE; ++u) {
          double d[NS];
#pragma unroll
          for (int q = 0; q < NS; ++q) {
            d[q] = (double)v[q][u] - c[q];
            sum[q] += d[q];
          }
#pragma unroll
          for (int j = 0; j < NBT; ++j) {
            const double2 w = tw[j * TC + t + u];
#pragma unroll
            for (int q = 0; q < NS; ++q) {
              are[q][j] = fma(d[q], w.x, are[q][j]);
              aim[q][j] = fma(d[q], w.y, aim[q][j]);
            }
          }
        }
      }
    } else {
      for (int t = 0; t < tn; ++t) {
        double d[NS];
#pragma unroll
        for (int q = 0; q < NS; ++q) {
          d[q] = (double)rows[(tid + kSpecNodes * q) * RS + t] - c[q];
          sum[q] += d[q];
        }
#pragma unroll
        for (int j = 0; j < NBT; ++j) {
          const double2 w = tw[j * TC + t];
#pragma unroll
          for (int q = 0; q < NS; ++q) {
            are[q][j] = fma(d[q], w.x, are[q][j]);
            aim[q][j] = fma(d[q], w.y, aim[q][j]);
          }
        }
      }
    }
    __syncthreads();
  }

  const int slot = (slot0 + k) % slot_cap;
#pragma unroll
  for (int q = 0; q < NS; ++q) {
    const int n = n0 + tid + kSpecNodes * q;
    if (n >= N) continue;
    const double mean = sum[q] / (double)T_eff;
#pragma unroll
    for (int j = 0; j < NBT; ++j) {
      if (j >= nbt) break;
      const int b = b0 + j;
      const double2 W = wsum[(int64_t)l * nb + b];
      double re = fma(-mean, W.x, are[q][j]), im = fma(-mean, W.y, aim[q][j]);
      if (b == dc_local) re = im = 0.0;       // spectral.py:96: DC is exactly zero
      if (b == nyq_local) im = 0.0;           // Nyquist of a real signal is real
      const int64_t o = (((int64_t)slot * L + l) * nb + b) * ldn + n;  // ring rows of ldn nodes
      X64[o] = make_double2(re, im);
      X32[o] = make_float2((float)(re * (double)scale), (float)(im * (double)scale));
    }
  }
}

template <typename Tin, int NBT>
static void launch_spectra(const Plan& p, const void* x, int64_t ts, int64_t ns, int slot0,
                           int kc, cudaStream_t st) {
  constexpr int NS = NBT <= 8 ? 2 : 1;
  using Sh = SpecShape<Tin, NBT, NS>;
  const size_t smem = Sh::SMEM;
  CS_SMEM_ONCE((k_spectra<Tin, NBT, NS>), smem);
  const int vec16 = ((uintptr_t)x % 16 == 0) && ((ns * (int64_t)sizeof(Tin)) % 16 == 0) &&
                    ((ts * (int64_t)sizeof(Tin)) % 16 == 0) && ((p.seg_stride * (int64_t)sizeof(Tin)) % 16 == 0);
  dim3 grid((p.N + Sh::ROWS - 1) / Sh::ROWS, (p.nb + NBT - 1) / NBT, kc * p.L);
  k_spectra<Tin, NBT, NS><<<grid, kSpecNodes, smem, st>>>((const Tin*)x, ts, ns, p.N, p.T_eff, p.nb,
                                                           p.L, p.tww, p.wsum, slot0, p.slot_cap, p.X64,
                                                           p.X32, p.scale, p.dc_local, p.nyq_local, vec16,
                                                           p.seg_stride, p.ldn);
}

// ---------------------------------------------------------------------------
// DFT on the fp64 tensor cores (mma.sync m8n8k4 f64, B200: 18.5 T FMA/s vs 17 for
// DFMA, with 1/8 of the instructions).  Per warp: 8 signals x 4 samples (A) times
// 4 samples x 8 columns (B) per MMA; columns are (Re, Im) of each plan bin plus one
// column of ones (sum of the shifted samples, for the mean correction), padded to
// NT x 8.  B fragments come from a host table already in fragment order
// (tf[l][k-step][nt][lane]), so every lane reads consecutive doubles.
constexpr int kDW = 8;                 // warps per CTA
constexpr int kDRows = 8 * kDW;        // signals per CTA
constexpr int kDTC = 64;               // samples per staged chunk

template <typename Tin, int NT>
__global__ void __launch_bounds__(kDW * 32)
k_spectra_dmma(const Tin* __restrict__ x, int64_t trial_stride, int64_t node_stride, int N, int T_eff, int nb,
               int L, const double* __restrict__ tf, const double2* __restrict__ wsum, int slot0, int slot_cap,
               double2* __restrict__ X64, float2* __restrict__ X32, float scale, int dc_local, int nyq_local,
               int vec16, int seg_stride, int ldn) {
  constexpr int RS = kDTC + 16 / (int)sizeof(Tin);        // padded row (conflict-free A-fragment reads)
  constexpr int KS = kDTC / 4;                             // k-steps per chunk
  extern __shared__ __align__(16) unsigned char dm_smem[];
  Tin* sx = (Tin*)dm_smem;                                                  // [2][64][RS]
  double* stf = (double*)(dm_smem + 2 * kDRows * RS * sizeof(Tin));        // [2][KS][NT][32]
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const int n0 = blockIdx.x * kDRows;
  const int k = blockIdx.y / L, l = blockIdx.y % L;
  const Tin* xk = x + (int64_t)k * trial_stride + (int64_t)l * seg_stride;
  const int nks = (T_eff + 3) / 4;                         // k-steps over the signal
  const double* tfl = tf + (int64_t)l * nks * NT * 32;
  const int n_chunk = (T_eff + kDTC - 1) / kDTC;

  auto issue = [&](int ch, int buf) {
    const int t0 = ch * kDTC;
    Tin* dst = sx + buf * kDRows * RS;
    if (vec16) {
      constexpr int EPP = 16 / sizeof(Tin), PER_ROW = kDTC / EPP;
      for (int e = tid; e < kDRows * PER_ROW; e += kDW * 32) {
        const int row = e / PER_ROW, piece = e % PER_ROW;
        const int n = n0 + row, t = t0 + piece * EPP;
        int bytes = 0;
        if (n < N && t < T_eff) bytes = min(EPP, T_eff - t) * (int)sizeof(Tin);
        cp_async16(dst + row * RS + piece * EPP, bytes ? xk + (int64_t)n * node_stride + t : xk, bytes);
      }
    } else {
      for (int e = tid; e < kDRows * kDTC; e += kDW * 32) {
        const int row = e / kDTC, col = e % kDTC;
        const int n = n0 + row, t = t0 + col;
        const bool ok = n < N && t < T_eff;
        const Tin* src = ok ? xk + (int64_t)n * node_stride + t : xk;
        cp_async4(dst + row * RS + col, src, ok ? 4 : 0);
        if (sizeof(Tin) == 8) cp_async4((char*)(dst + row * RS + col) + 4, (const char*)src + 4, ok ? 4 : 0);
      }
    }
    double* tdst = stf + buf * KS * NT * 32;
    const int k0 = ch * KS;
    for (int e = tid; e < KS * NT * 16; e += kDW * 32) {   // 16-byte pieces
      const int kk = k0 + e / (NT * 16);
      const bool ok = kk < nks;
      cp_async16(tdst + 2 * e, ok ? (const void*)(tfl + (int64_t)k0 * NT * 32 + 2 * e) : (const void*)tfl, ok ? 16 : 0);
    }
    cp_async_commit();
  };

  const int row = warp * 8 + (lane >> 2), q = lane & 3;
  double acc[NT][2];
#pragma unroll
  for (int nt = 0; nt < NT; ++nt) acc[nt][0] = acc[nt][1] = 0.0;
  double c = 0.0;

  issue(0, 0);
  for (int ch = 0; ch < n_chunk; ++ch) {
    const int buf = ch & 1;
    if (ch + 1 < n_chunk) {
      issue(ch + 1, buf ^ 1);
      cp_async_wait1();
    } else {
      cp_async_wait0();
    }
    __syncthreads();
    const Tin* rs = sx + buf * kDRows * RS + row * RS;
    const double* tb = stf + buf * KS * NT * 32;
    if (ch == 0) c = (double)rs[0];
    const int t0 = ch * kDTC;
#pragma unroll
    for (int kk = 0; kk < KS; ++kk) {
      const int t = t0 + 4 * kk + q;
      const double av = t < T_eff ? (double)rs[4 * kk + q] - c : 0.0;
#pragma unroll
      for (int nt = 0; nt < NT; ++nt) {
        const double bv = tb[(kk * NT + nt) * 32 + lane];
        asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};"
                     : "+d"(acc[nt][0]), "+d"(acc[nt][1]) : "d"(av), "d"(bv));
      }
    }
    __syncthreads();
  }

  // lane holds row `row`, columns (2 q + 8 nt, 2 q + 8 nt + 1) = (Re, Im) of bin 4 nt + q;
  // the ones column 2 nb sits at (nt = nb / 4, q = nb % 4, element 0)
  double sum_d = 0.0;
#pragma unroll
  for (int nt = 0; nt < NT; ++nt)
    if (nt == nb / 4) sum_d = acc[nt][0];
  sum_d = __shfl_sync(0xffffffffu, sum_d, (lane & ~3) | (nb & 3));
  const int n = n0 + row;
  if (n >= N) return;
  const double mean = sum_d / (double)T_eff;
  const int slot = (slot0 + k) % slot_cap;
#pragma unroll
  for (int nt = 0; nt < NT; ++nt) {
    const int b = 4 * nt + q;
    if (b >= nb) continue;
    const double2 W = wsum[(int64_t)l * nb + b];
    double re = fma(-mean, W.x, acc[nt][0]), im = fma(-mean, W.y, acc[nt][1]);
    if (b == dc_local) re = im = 0.0;       // spectral.py:96
    if (b == nyq_local) im = 0.0;
    const int64_t o = (((int64_t)slot * L + l) * nb + b) * ldn + n;  // ring rows of ldn nodes
    X64[o] = make_double2(re, im);
    X32[o] = make_float2((float)(re * (double)scale), (float)(im * (double)scale));
  }
}

template <typename Tin, int NT>
static void launch_dmma(const Plan& p, const void* x, int64_t ts, int64_t ns, int slot0, int kc, cudaStream_t st) {
  constexpr int RS = kDTC + 16 / (int)sizeof(Tin);
  const size_t smem = 2 * (size_t)kDRows * RS * sizeof(Tin) + 2 * (size_t)(kDTC / 4) * NT * 32 * sizeof(double);
  CS_SMEM_ONCE((k_spectra_dmma<Tin, NT>), smem);
  const int vec16 = ((uintptr_t)x % 16 == 0) && ((ns * (int64_t)sizeof(Tin)) % 16 == 0) &&
                    ((ts * (int64_t)sizeof(Tin)) % 16 == 0) && ((p.seg_stride * (int64_t)sizeof(Tin)) % 16 == 0);
  dim3 grid((p.N + kDRows - 1) / kDRows, kc * p.L);
  k_spectra_dmma<Tin, NT><<<grid, kDW * 32, smem, st>>>((const Tin*)x, ts, ns, p.N, p.T_eff, p.nb, p.L, p.dft_tf,
                                                         p.wsum, slot0, p.slot_cap, p.X64, p.X32, p.scale, p.dc_local,
                                                         p.nyq_local, vec16, p.seg_stride, p.ldn);
}

template <typename Tin>
static void dispatch_spectra(const Plan& p, const void* x, int64_t ts, int64_t ns, int slot0,
                             int kc, cudaStream_t st) {
  if (p.dft_tf) {  // fp64 tensor-core DFT (2 nb + 1 columns <= 24)
    const int nt = (2 * p.nb + 1 + 7) / 8;
    if (nt <= 1) launch_dmma<Tin, 1>(p, x, ts, ns, slot0, kc, st);
    else if (nt == 2) launch_dmma<Tin, 2>(p, x, ts, ns, slot0, kc, st);
    else launch_dmma<Tin, 3>(p, x, ts, ns, slot0, kc, st);
    return;
  }
  // per-thread bin count: wide bands use 16-bin chunks on gridDim.y
  switch (p.nb) {
    case 1: launch_spectra<Tin, 1>(p, x, ts, ns, slot0, kc, st); break;
    case 2: launch_spectra<Tin, 2>(p, x, ts, ns, slot0, kc, st); break;
    case 3: launch_spectra<Tin, 3>(p, x, ts, ns, slot0, kc, st); break;
    case 4: launch_spectra<Tin, 4>(p, x, ts, ns, slot0, kc, st); break;
    case 5: launch_spectra<Tin, 5>(p, x, ts, ns, slot0, kc, st); break;
    case 6: launch_spectra<Tin, 6>(p, x, ts, ns, slot0, kc, st); break;
    case 7:
    case 8: launch_spectra<Tin, 8>(p, x, ts, ns, slot0, kc, st); break;
    case 9:
    case 10:
    case 11:
    case 12: launch_spectra<Tin, 12>(p, x, ts, ns, slot0, kc, st); break;
    default: launch_spectra<Tin, 16>(p, x, ts, ns, slot0, kc, st); break;
  }
}

bool run_spectra_fft(const Plan& p, const void* x, int dtype, int64_t ts, int64_t ns, int slot0, int kc,
                     cudaStream_t st);

void run_spectra(const Plan& p, const void* x, int dtype, int64_t ts, int64_t ns, int slot0,
                 int kc, cudaStream_t st) {
  if (p.use_fft) {
    run_spectra_fft(p, x, dtype, ts, ns, slot0, kc, st);
    return;
  }
  if (dtype == CS_F64)
    dispatch_spectra<double>(p, x, ts, ns, slot0, kc, st);
  else
    dispatch_spectra<float>(p, x, ts, ns, slot0, kc, st);
}

// Per-call node statistics over the selected trials: psd = sum_k sum_l |X|^2
// (fp32 scaled units; the 1/L taper mean cancels in every ratio) and
// mag = max_k sqrt(sum_l |X|^2), the bound used by the exact-sign guard.
// 32 nodes x 8 trial lanes per block (small windows would otherwise leave one
// serial K-loop of dependent gathers per thread and under a wave of blocks).
constexpr int kNsNodes = 32, kNsLanes = 8;
__global__ void __launch_bounds__(kNsNodes * kNsLanes)
k_node_stats(const float2* __restrict__ X32, const int* __restrict__ slots, int K, int N, int nb, int L,
             int bin_lo, int nbb, float* __restrict__ psd, float* __restrict__ mag, float* __restrict__ nscale) {
  __shared__ double ss[kNsLanes][kNsNodes];
  __shared__ float sm[kNsLanes][kNsNodes];
  const int tx = threadIdx.x, g = threadIdx.y;
  const int n = blockIdx.x * kNsNodes + tx;
  const int bl = blockIdx.y;  // 0..nbb-1
  const int b = bin_lo + bl;
  double s = 0.0;
  float m = 0.f;
  if (n < N)
    for (int k = g; k < K; k += kNsLanes) {
      const int slot = slots[k];
      float e = 0.f;
      for (int l = 0; l < L; ++l) {
        const float2 v = X32[(((int64_t)slot * L + l) * nb + b) * N + n];
        e = fmaf(v.x, v.x, fmaf(v.y, v.y, e));
      }
      s += (double)e;
      m = fmaxf(m, sqrtf(e));
    }
  ss[g][tx] = s;
  sm[g][tx] = m;
  __syncthreads();
  if (g != 0 || n >= N) return;
#pragma unroll
  for (int q = 1; q < kNsLanes; ++q) {
    s += ss[q][tx];
    m = fmaxf(m, sm[q][tx]);
  }
  psd[(int64_t)bl * N + n] = (float)s;
  mag[(int64_t)bl * N + n] = m;
  int e = 0;
  if (m > 0.f) frexpf(m, &e);  // m = f * 2^e, f in [0.5, 1)  ->  m * 2^-e <= 1
  nscale[(int64_t)bl * N + n] = m > 0.f ? ldexpf(1.f, -e) : 1.f;
}

void run_node_stats(const Plan& p, const int* slots, int K, int bin_lo, int nbb,
                    cudaStream_t st) {
  dim3 grid((p.N + kNsNodes - 1) / kNsNodes, nbb);
  k_node_stats<<<grid, dim3(kNsNodes, kNsLanes), 0, st>>>(p.X32, slots, K, p.N, p.nb, p.L, bin_lo, nbb, p.psd,
                                                          p.mag, p.nscale);
}

// complex128 [n_slots][N][nbins] copy-out of the fp64 ring (taper 0), trial_spectra layout.
__global__ void k_get_spectra(const double2* __restrict__ X64, const int* __restrict__ slots,
                              int N, int nb, int L, int bin_lo, int nbins, double2* __restrict__ dst) {
  const int64_t idx = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  const int k = blockIdx.y;
  if (idx >= (int64_t)N * nbins) return;
  const int n = (int)(idx / nbins), bl = (int)(idx % nbins);
  dst[((int64_t)k * N + n) * nbins + bl] = X64[(((int64_t)slots[k] * L) * nb + bin_lo + bl) * N + n];
}

void run_get_spectra(const Plan& p, const int* slots, int ns, int bin_lo, int nbins, void* dst,
                     cudaStream_t st) {
  dim3 grid((unsigned)(((int64_t)p.N * nbins + 255) / 256), ns);
  k_get_spectra<<<grid, 256, 0, st>>>(p.X64, slots, p.N, p.nb, p.L, bin_lo, nbins, (double2*)dst);
}

}  // namespace cs

// ---------------------------------------------------------------------------
// Live pipe-peak probes for the roofline denominators that MEASURED_PEAKS.json
// does not carry (FP32 FMA-pipe lane ops/s and FP64 DFMA/s on this device).
// ---------------------------------------------------------------------------
namespace cs {
constexpr int kProbeIters = 4096;
__global__ void k_probe_fp32(float* out, float a, float b) {
  float x[8];
#pragma unroll
  for (int i = 0; i < 8; i++) x[i] = threadIdx.x + i;
  for (int it = 0; it < kProbeIters; it++) {
#pragma unroll
    for (int i = 0; i < 8; i++) x[i] = fmaf(x[i], a, b);
  }
  float s = 0;
#pragma unroll
  for (int i = 0; i < 8; i++) s += x[i];
  if (s == 12345.f) out[0] = s;
}
__global__ void k_probe_fp64(double* out, double a, double b) {
  double x[8];
#pragma unroll
  for (int i = 0; i < 8; i++) x[i] = threadIdx.x + i;
  for (int it = 0; it < kProbeIters; it++) {
#pragma unroll
    for (int i = 0; i < 8; i++) x[i] = fma(x[i], a, b);
  }
  double s = 0;
#pragma unroll
  for (int i = 0; i < 8; i++) s += x[i];
  if (s == 12345.0) out[0] = s;
}
}  // namespace cs

extern "C" int cs_probe_peaks(int device, double* fp32_lane_ops, double* fp64_fma) {
  int prev = 0;
  cudaGetDevice(&prev);
  cudaSetDevice(device);
  int nsm = 0;
  cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, device);
  void* buf = nullptr;
  cudaMalloc(&buf, 64);
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  const int grid = nsm * 8, blk = 256;
  float best32 = 1e30f, best64 = 1e30f;
  for (int rep = 0; rep < 4; ++rep) {
    float ms;
    cudaEventRecord(e0);
    cs::k_probe_fp32<<<grid, blk>>>((float*)buf, 1.0001f, 0.5f);
    cudaEventRecord(e1);
    cudaEventSynchronize(e1);
    cudaEventElapsedTime(&ms, e0, e1);
    if (rep) best32 = ms < best32 ? ms : best32;
    cudaEventRecord(e0);
    cs::k_probe_fp64<<<grid, blk>>>((double*)buf, 1.0001, 0.5);
    cudaEventRecord(e1);
    cudaEventSynchronize(e1);
    cudaEventElapsedTime(&ms, e0, e1);
    if (rep) best64 = ms < best64 ? ms : best64;
  }
  const double ops = (double)grid * blk * cs::kProbeIters * 8;
  *fp32_lane_ops = ops / (best32 * 1e-3);
  *fp64_fma = ops / (best64 * 1e-3);
  cudaEventDestroy(e0);
  cudaEventDestroy(e1);
  cudaFree(buf);
  cudaSetDevice(prev);
  return cudaGetLastError() == cudaSuccess ? CS_OK : CS_ECUDA;
}

// Externally computed spectra (complex128 [n][N][nbins], trial_spectra layout) into
// ring slots slot0.. (taper 0, plan-local bins [bin_lo, bin_lo + nbins)).
namespace cs {
__global__ void k_put_spectra(const double2* __restrict__ src, int n, int N, int nb, int L, int bin_lo,
                              int nbins, int slot0, int slot_cap, int taper, double w, float scale,
                              double2* __restrict__ X64, float2* __restrict__ X32, int real0, int real1,
                              int* __restrict__ complex_edge) {
  const int64_t idx = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  const int k = blockIdx.y;
  if (idx >= (int64_t)N * nbins) return;
  const int node = (int)(idx / nbins), bl = (int)(idx % nbins);
  double2 v = src[((int64_t)k * N + node) * nbins + bl];
  v.x *= w;
  v.y *= w;
  const int slot = (slot0 + k) % slot_cap;
  const int64_t o = (((int64_t)slot * L + taper) * nb + bin_lo + bl) * N + node;
  X64[o] = v;
  X32[o] = make_float2((float)(v.x * (double)scale), (float)(v.y * (double)scale));
  // a caller spectrum that is not exactly real at DC / Nyquist: the phase-lag kernel must fold
  // those bins like any other (spectral.py:216-241) instead of treating them as real
  if (v.y != 0.0 && (bin_lo + bl == real0 || bin_lo + bl == real1)) atomicOr(complex_edge, 1);
}
void run_put_spectra(const Plan& p, const void* src, int n, int bin_lo, int nbins, int slot0, int taper, double w,
                     cudaStream_t st) {
  dim3 grid((unsigned)(((int64_t)p.N * nbins + 255) / 256), n);
  k_put_spectra<<<grid, 256, 0, st>>>((const double2*)src, n, p.N, p.nb, p.L, bin_lo, nbins, slot0, p.slot_cap,
                                       taper, w, p.scale, p.X64, p.X32, p.dc_local, p.nyq_local, p.counters + 3);
}
}  // namespace cs

// ---------------------------------------------------------------------------
// K1, wide bands: fp64 real FFT (nfft a power of two).  One warp per signal:
// demean (shifted, exact for fp32 input) + taper, pack z_n = x_2n + i x_2n+1 in
// bit-reversed order into shared memory, radix-2 DIT FFT of size M = nfft/2, then
// the real-FFT split X_k = (Z_k + conj Z_{M-k})/2 - i W^k (Z_k - conj Z_{M-k})/2
// for the plan bins only.  ~5 M log2 M flops per signal instead of 4 T nb for the
// direct transform (cfg2: 102 bins -> ~10x fewer).
// ---------------------------------------------------------------------------
namespace cs {
constexpr int kFftWarps = 4;

template <typename Tin>
__global__ void __launch_bounds__(kFftWarps * 32)
k_spectra_fft(const Tin* __restrict__ x, int64_t trial_stride, int64_t node_stride, int N, int T_eff, int nfft,
              int log2M, int lo, int nb, int L, const double* __restrict__ taper, const double2* __restrict__ tw,
              const double2* __restrict__ post_tw, int slot0, int slot_cap, double2* __restrict__ X64,
              float2* __restrict__ X32, float scale, int dc_local, int nyq_local, int seg_stride, int ldn) {
  extern __shared__ double2 fft_smem[];
  const int M = nfft >> 1;
  double2* stw = fft_smem;                                  // [M/2] twiddles, shared by the CTA
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  for (int j = threadIdx.x; j < (M >> 1); j += blockDim.x) stw[j] = tw[j];
  __syncthreads();
  const int n = blockIdx.x * kFftWarps + warp;
  const int k = blockIdx.y;
  double2* z = fft_smem + (M >> 1) + warp * M;
  if (n >= N) return;  // warp-uniform
  const Tin* xr = x + (int64_t)k * trial_stride + (int64_t)n * node_stride;

  const int slot = (slot0 + k) % slot_cap;
  double mu = 0.0;
  const Tin* xr0 = xr;
  for (int l = 0; l < L; ++l) {  // all tapers of this signal in one warp: samples read once from HBM
    const double* w = taper ? taper + (int64_t)l * T_eff : nullptr;
    if (l == 0 || seg_stride) {  // welch: segment l has its own samples and mean
      xr = xr0 + (int64_t)l * seg_stride;
      // mean of the real samples, shifted by the first sample (fp64)
      const double c = (double)xr[0];
      double s = 0.0;
      for (int t = lane; t < T_eff; t += 32) s += (double)xr[t] - c;
#pragma unroll
      for (int o = 16; o > 0; o >>= 1) s += __shfl_xor_sync(0xffffffffu, s, o);
      mu = c + s / (double)T_eff;
    }
    // z_q = v_2q + i v_2q+1 (v = (x - mu) * taper, zero padded), stored at bitrev(q)
    for (int q = lane; q < M; q += 32) {
      const int t0 = 2 * q, t1 = 2 * q + 1;
      double a = 0.0, b = 0.0;
      if (t0 < T_eff) a = ((double)xr[t0] - mu) * (w ? w[t0] : 1.0);
      if (t1 < T_eff) b = ((double)xr[t1] - mu) * (w ? w[t1] : 1.0);
      z[__brev(q) >> (32 - log2M)] = make_double2(a, b);
    }
    __syncwarp();
    // iterative radix-2 DIT; twiddles from shared memory
    for (int sgn = 0; sgn < log2M; ++sgn) {
      const int half = 1 << sgn;
      const int tstride = M >> (sgn + 1);
#pragma unroll 4
      for (int bq = lane; bq < (M >> 1); bq += 32) {
        const int pos = bq & (half - 1);
        const int i0 = ((bq >> sgn) << (sgn + 1)) + pos;
        const int i1 = i0 + half;
        const double2 wv = stw[pos * tstride];
        const double2 u = z[i0], v0 = z[i1];
        const double2 v = make_double2(fma(v0.x, wv.x, -v0.y * wv.y), fma(v0.x, wv.y, v0.y * wv.x));
        z[i0] = make_double2(u.x + v.x, u.y + v.y);
        z[i1] = make_double2(u.x - v.x, u.y - v.y);
      }
      __syncwarp();
    }
    // real-FFT split for the plan bins
    for (int b = lane; b < nb; b += 32) {
      const int kk = lo + b;
      const double2 zk = z[kk == M ? 0 : kk];
      const double2 zm = z[(M - kk) & (M - 1)];  // Z_{M-k}, with Z_M = Z_0
      const double er = 0.5 * (zk.x + zm.x), ei = 0.5 * (zk.y - zm.y);   // E_k = (Z_k + conj Z_{M-k}) / 2
      const double dr = 0.5 * (zk.x - zm.x), di = 0.5 * (zk.y + zm.y);   // D = (Z_k - conj Z_{M-k}) / 2
      const double2 wk = post_tw[kk];                                    // e^{-2 pi i k / nfft}
      const double orr = di, oi = -dr;                                   // O_k = -i D
      double re = er + (wk.x * orr - wk.y * oi);
      double im = ei + (wk.x * oi + wk.y * orr);
      if (b == dc_local) re = im = 0.0;
      if (b == nyq_local) im = 0.0;
      const int64_t o = (((int64_t)slot * L + l) * (int64_t)nb + b) * ldn + n;  // ring rows of ldn nodes
      X64[o] = make_double2(re, im);
      X32[o] = make_float2((float)(re * (double)scale), (float)(im * (double)scale));
    }
    __syncwarp();
  }
}

// ---------------------------------------------------------------------------
// Four-step register FFT for M = nfft/2 = 32 A complex points (A = 8, 16), one
// warp per (node, trial), all tapers.  The real signal is packed as
// z_q = v_2q + i v_2q+1 (M-point complex FFT + real split).  With q = 32 a + b:
//   Z[k_a + A k_b] = sum_b W_32^{b k_b} W_M^{b k_a} sum_a z[32 a + b] W_A^{a k_a}
// step 1: lane b runs the A-point DFT over a in registers; step 2: twiddle
// W_M^{b k_a} (table [k_a][b], conflict-free); step 3: one shared-memory
// transpose gives lane (k_a, h) the b = h + R m, m < A (R = 32/A), an A-point
// register DFT over m, twiddle W_32^{h k'} and an R-point DFT across the R lanes
// by shuffles.  Shared memory is touched twice per element (no per-stage
// exchanges), butterflies stay in registers: FP64-pipe bound.
constexpr int kFft4Warps = 8;

__constant__ double2 c_w16[16] = {
    {1.0, 0.0},
    {0.92387953251128675613, -0.38268343236508977173},
    {0.70710678118654752440, -0.70710678118654752440},
    {0.38268343236508977173, -0.92387953251128675613},
    {0.0, -1.0},
    {-0.38268343236508977173, -0.92387953251128675613},
    {-0.70710678118654752440, -0.70710678118654752440},
    {-0.92387953251128675613, -0.38268343236508977173},
    {-1.0, 0.0},
    {-0.92387953251128675613, 0.38268343236508977173},
    {-0.70710678118654752440, 0.70710678118654752440},
    {-0.38268343236508977173, 0.92387953251128675613},
    {0.0, 1.0},
    {0.38268343236508977173, 0.92387953251128675613},
    {0.70710678118654752440, 0.70710678118654752440},
    {0.92387953251128675613, 0.38268343236508977173}};

__device__ __forceinline__ double2 cmul(double2 a, double2 w) {
  return make_double2(fma(a.x, w.x, -a.y * w.y), fma(a.x, w.y, a.y * w.x));
}
__host__ __device__ constexpr int brev_c(int i, int lg) {
  int r = 0;
  for (int k = 0; k < lg; ++k) r |= ((i >> k) & 1) << (lg - 1 - k);
  return r;
}
// in-register A-point DFT (natural order in and out), radix-2 DIT
template <int A>
__device__ __forceinline__ void dft_reg(double2 (&v)[A]) {
  constexpr int LG = A == 16 ? 4 : (A == 8 ? 3 : (A == 4 ? 2 : 1));
  double2 t[A];
#pragma unroll
  for (int i = 0; i < A; ++i) t[i] = v[brev_c(i, LG)];
#pragma unroll
  for (int s = 1; s < A; s <<= 1)
#pragma unroll
    for (int k = 0; k < A; k += 2 * s)
#pragma unroll
      for (int j = 0; j < s; ++j) {
        const int wi = j * (16 / (2 * s));  // W_{2s}^j = W_16^{16 j / 2s}
        double2 b = t[k + j + s];
        if (wi == 4) b = make_double2(b.y, -b.x);
        else if (wi != 0) b = cmul(b, c_w16[wi]);
        const double2 a = t[k + j];
        t[k + j] = make_double2(a.x + b.x, a.y + b.y);
        t[k + j + s] = make_double2(a.x - b.x, a.y - b.y);
      }
#pragma unroll
  for (int i = 0; i < A; ++i) v[i] = t[i];
}
__device__ __forceinline__ double2 shfl_xor2(double2 v, int m) {
  return make_double2(__shfl_xor_sync(0xffffffffu, v.x, m), __shfl_xor_sync(0xffffffffu, v.y, m));
}

template <typename Tin, int A>
__global__ void __launch_bounds__(kFft4Warps * 32, 2)
k_spectra_fft4(const Tin* __restrict__ x, int64_t trial_stride, int64_t node_stride, int N, int T_eff, int lo,
               int nb, int L, const double* __restrict__ taper, const double2* __restrict__ tw4,
               const double2* __restrict__ post_tw, const double2* __restrict__ wsum, int slot0, int slot_cap,
               double2* __restrict__ X64, float2* __restrict__ X32, float scale, int dc_local, int nyq_local,
               int n_trials, int vec16, int seg_stride, int ldn) {
  constexpr int R = 32 / A, M = 32 * A, S = 32 + R, PAD = 8 / R;
  constexpr int BUF = (A * S > M + PAD * R) ? A * S : M + PAD * R;
  extern __shared__ double2 f4_smem[];
  double2* tabM = f4_smem;        // [A][32]  W_M^{b k_a}
  double2* w32 = tabM + A * 32;   // [32]     W_32^j
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  for (int j = threadIdx.x; j < A * 32 + 32; j += blockDim.x) f4_smem[j] = tw4[j];
  __syncthreads();
  double2* buf = w32 + 32 + kFft4Warps * BUF * 0 + warp * BUF;
  // per-warp sample staging (cp.async): the next signal streams in while this one transforms
  Tin* stage = (Tin*)(w32 + 32 + kFft4Warps * BUF) + warp * (32 * A * 2);
  const int ka2 = lane / R, h = lane % R;
  const int j_out = R == 4 ? (((h & 1) << 1) | (h >> 1)) : h;  // R-point DIF output order
  // unit = (node, trial) with all tapers; welch: (node, trial, segment), one segment each
  const int n_units_l = seg_stride ? L : 1;
  const int64_t n_sig = (int64_t)N * n_trials * n_units_l;
  const int64_t gw = (int64_t)blockIdx.x * kFft4Warps + warp, nw = (int64_t)gridDim.x * kFft4Warps;
  constexpr int V = 16 / sizeof(Tin);  // elements per 16-byte copy
  auto prefetch = [&](int64_t sig) {
    if (sig < n_sig) {
      const int n = (int)(sig % N), k = (int)((sig / N) % n_trials), ls = (int)(sig / N / n_trials);
      const Tin* xr = x + (int64_t)k * trial_stride + (int64_t)n * node_stride + (int64_t)ls * seg_stride;
      if (vec16) {
        for (int e = lane * V; e < T_eff; e += 32 * V) cp_async16(stage + e, xr + e, 16);
      } else {
        for (int e = lane; e < T_eff; e += 32) cp_async4_any(stage + e, xr + e);
      }
    }
    cp_async_commit();
  };
  prefetch(gw);
  for (int64_t sig = gw; sig < n_sig; sig += nw) {
    const int n = (int)(sig % N), k = (int)((sig / N) % n_trials);
    const int l_begin = seg_stride ? (int)(sig / N / n_trials) : 0, l_end = seg_stride ? l_begin + 1 : L;
    const int slot = (slot0 + k) % slot_cap;
    cp_async_wait0();
    __syncwarp();
    // d_t = x_t - c (c = first sample, exact for fp32 input); the mean is removed after
    // the transform by linearity: X_b = FFT(d w)_b - mean(d) W_b, W_b = sum_t w_t e_bt
    // (plan table wsum)
    const double c = (double)stage[0];
    double mean_d = 0.0;
    for (int l = l_begin; l < l_end; ++l) {
      const double* w = taper ? taper + (int64_t)l * T_eff : nullptr;
      double2 v[A];
      double sum = 0.0;
#pragma unroll
      for (int a = 0; a < A; ++a) {
        const int t0 = 2 * (32 * a + lane);
        const double d0 = t0 < T_eff ? (double)stage[t0] - c : 0.0;
        const double d1 = t0 + 1 < T_eff ? (double)stage[t0 + 1] - c : 0.0;
        sum += d0 + d1;
        v[a] = w ? make_double2(d0 * (t0 < T_eff ? w[t0] : 0.0), d1 * (t0 + 1 < T_eff ? w[t0 + 1] : 0.0))
                 : make_double2(d0, d1);
      }
      if (l == l_end - 1) {  // samples are in registers: stream the next signal in
        __syncwarp();
        prefetch(sig + nw);
      }
      if (l == l_begin) {
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) sum += __shfl_xor_sync(0xffffffffu, sum, o);
        mean_d = sum / (double)T_eff;
      }
      dft_reg<A>(v);                       // over a -> k_a
#pragma unroll
      for (int ka = 1; ka < A; ++ka) v[ka] = cmul(v[ka], tabM[ka * 32 + lane]);
#pragma unroll
      for (int ka = 0; ka < A; ++ka) buf[ka * S + lane] = v[ka];
      __syncwarp();
#pragma unroll
      for (int m = 0; m < A; ++m) v[m] = buf[ka2 * S + h + R * m];
      __syncwarp();
      dft_reg<A>(v);                       // over m -> k'
#pragma unroll
      for (int kp = 1; kp < A; ++kp) v[kp] = cmul(v[kp], w32[(h * kp) & 31]);
      if (R == 2) {
#pragma unroll
        for (int kp = 0; kp < A; ++kp) {
          const double2 o = shfl_xor2(v[kp], 1);
          v[kp] = h == 0 ? make_double2(v[kp].x + o.x, v[kp].y + o.y) : make_double2(o.x - v[kp].x, o.y - v[kp].y);
        }
      } else {  // R == 4: two radix-2 DIF stages across lanes h ^ 2, h ^ 1
#pragma unroll
        for (int kp = 0; kp < A; ++kp) {
          const double2 o = shfl_xor2(v[kp], 2);
          if (h < 2) {
            v[kp] = make_double2(v[kp].x + o.x, v[kp].y + o.y);
          } else {
            const double2 d = make_double2(o.x - v[kp].x, o.y - v[kp].y);
            v[kp] = h == 3 ? make_double2(d.y, -d.x) : d;
          }
        }
#pragma unroll
        for (int kp = 0; kp < A; ++kp) {
          const double2 o = shfl_xor2(v[kp], 1);
          v[kp] = (h & 1) == 0 ? make_double2(v[kp].x + o.x, v[kp].y + o.y)
                               : make_double2(o.x - v[kp].x, o.y - v[kp].y);
        }
      }
      // Z[k], k = k_a + A k' + A^2 j, stored at k + PAD j (conflict-free)
#pragma unroll
      for (int kp = 0; kp < A; ++kp) buf[ka2 + A * kp + (A * A + PAD) * j_out] = v[kp];
      __syncwarp();
      for (int b = lane; b < nb; b += 32) {
        const int kk = lo + b;
        const int k1 = kk == M ? 0 : kk, k2 = (M - kk) & (M - 1);
        const double2 zk = buf[k1 + PAD * (k1 / (A * A))];
        const double2 zm = buf[k2 + PAD * (k2 / (A * A))];
        const double er = 0.5 * (zk.x + zm.x), ei = 0.5 * (zk.y - zm.y);
        const double dr = 0.5 * (zk.x - zm.x), di = 0.5 * (zk.y + zm.y);
        const double2 wk = post_tw[kk];
        const double orr = di, oi = -dr;
        const double2 ws = wsum[l * nb + b];
        double re = er + (wk.x * orr - wk.y * oi) - mean_d * ws.x;
        double im = ei + (wk.x * oi + wk.y * orr) - mean_d * ws.y;
        if (b == dc_local) re = im = 0.0;
        if (b == nyq_local) im = 0.0;
        const int64_t o = (((int64_t)slot * L + l) * (int64_t)nb + b) * ldn + n;  // ring rows of ldn nodes
        X64[o] = make_double2(re, im);
        X32[o] = make_float2((float)(re * (double)scale), (float)(im * (double)scale));
      }
      __syncwarp();
    }
  }
  cp_async_wait0();
}

template <typename Tin, int A>
void launch_fft4(const Plan& p, const void* x, int64_t ts, int64_t ns, int slot0, int kc, cudaStream_t st) {
  constexpr int R = 32 / A, M = 32 * A, S = 32 + R, PAD = 8 / R;
  constexpr int BUF = (A * S > M + PAD * R) ? A * S : M + PAD * R;
  const size_t smem = (size_t)(A * 32 + 32 + kFft4Warps * BUF) * sizeof(double2) +
                      (size_t)kFft4Warps * 64 * A * sizeof(Tin);
  CS_SMEM_ONCE((k_spectra_fft4<Tin, A>), smem);
  static std::atomic<int> occ{0};  // same on every B200
  int ctas_per_sm = occ.load(std::memory_order_relaxed);
  if (!ctas_per_sm) {
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&ctas_per_sm, k_spectra_fft4<Tin, A>, kFft4Warps * 32, smem);
    if (ctas_per_sm < 1) ctas_per_sm = 1;
    occ.store(ctas_per_sm);
  }
  int nsm = 148;
  cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, p.device);
  const int64_t sigs = (int64_t)p.N * kc * (p.seg_stride ? p.L : 1);
  int64_t grid = (int64_t)nsm * ctas_per_sm;
  const int64_t need = (sigs + kFft4Warps - 1) / kFft4Warps;
  if (grid > need) grid = need;
  // 16-byte staging copies when every row start and the row length allow it
  const int vec16 = ((uintptr_t)x % 16 == 0) && ((ts * (int64_t)sizeof(Tin)) % 16 == 0) &&
                    ((ns * (int64_t)sizeof(Tin)) % 16 == 0) && ((p.T_eff * (int)sizeof(Tin)) % 16 == 0) &&
                    ((p.seg_stride * (int64_t)sizeof(Tin)) % 16 == 0);
  k_spectra_fft4<Tin, A><<<(unsigned)grid, kFft4Warps * 32, smem, st>>>((const Tin*)x, ts, ns, p.N, p.T_eff,
      p.lo, p.nb, p.L, p.taper, p.fft4_tw, p.post_tw, p.wsum, slot0, p.slot_cap, p.X64, p.X32, p.scale,
      p.dc_local, p.nyq_local, kc, vec16, p.seg_stride, p.ldn);
}

bool run_spectra_fft(const Plan& p, const void* x, int dtype, int64_t ts, int64_t ns, int slot0, int kc,
                     cudaStream_t st) {
  const int M = p.nfft / 2;
  if (p.fft4_tw && (M == 256 || M == 512)) {  // four-step register FFT
    if (dtype == CS_F64) {
      if (M == 256) launch_fft4<double, 8>(p, x, ts, ns, slot0, kc, st);
      else launch_fft4<double, 16>(p, x, ts, ns, slot0, kc, st);
    } else {
      if (M == 256) launch_fft4<float, 8>(p, x, ts, ns, slot0, kc, st);
      else launch_fft4<float, 16>(p, x, ts, ns, slot0, kc, st);
    }
    return true;
  }
  int log2M = 0;
  while ((1 << log2M) < M) ++log2M;
  const size_t smem = (size_t)(kFftWarps * M + M / 2) * sizeof(double2);
  dim3 grid((p.N + kFftWarps - 1) / kFftWarps, kc);
  if (dtype == CS_F64) {
    CS_SMEM_ONCE(k_spectra_fft<double>, 200 * 1024);
    k_spectra_fft<double><<<grid, kFftWarps * 32, smem, st>>>((const double*)x, ts, ns, p.N, p.T_eff, p.nfft, log2M,
        p.lo, p.nb, p.L, p.taper, p.fft_tw, p.post_tw, slot0, p.slot_cap, p.X64, p.X32, p.scale, p.dc_local, p.nyq_local,
        p.seg_stride, p.ldn);
  } else {
    CS_SMEM_ONCE(k_spectra_fft<float>, 200 * 1024);
    k_spectra_fft<float><<<grid, kFftWarps * 32, smem, st>>>((const float*)x, ts, ns, p.N, p.T_eff, p.nfft, log2M,
        p.lo, p.nb, p.L, p.taper, p.fft_tw, p.post_tw, slot0, p.slot_cap, p.X64, p.X32, p.scale, p.dc_local, p.nyq_local,
        p.seg_stride, p.ldn);
  }
  return true;
}
}  // namespace cs
