// Shared definitions for the csconn CUDA sources (sm_100a only).
#pragma once
#include <cuda_runtime.h>
#include <stdint.h>

#include <atomic>
#include <vector>

#include "../../include/csconn.h"

#ifndef __CUDA_ARCH__
#define CS_HOST_ONLY 1
#endif

// Opt a kernel into more than 48 KB of dynamic shared memory, once per device (the
// attribute belongs to the kernel on the current device; plans may live on several).
#define CS_SMEM_ONCE(fn, bytes)                                                                  \
  do {                                                                                           \
    static std::atomic<unsigned long long> done_{0};                                              \
    int dev_ = 0;                                                                                \
    cudaGetDevice(&dev_);                                                                        \
    const unsigned long long bit_ = 1ull << (dev_ & 63);                                         \
    if (!(done_.load(std::memory_order_relaxed) & bit_)) {                                       \
      cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)(bytes));        \
      done_.fetch_or(bit_);                                                                      \
    }                                                                                            \
  } while (0)

namespace cs {


// fp16 split operand planes per (bin, pass) (k_tc_prep): re_h, re_l, im_h, im_l, -im_h, -im_l
// (the negated Im planes are the CTA-pair kernel's second B half, pairs_tc.cu)
constexpr int kTcPlanes = 6;

constexpr int kTile = 64;        // node tile edge of the upper-triangular pair tiling
constexpr int kThreads = 256;    // pair-kernel CTA size (16 x 16 threads, 4 x 4 pairs each)
// The phase-lag kernel's register tile (pairs_lag1.cu): every compute thread owns
// kGuardTR x kGuardTC pairs (i = row0 + ty + kGuardRowStep r, j = col0 + tx + kGuardColStep c).
// Exact-sign guard overflow records (guard_push; window.cu): kGuardRecI4 int4 each, a header
// (row of the warp's lane 0, column base, bin, lanes per row) then kGuardNP mask words; bit
// lane of word (r kGuardTC + c) -> pair (h.x + lane / h.w + kGuardRowStep r,
// h.y + lane % h.w + kGuardColStep c)
constexpr int kGuardTR = 4, kGuardTC = 2, kGuardNP = kGuardTR * kGuardTC;
constexpr int kGuardRowStep = 64 / kGuardTR, kGuardColStep = 64 / kGuardTC;
constexpr int kGuardWarps = kGuardRowStep * kGuardColStep / 32;
constexpr int kGuardRecI4 = 1 + kGuardNP / 4;

struct Plan {
  int device = 0;
  int N = 0, T = 0, nfft = 0, lo = 0, hi = 0, nb = 0, L = 1, T_eff = 0;
  int slot_cap = 0;
  float scale = 1.f;             // power of two applied to the fp32 spectra
  int dc_local = -1, nyq_local = -1;  // plan-local indices of exactly-real bins
  double2* tww = nullptr;        // [L][nb][T_eff]   taper x twiddle
  double2* wsum = nullptr;       // [L][nb]          sum_t tww (mean correction)
  double* taper = nullptr;       // [L][T_eff] tapers (null: rectangular)        -- FFT path
  double2* fft_tw = nullptr;     // [nfft/4] e^{-2 pi i j / (nfft/2)}             -- FFT path
  double2* post_tw = nullptr;    // [nfft/2 + 1] e^{-2 pi i k / nfft}            -- FFT path
  double2* fft4_tw = nullptr;    // [A][32] W_M^{b k_a}, then [32] W_32^j       -- four-step FFT (M = 32 A)
  bool use_fft = false;          // power-of-two nfft and a band wide enough to prefer the FFT
  int seg_stride = 0;            // welch: sample offset between segments (= nfft), else 0
  double* dft_tf = nullptr;      // [L][ceil(T_eff/4)][NT][32] fp64 DFT B fragments (tensor-core DFT), or null
  int ldn = 0;                   // ring row stride in nodes (N; a node-range view of K1 keeps the full plan's)
  double2* X64 = nullptr;        // [slot][L][nb][N]  fp64 spectra (fp64 guard / fallback)
  float2* X32 = nullptr;         // [slot][L][nb][N]  fp32 scaled spectra
  float* psd = nullptr;          // [nb][N] per-call node statistics
  float* mag = nullptr;          // [nb][N] max_k sqrt(sum_l |X|^2)
  float* nscale = nullptr;       // [nb][N] 2^-ceil(log2 mag): per-node-bin fp16 operand scale
  void* tc_ops = nullptr;        // tensor-core operand planes (grown on demand)
  bool tc_neg_planes = false;    // ... the last prep also wrote the -Im planes (CTA-pair kernel)
  size_t tc_bytes = 0;
  void* lag_ops = nullptr;       // packed trial-pair operands of the phase-lag kernel
  size_t lag_bytes = 0;
  struct TileList {              // tensor-core tile order (int2 list) of one row range
    uint64_t key = 0;
    void* ptr = nullptr;
    int64_t n = 0;
  };
  static constexpr int kTileCache = 16;  // row-chunked callers cycle through a few ranges
  TileList tc_tiles[kTileCache];
  int tc_tiles_next = 0;
  int4* flags = nullptr;         // fp64-fallback work list (i, j, local bin, -)
  int* counters = nullptr;       // [0] flagged entries, [1] list overflowed, [2] overflow records,
                                 // [3] caller spectra put a non-real value into an exactly-real bin
  int4* recs = nullptr;          // guard overflow records (3 int4 each), grown on demand
  size_t rec_cap = 0;            // records
  int flag_cap = 0;
  // node statistics + operand packing of the last cs_pair_metrics call, reusable by a
  // following call over another row range (CS_PM_REUSE_PREP)
  struct PrepKey {
    const int* slots = nullptr;
    int K = 0, bin_lo = 0, nbb = 0;
    unsigned mask = 0;
    bool operator==(const PrepKey& o) const {
      return slots == o.slots && K == o.K && bin_lo == o.bin_lo && nbb == o.nbb && mask == o.mask;
    }
  };
  PrepKey prep_key;
  bool prep_valid = false;
  bool reuse_prep = false;       // set for the duration of one call
  bool imag_handoff = false;     // the last call handed IMAGCOHY from K2 to K3
  bool spectra_put = false;      // caller spectra entered the ring (cs_put_spectra): counters[3] says
                                 // whether one was complex at DC / Nyquist (then those bins are not real)
  // multi-GPU (shard.cu): peers' rings attached by cs_ring_attach[_ptrs]
  int n_ranks = 0, rank = 0, node_block = 0;  // node n's fp64 spectra live on rank n / node_block
  double2** peer_x64 = nullptr;  // device [n_ranks] fp64 ring of every rank (own included)
  std::vector<float2*> peers32;  // fp32 rings of the peers (push targets; own = null)
  std::vector<void*> ipc_opened; // IPC mappings to close on destroy
  int64_t fft_calls = 0;
  int64_t launches = 0;          // kernels launched by this plan (bench evidence)
  bool profiling = false;        // record CUDA events around every kernel phase
  void* prof = nullptr;          // host-side event records (api.cu)
};

// packed fp32x2 helpers (Blackwell f32x2 ALU instructions)
typedef unsigned long long f2;
__device__ __forceinline__ f2 pk(float lo, float hi) {
  f2 r;
  asm("mov.b64 %0, {%1, %2};" : "=l"(r) : "f"(lo), "f"(hi));
  return r;
}
__device__ __forceinline__ float lo_of(f2 v) {
  float a, b;
  asm("mov.b64 {%0, %1}, %2;" : "=f"(a), "=f"(b) : "l"(v));
  return a;
}
__device__ __forceinline__ float hi_of(f2 v) {
  float a, b;
  asm("mov.b64 {%0, %1}, %2;" : "=f"(a), "=f"(b) : "l"(v));
  return b;
}
__device__ __forceinline__ f2 fmul2(f2 a, f2 b) {
  f2 d;
  asm("mul.rn.f32x2 %0, %1, %2;" : "=l"(d) : "l"(a), "l"(b));
  return d;
}
__device__ __forceinline__ f2 ffma2(f2 a, f2 b, f2 c) {
  f2 d;
  asm("fma.rn.f32x2 %0, %1, %2, %3;" : "=l"(d) : "l"(a), "l"(b), "l"(c));
  return d;
}
__device__ __forceinline__ f2 fadd2(f2 a, f2 b) {
  f2 d;
  asm("add.rn.f32x2 %0, %1, %2;" : "=l"(d) : "l"(a), "l"(b));
  return d;
}

// Upper-triangle pair index of (i < j) over n nodes (spectral.py:119-122).
__host__ __device__ __forceinline__ int64_t pair_of(int64_t i, int64_t j, int64_t n) {
  return i * (n - 1) - i * (i - 1) / 2 + (j - i - 1);
}

// Decode the t-th tile (I <= J) of the row-tile range starting at row_begin.
// Upper-triangle tile t (row-major from row_begin, row r holding nt - r tiles) ->
// (I, J).  The first m rows hold S(m) = m (nt - row_begin) - m (m - 1) / 2 tiles;
// m comes from the quadratic's root, then at most a step of integer fix-up.
__device__ __forceinline__ void decode_tile(int64_t t, int nt, int row_begin, int& I, int& J) {
  const int64_t w = nt - row_begin;
  const double b = (double)w + 0.5;
  int64_t m = (int64_t)(b - sqrt(fmax(b * b - 2.0 * (double)t, 0.0)));
  if (m < 0) m = 0;
  while (m > 0 && m * w - m * (m - 1) / 2 > t) --m;
  while ((m + 1) * w - (m + 1) * m / 2 <= t) ++m;
  I = row_begin + (int)m;
  J = I + (int)(t - (m * w - m * (m - 1) / 2));
}

// Profiling phase (CUDA events on the launching stream around one kernel);
// implemented in api.cu, a no-op unless cs_plan_set_profiling() is on.
struct PhaseMark {
  void* rec = nullptr;
  PhaseMark(Plan& p, const char* name, cudaStream_t st);
  ~PhaseMark();
};

}  // namespace cs

void cs_set_error(const char* fmt, ...);
