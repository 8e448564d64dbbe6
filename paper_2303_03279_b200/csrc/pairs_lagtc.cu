// K3 on the tensor cores (single taper): the per-trial products
// t_k = Im(X_ik conj X_jk) of a 128 x 64 pair tile come out of tcgen05.mma, and the
// nonlinear per-trial statistics (sign counts, sum |t|, the exact-sign guard min |t|)
// run on the FP32/ALU pipes straight from TMEM.
//
// Reference: spectral.py:216-241 (_fold_csd: Im flush, sign(Im), |Im|, Im sums),
// metrics.py:49-86 (imagcohy / pli / uspli / wpli / dswpli), metrics.py:115-134 and
// core.py:208-215 (band mean).
//
// Why: on the CUDA cores t costs FMUL2 + FFMA2 per two updates and the loop is bound
// by the FMA pipe at 4 lane-ops per update (pairs_lag1.cu).  Here one
// 128 x 128 x 16 f16 MMA yields t for 128 x 64 pairs and two trials, leaving ~2.3
// issue slots per update (FADD |t|, a PRMT sign byte pair, FMNMX3) for the statistics.
//
// Operands (k_lagtc_prep), per node-bin power of two so |x| <= 1, split x = h + l in
// fp16 (from the fp64 ring), 8 halves = 16 B per node and trial:
//   A side (rows i):  [Im_h, Im_l, Im_h, Im_l, -Re_h, -Re_l, -Re_h, -Re_l]
//   B side (cols j):  [Re_h, Re_h, Re_l, Re_l,  Im_h,  Im_h,  Im_l,  Im_l]
// so A . B = (Im_i)(Re_j) - (Re_i)(Im_j) with all four hi/lo cross products.
// A stage holds two trials k0, k1 (no-swizzle K-major, 8-row x 16 B core matrices):
//   A  [k0: 128 rows][k1: 128 rows]          K = 16 (k0 | k1), LBO 2048, SBO 128
//   B  [k0: 64 rows][zeros 1 KB][k1: 64 rows]
// Read with LBO 1024 and N = 128 the B stage is block diagonal: column (j, k0) sees
// (B_k0, 0), column (64 + j, k1) sees (0, B_k1), so one MMA gives both trials' t in
// 128 TMEM columns.  Read with LBO 2048 and N = 64 it is [B_k0 | B_k1] per column j,
// and an accumulating MMA sums t over trials (sum Im CSD for IMAGCOHY and WPLI).
//
// Error: the split keeps 22 bits (|x - h - l| <= 2^-22 M), so |t_tc - t| <=
// 2 sqrt(2) 2^-22 M_i M_j + accumulation (measured <= 3.2 2^-24, tools/ubench/tc_lag_probe.cu);
// the guard factor is g = 1.5 (11.4 + 8) 2^-24.  Entries with min_k |t_k| <= g M_i M_j
// go to the fp64 fallback (k_lag_fallback), as in the CUDA-core kernel.
//
// CTA: 16 warps, persistent over (tile, bin chunk) units.  Warp 0 lane 0 also issues the
// TMA loads (4-stage ring, two trials per stage) and the MMAs (3 TMEM buffers of 128
// columns for t, 2 x 64 for the running sum), one step ahead of the consumers.  Warp w
// reads TMEM lane quadrant w % 4 and columns 16 (w / 4) + [0, 16): 16 pairs per thread.
#include <cuda.h>
#include <cuda_fp16.h>

#include <climits>
#include <cstdlib>
#include <vector>

#include "common.cuh"
#include "ptx.cuh"

namespace cs {

constexpr int kLtI = 128, kLtJ = 64;
constexpr int kLtStages = 8;
constexpr int kLtStageBytes = 7168;            // A 4096 + B 3072
constexpr int kLtConsumers = 16;               // consumer warps (4 per TMEM lane quadrant)
constexpr int kLtThreads = (4 + kLtConsumers) * 32;
constexpr int kLtStgStride = 17;               // per-warp transpose staging row stride (floats)
constexpr int kLtBandBytes = 4 * kLtI * kLtJ * 4;   // PLI, USPLI, WPLI, DSWPLI (IMAGCOHY band in TMEM)
constexpr int kLtStgBytes = kLtConsumers * 32 * kLtStgStride * 4;
constexpr int kLtTmemSum = 384;                // TMEM: t buffers [0,384), running sum [384,448),
constexpr int kLtTmemBand = 448;               //       IMAGCOHY band sums [448,512)
constexpr float kLtPhantom = 0.03125f;         // 2^-5: odd-K phantom trial, t = 2^-10 exactly
constexpr unsigned kLtSign = 1, kLtSum = 2, kLtAbs = 4, kLtAll = 7;

struct LtArgs {
  int N, K, K2, Npad, nbb, bin_lo;
  int i_lo, i_hi;
  int n_units, nbc, bpc;
  const int2* tiles;
  const uint4* GA;          // [nbb][K2][Npad] A-side operands (8 halves)
  const uint4* GB;          // [nbb][K2][Npad] B-side operands
  const float2* nf;         // [nbb][N] (M_hat = scaled max |X|, 0 for dead / exactly-real; rsqrt(psd s^2))
  int64_t pair_base, pair_stride;
  float* bins[5];           // IMAGCOHY, PLI, USPLI, WPLI, DSWPLI
  float* band[5];
  float g;
  int4* flags;
  int* counters;
  int flag_cap;
};

__device__ __forceinline__ uint64_t lt_desc(uint32_t addr, uint32_t lbo) {
  uint64_t d = 0;
  d |= (uint64_t)((addr >> 4) & 0x3FFF);
  d |= (uint64_t)((lbo >> 4) & 0x3FFF) << 16;   // K-direction core-matrix stride
  d |= (uint64_t)(128 >> 4) << 32;               // 8-row group stride
  d |= (uint64_t)1 << 46;                        // version (Blackwell), no swizzle
  return d;
}
__device__ __forceinline__ void bulk_g2s_elect(uint32_t dst, const void* src, uint32_t bytes, uint32_t bar) {
  asm volatile(
      "{\n\t.reg .pred e;\n\telect.sync _|e, 0xffffffff;\n\t"
      "@e cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];\n\t}"
      ::"r"(dst), "l"(src), "r"(bytes), "r"(bar)
      : "memory");
}
__device__ __forceinline__ void expect_tx_elect(uint32_t bar, uint32_t bytes) {
  asm volatile(
      "{\n\t.reg .pred e;\n\telect.sync _|e, 0xffffffff;\n\t"
      "@e mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;\n\t}"
      ::"r"(bar), "r"(bytes)
      : "memory");
}
__host__ __device__ constexpr uint32_t lt_idesc(int n) {
  return (1u << 4) | ((uint32_t)(n >> 3) << 17) | ((uint32_t)(kLtI >> 4) << 24);
}

__device__ __forceinline__ void lt_ld8x2(uint32_t ta, float* v, uint32_t tb, float* w) {
  uint32_t r[8], s[8];
  asm volatile("tcgen05.ld.sync.aligned.32x32b.x8.b32 {%0,%1,%2,%3,%4,%5,%6,%7}, [%8];"
               : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]), "=r"(r[7])
               : "r"(ta));
  asm volatile("tcgen05.ld.sync.aligned.32x32b.x8.b32 {%0,%1,%2,%3,%4,%5,%6,%7}, [%8];"
               : "=r"(s[0]), "=r"(s[1]), "=r"(s[2]), "=r"(s[3]), "=r"(s[4]), "=r"(s[5]), "=r"(s[6]), "=r"(s[7])
               : "r"(tb));
  asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
#pragma unroll
  for (int q = 0; q < 8; ++q) {
    v[q] = __uint_as_float(r[q]);
    w[q] = __uint_as_float(s[q]);
  }
}
__device__ __forceinline__ void lt_ld8(uint32_t ta, float* v) {
  uint32_t r[8];
  asm volatile("tcgen05.ld.sync.aligned.32x32b.x8.b32 {%0,%1,%2,%3,%4,%5,%6,%7}, [%8];"
               : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]), "=r"(r[7])
               : "r"(ta));
  asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
#pragma unroll
  for (int q = 0; q < 8; ++q) v[q] = __uint_as_float(r[q]);
}
__device__ __forceinline__ void lt_st8(uint32_t taddr, const float* v) {
  asm volatile("tcgen05.st.sync.aligned.32x32b.x8.b32 [%0], {%1,%2,%3,%4,%5,%6,%7,%8};"
               ::"r"(taddr), "r"(__float_as_uint(v[0])), "r"(__float_as_uint(v[1])), "r"(__float_as_uint(v[2])),
               "r"(__float_as_uint(v[3])), "r"(__float_as_uint(v[4])), "r"(__float_as_uint(v[5])),
               "r"(__float_as_uint(v[6])), "r"(__float_as_uint(v[7])));
}
__device__ __forceinline__ void lt_ld16(uint32_t ta, float* v) {
  uint32_t r[16];
  asm volatile(
      "tcgen05.ld.sync.aligned.32x32b.x16.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15}, [%16];"
      : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]), "=r"(r[7]),
        "=r"(r[8]), "=r"(r[9]), "=r"(r[10]), "=r"(r[11]), "=r"(r[12]), "=r"(r[13]), "=r"(r[14]), "=r"(r[15])
      : "r"(ta));
  asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
#pragma unroll
  for (int q = 0; q < 16; ++q) v[q] = __uint_as_float(r[q]);
}


// Consumer wait: try_wait with a suspend-time hint, so waiting warps sleep instead of
// taking issue slots from warp 0 (which also issues the TMA loads and the MMAs).
__device__ __forceinline__ void mbar_wait_sleep(uint64_t* bar, uint32_t parity) {
  uint32_t done;
  const long long t0 = clock64();
  while (true) {
    asm volatile(
        "{\n\t.reg .pred P1;\n\t"
        "mbarrier.try_wait.parity.shared::cta.b64 P1, [%1], %2, %3;\n\t"
        "selp.u32 %0, 1, 0, P1;\n\t}"
        : "=r"(done)
        : "r"(smem_u32(bar)), "r"(parity), "r"(1000000u)
        : "memory");
    if (done) return;
    if (clock64() - t0 > 20000000000ll) __trap();
  }
}

// Step iterator over this CTA's (unit, bin, trial pair) sequence.
struct LtIt {
  int u, bl, bl1, sp, bseq;
  int2 tij;  // tile of the current unit (loaded once per unit)
  __device__ void start(const LtArgs& a) {
    u = blockIdx.x;
    bseq = 0;
    sp = 0;
    set_unit(a);
  }
  __device__ void set_unit(const LtArgs& a) {
    if (u < a.n_units) {
      const int tu = u / a.nbc;
      bl = (u - tu * a.nbc) * a.bpc;
      bl1 = min(a.nbb, bl + a.bpc);
      tij = a.tiles[tu];
    }
  }
  __device__ bool done(const LtArgs& a) const { return u >= a.n_units; }
  // advance one step; returns true when the step just left was the last of its bin
  __device__ void next(const LtArgs& a) {
    if (++sp < a.K2 / 2) return;
    sp = 0;
    ++bseq;
    if (++bl < bl1) return;
    u += gridDim.x;
    set_unit(a);
  }
};

// Warp roles (20 warps, register budgets rebalanced with setmaxnreg):
//   warp 0        TMA producer: 1D bulk copies of each step's two trials into the ring
//   warp 1        MMA issuer: per step one N = 128 MMA (t of both trials) into a TMEM
//                 buffer and, for sum t, one accumulating N = 64 MMA into the running sum
//   warp 2        TMEM allocator; warps 0-3 drop to 24 registers
//   warps 4-19    consumers, 112 registers (the CTA keeps its launch pool of 640 x 96 =
//                 128 x 24 + 512 x 112): TMEM lane quadrant warp % 4, 16 columns each
template <unsigned STATS>
__global__ void __launch_bounds__(kLtThreads, 1)
k_pairs_lagtc(const LtArgs a) {
  extern __shared__ __align__(1024) unsigned char lt_smem[];
  unsigned char* stages = lt_smem;
  float* band_s = (float*)(lt_smem + kLtStages * kLtStageBytes);            // [4][128][64], column ^ 16 (row & 1)
  float* stg = (float*)((unsigned char*)band_s + kLtBandBytes);             // [16][32][17]
  int* rel_s = (int*)((unsigned char*)stg + kLtStgBytes);                   // [128] row offsets rel. to quadrant row 0
  long long* base_s = (long long*)(rel_s + kLtI);                          // [4] pair offset of quadrant row 0
  float2* colnf = (float2*)(base_s + 4);                                   // [2][64] column node factors
  uint64_t* full = (uint64_t*)(colnf + 2 * kLtJ);
  uint64_t* empty = full + kLtStages;
  uint64_t* tfull = empty + kLtStages;    // [3]
  uint64_t* tempty = tfull + 3;           // [3]
  uint64_t* sempty = tempty + 3;          // running-sum region released by the epilogue
  uint32_t* tmem_slot = (uint32_t*)(sempty + 1);

  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int n_sp = a.K2 / 2;

  // zero blocks between the two B trials of every stage (never written by TMA)
  for (int e = threadIdx.x; e < kLtStages * 64; e += kLtThreads) {
    const int s = e >> 6, o = e & 63;
    ((uint4*)(stages + s * kLtStageBytes + 4096 + 1024))[o] = make_uint4(0, 0, 0, 0);
  }
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
  if (threadIdx.x == 0) {
    for (int s = 0; s < kLtStages; ++s) {
      mbar_init(&full[s], 1);
      mbar_init(&empty[s], 1);
    }
    for (int b = 0; b < 3; ++b) {
      mbar_init(&tfull[b], 1);
      mbar_init(&tempty[b], kLtConsumers);
    }
    mbar_init(sempty, kLtConsumers);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  if (warp == 2) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 512;" ::"r"(smem_u32(tmem_slot)));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = *tmem_slot;
  const uint32_t st_base = smem_u32(stages);

  if (warp < 4) {
    asm volatile("setmaxnreg.dec.sync.aligned.u32 24;");
    if (warp == 0) {
      // ---------------------------------------------------------- TMA producer
      LtIt ti;
      ti.start(a);
      for (int t = 0; !ti.done(a); ++t) {
        const int st = t % kLtStages;
        mbar_wait_sleep(&empty[st], ((t / kLtStages) & 1) ^ 1);
        const int64_t row = ((int64_t)ti.bl * a.K2 + 2 * ti.sp) * a.Npad;
        const uint32_t sb = st_base + st * kLtStageBytes, fb = smem_u32(&full[st]);
        // each trial's 128 (64) node rows are one contiguous 2 KB (1 KB) run: 1D bulk copies
        expect_tx_elect(fb, 6144);
        bulk_g2s_elect(sb, a.GA + row + ti.tij.x * kLtI, 2048, fb);
        bulk_g2s_elect(sb + 2048, a.GA + row + a.Npad + ti.tij.x * kLtI, 2048, fb);
        bulk_g2s_elect(sb + 4096, a.GB + row + ti.tij.y * kLtJ, 1024, fb);
        bulk_g2s_elect(sb + 4096 + 2048, a.GB + row + a.Npad + ti.tij.y * kLtJ, 1024, fb);
        ti.next(a);
      }
    } else if (warp == 1) {
      // ---------------------------------------------------------- MMA issuer
      constexpr uint32_t idT = lt_idesc(128), idS = lt_idesc(64);
      LtIt mi;
      mi.start(a);
      for (int t = 0; !mi.done(a); ++t) {
        const int st = t % kLtStages, b = t % 3;
        mbar_wait_sleep(&full[st], (t / kLtStages) & 1);
        mbar_wait_sleep(&tempty[b], ((t / 3) & 1) ^ 1);
        if ((STATS & kLtSum) && mi.sp == 0) mbar_wait_sleep(sempty, (mi.bseq & 1) ^ 1);
        tc_fence_after();
        const uint32_t sa = st_base + st * kLtStageBytes;
        tc_mma_elect(tmem + b * 128, lt_desc(sa, 2048), lt_desc(sa + 4096, 1024), idT, 0u);
        if (STATS & kLtSum)
          tc_mma_elect(tmem + kLtTmemSum, lt_desc(sa, 2048), lt_desc(sa + 4096, 2048), idS, mi.sp > 0 ? 1u : 0u);
        tc_commit_elect(&empty[st]);
        tc_commit_elect(&tfull[b]);
        mi.next(a);
      }
    }
  } else {
    asm volatile("setmaxnreg.inc.sync.aligned.u32 112;");
    // -------------------------------------------------------------- consumers
    const int cw = warp - 4, ct = threadIdx.x - 128;
    const int q = warp & 3, cgrp = cw >> 2;
    const uint32_t lane_addr = (uint32_t)(q * 32) << 16;
  const float invK = 1.f / (float)a.K;
  const float uspA = a.K > 1 ? (float)a.K / (float)(a.K - 1) : 0.f;
  const float uspB = a.K > 1 ? 1.f / (float)(a.K - 1) : 0.f;
  const float tph = (a.K & 1) ? kLtPhantom * kLtPhantom : 0.f;
  const float inv_nb = 1.f / (float)a.nbb;

  int s = 0;  // global step counter (TMEM buffer b = s % 3)
  for (int u = blockIdx.x; u < a.n_units; u += gridDim.x) {
    const int tu = u / a.nbc;
    const int bl_first = (u - tu * a.nbc) * a.bpc, bl_end = min(a.nbb, bl_first + a.bpc);
    const int2 tij = a.tiles[tu];
    const int iBase = tij.x * kLtI, jBase = tij.y * kLtJ;
    if (ct < kLtI) {  // row offsets of the tile rows
      const int ii = iBase + ct, i0 = iBase + (ct & ~31);
      const bool ok = ii >= a.i_lo && ii < a.i_hi && ii < a.N;
      const long long o0 = (long long)i0 * (a.N - 1) - (long long)i0 * (i0 - 1) / 2 - i0 - 1;
      const long long oi = (long long)ii * (a.N - 1) - (long long)ii * (ii - 1) / 2 - ii - 1;
      rel_s[ct] = ok ? (int)(oi - o0) : INT_MIN;
      if ((ct & 31) == 0) base_s[ct >> 5] = o0 - a.pair_base;
    }
    asm volatile("bar.sync 1, %0;" ::"n"(kLtConsumers * 32) : "memory");  // rel_s / base_s visible to all warps
  for (int bl = bl_first; bl < bl_end; ++bl) {
    float sabs[16], mn[16];
    unsigned neg[16];
#pragma unroll
    for (int p = 0; p < 16; ++p) {
      sabs[p] = 0.f;
      mn[p] = 3.0e38f;
      neg[p] = 0u;
    }
    const uint32_t tcol = tmem + lane_addr + cgrp * 16;
    for (int sp = 0; sp < n_sp; ++sp, ++s) {
      const int b = s % 3;
      mbar_wait_sleep(&tfull[b], (s / 3) & 1);
      tc_fence_after();
      // two halves of 8 columns (keeps 16 t registers live instead of 32)
#pragma unroll
      for (int hf = 0; hf < 2; ++hf) {
        float t0[8], t1[8];
        const uint32_t ta = tcol + b * 128 + hf * 8;
        lt_ld8x2(ta, t0, ta + 64, t1);
        if (hf == 1) {
          tc_fence_before();
          __syncwarp();
          if (lane == 0) mbar_arrive(&tempty[b]);
        }
#pragma unroll
        for (int v = 0; v < 8; ++v) {
          const int p = hf * 8 + v;
          if (STATS & kLtAbs) {
            sabs[p] += fabsf(t0[v]);
            sabs[p] += fabsf(t1[v]);
          }
          if (STATS & kLtSign) {  // sign bytes of (t0, t1) -> 0x0000FFFF [t0 < 0] + 0xFFFF0000 [t1 < 0]
            unsigned r;
            asm("prmt.b32 %0, %1, %2, 0xFFBB;" : "=r"(r) : "r"(__float_as_uint(t0[v])), "r"(__float_as_uint(t1[v])));
            asm("mad.lo.u32 %0, %1, 1, %0;" : "+r"(neg[p]) : "r"(r));  // IMAD: on the FMA pipe, not the ALU
          }
          mn[p] = fminf(mn[p], fminf(fabsf(t0[v]), fabsf(t1[v])));
        }
      }
    }
    const bool unit_last = bl + 1 == bl_end;

    // ------------------------------------------------ per-(pair, bin) epilogue
    float dsum[16];
    if (STATS & kLtSum) {
      lt_ld16(tmem + lane_addr + kLtTmemSum + cgrp * 16, dsum);
      tc_fence_before();
      __syncwarp();
      if (lane == 0) mbar_arrive(sempty);
    } else {
#pragma unroll
      for (int p = 0; p < 16; ++p) dsum[p] = 0.f;
    }
    const int r = q * 32 + lane, i = iBase + r;
    float Mi = 0.f, rPi = 0.f;
    if (i < a.N) {
      const float2 f = a.nf[(int64_t)bl * a.N + i];
      Mi = f.x;
      rPi = f.y;
    }
    const float gMi = a.g * Mi;
    const bool row_ok = i >= a.i_lo && i < a.i_hi && i < a.N;
    // final per-pair statistics -> three live arrays (IMAGCOHY, PLI, WPLI); the other
    // metrics are functions of these
    // final per-pair values, in place: dsum -> IMAGCOHY, neg -> PLI (float bits),
    // sabs -> WPLI; the other metrics are functions of these
    // column factors of the tile through shared memory (double-buffered by bin parity;
    // the barrier keeps warps within one bin of each other)
    float2* cnf = colnf + (bl & 1) * kLtJ;
    if (ct < kLtJ) {
      const int j = jBase + ct;
      cnf[ct] = j < a.N ? a.nf[(int64_t)bl * a.N + j] : make_float2(0.f, 0.f);
    }
    asm volatile("bar.sync 1, %0;" ::"n"(kLtConsumers * 32) : "memory");
    unsigned fmask = 0;
#pragma unroll
    for (int p = 0; p < 16; ++p) {
      const int j = jBase + cgrp * 16 + p;
      const float2 f = cnf[cgrp * 16 + p];
      const bool valid = row_ok && i < j && j < a.N;
      const bool dead = Mi * f.x == 0.f;
      if (valid && !dead && mn[p] <= gMi * f.x) {  // rare: the fp64 fallback writes this (pair, bin)
        fmask |= 1u << p;
        const int slot = atomicAdd(&a.counters[0], 1);
        if (slot < a.flag_cap)
          a.flags[slot] = make_int4(i, j, bl, 0);
        else
          a.counters[1] = 1;
      }
      const unsigned nA = (0u - neg[p]) & 0xFFFFu, nB = ((65535u * nA - neg[p]) >> 16) & 0xFFFFu;
      const float s_im = dead ? 0.f : dsum[p] - tph;   // sum Im (scaled)
      const float s_abs = dead ? 0.f : sabs[p] - tph;  // sum |Im|
      neg[p] = __float_as_uint(dead ? 0.f : fabsf((float)(a.K - 2 * (int)(nA + nB))) * invK);
      dsum[p] = s_im * rPi * f.y;
      sabs[p] = s_abs > 0.f ? fminf(fabsf(s_im) * rcp_approx(s_abs), 1.f) : 0.f;
    }
    const bool first_bin = bl == bl_first;
    const int64_t bo = (int64_t)bl * a.pair_stride;
    float* my_stg = stg + cw * 32 * kLtStgStride;
#pragma unroll
    for (int m = 0; m < 5; ++m) {
      float* const dst = a.bins[m];
      const bool do_band = a.band[m] != nullptr;
      if (!dst && !do_band) continue;
#pragma unroll
      for (int p = 0; p < 16; ++p) {
        float v;
        const float pli = __uint_as_float(neg[p]);
        if (m == 0) v = dsum[p];
        else if (m == 1) v = pli;
        else if (m == 2) v = pli * pli * uspA - uspB;
        else if (m == 3) v = sabs[p];
        else v = sabs[p] * sabs[p];
        if (fmask & (1u << p)) v = __int_as_float(0x7fffffff);  // NaN: written by the fallback
        my_stg[lane * kLtStgStride + p] = v;
      }
      if (m == 0 && do_band) {  // IMAGCOHY band sums live in TMEM (this thread's row, 16 columns)
#pragma unroll
        for (int hf = 0; hf < 2; ++hf) {
          float bs[8];
          const uint32_t tb = tmem + lane_addr + kLtTmemBand + cgrp * 16 + hf * 8;
          if (!first_bin) lt_ld8(tb, bs);
#pragma unroll
          for (int u = 0; u < 8; ++u) {
            const int p = hf * 8 + u, j = jBase + cgrp * 16 + p;
            const float add = (row_ok && i < j && j < a.N && !(fmask & (1u << p))) ? dsum[p] : 0.f;
            bs[u] = first_bin ? add : bs[u] + add;
          }
          lt_st8(tb, bs);
        }
      }
      __syncwarp();
      // transposed: half-warp h covers row rr + h, lanes over 16 contiguous columns
      const int hr = lane >> 4, cl = lane & 15;
      const int C = cgrp * 16 + cl, gj = jBase + C;
      const long long wbase = base_s[q];
      float* const bm = band_s + (m - 1) * kLtI * kLtJ;
      const bool sband = do_band && m > 0;
#pragma unroll 1
      for (int rr = 0; rr < 32; rr += 2) {
        const int rl = rr + hr, R = q * 32 + rl, gi = iBase + R;
        const float v = my_stg[rl * kLtStgStride + cl];
        const int rel = rel_s[R];
        const bool ok = rel != INT_MIN && gi < gj && gj < a.N && v == v;
        if (dst && ok) __stcs(dst + bo + wbase + rel + gj, v);
        if (sband) {
          float* bp = bm + R * kLtJ + (C ^ ((R & 1) << 4));
          const float add = ok ? v : 0.f;
          *bp = first_bin ? add : *bp + add;
        }
      }
      __syncwarp();
    }
    if (unit_last) {
      // band means of the unit: rows w, w + 16, ... (all warps' band slots complete)
      asm volatile("bar.sync 1, %0;" ::"n"(kLtConsumers * 32) : "memory");
      if (a.band[0]) {  // IMAGCOHY: TMEM -> per-warp staging -> rows
        float bs[16];
        asm volatile("tcgen05.wait::st.sync.aligned;" ::: "memory");
        lt_ld16(tmem + lane_addr + kLtTmemBand + cgrp * 16, bs);
        float* my_stg = stg + cw * 32 * kLtStgStride;
#pragma unroll
        for (int p = 0; p < 16; ++p) my_stg[lane * kLtStgStride + p] = bs[p];
        __syncwarp();
        const int hr = lane >> 4, cl = lane & 15;
        const int C = cgrp * 16 + cl, gj = jBase + C;
        for (int rr = 0; rr < 32; rr += 2) {
          const int rl = rr + hr, R = q * 32 + rl, gi = iBase + R;
          const int rel = rel_s[R];
          if (rel != INT_MIN && gi < gj && gj < a.N) {
            const float v = my_stg[rl * kLtStgStride + cl] * inv_nb;
            float* d = a.band[0] + base_s[q] + rel + gj;
            if (a.nbc > 1) atomicAdd(d, v);
            else __stcs(d, v);
          }
        }
        __syncwarp();
      }
      for (int m = 1; m < 5; ++m) {
        float* const dst = a.band[m];
        if (!dst) continue;
        for (int R = cw; R < kLtI; R += kLtConsumers) {
          const int rel = rel_s[R];
          if (rel == INT_MIN) continue;
          const int gi = iBase + R;
          const long long ro = base_s[R >> 5] + rel;
#pragma unroll
          for (int h = 0; h < 2; ++h) {
            const int C = lane + 32 * h, gj = jBase + C;
            if (gi < gj && gj < a.N) {
              const float v = band_s[(m - 1) * kLtI * kLtJ + R * kLtJ + (C ^ ((R & 1) << 4))] * inv_nb;
              if (a.nbc > 1) atomicAdd(dst + ro + gj, v);
              else __stcs(dst + ro + gj, v);
            }
          }
        }
      }
      // the next unit's rel_s / band writes wait for every warp's reads
      asm volatile("bar.sync 1, %0;" ::"n"(kLtConsumers * 32) : "memory");
    }
  }  // bins
  }  // units
  }

  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  if (warp == 2) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 512;" ::"r"(tmem));
}

// ---------------------------------------------------------------- operand prep
// GA/GB[bl][kk][n] (8 halves each) from the fp64 ring, kk < K2 (odd K: phantom at kk = K),
// n < Npad (zero padded).  Node factors nf[bl][n] from the node statistics.
__global__ void k_lagtc_prep(const double2* __restrict__ X64, const int* __restrict__ slots, int K, int K2, int N,
                             int Npad, int nb, int bin_lo, float scale, const float* __restrict__ nscale,
                             const float* __restrict__ mag, const float* __restrict__ psd, int real0, int real1,
                             uint4* __restrict__ GA, uint4* __restrict__ GB, float2* __restrict__ nf) {
  const int n = blockIdx.x * blockDim.x + threadIdx.x;
  const int kk = blockIdx.y, bl = blockIdx.z;
  if (n >= Npad) return;
  __half e[8], f[8];
  const __half z = __float2half_rn(0.f);
#pragma unroll
  for (int c = 0; c < 8; ++c) e[c] = f[c] = z;
  if (n < N) {
    const float s = nscale[(int64_t)bl * N + n];
    if (kk < K) {
      const double2 v = X64[((int64_t)slots[kk] * nb + bin_lo + bl) * N + n];
      const double sc = (double)scale * (double)s;
      const double re = v.x * sc, im = v.y * sc;
      const __half rh = __double2half(re), ih = __double2half(im);
      const __half rl = __double2half(re - (double)__half2float(rh)), il = __double2half(im - (double)__half2float(ih));
      const __half nrh = __hneg(rh), nrl = __hneg(rl);
      e[0] = ih; e[1] = il; e[2] = ih; e[3] = il; e[4] = nrh; e[5] = nrl; e[6] = nrh; e[7] = nrl;
      f[0] = rh; f[1] = rh; f[2] = rl; f[3] = rl; f[4] = ih; f[5] = ih; f[6] = il; f[7] = il;
    } else {  // phantom: A Im_h = 2^-5, B Re_h = 2^-5 -> t = 2^-10
      const __half ph = __float2half_rn(kLtPhantom);
      e[0] = ph; e[2] = ph;
      f[0] = ph; f[1] = ph;
    }
    if (kk == 0) {
      const int b = bin_lo + bl;
      const float m = mag[(int64_t)bl * N + n], pw = psd[(int64_t)bl * N + n];
      const float mh = (b == real0 || b == real1) ? 0.f : m * s;
      nf[(int64_t)bl * N + n] = make_float2(mh, pw > 0.f ? rsqrtf(pw * s * s) : 0.f);
    }
  }
  const int64_t o = ((int64_t)bl * K2 + kk) * Npad + n;
  GA[o] = *(const uint4*)e;
  GB[o] = *(const uint4*)f;
}

// ---------------------------------------------------------------- host side
const int2* tc_tile_list(Plan& p, int i_lo, int i_hi, int nt64, int64_t* n_tiles, cudaStream_t st);

size_t lagtc_smem_bytes() {
  return (size_t)kLtStages * kLtStageBytes + kLtBandBytes + kLtStgBytes + kLtI * 4 + 4 * 8 + 2 * kLtJ * 8 +
         (2 * kLtStages + 7) * 8 + 16;
}

bool run_pairs_lagtc(Plan& p, const int* slots, int K, int bin_lo, int nbb, int rb, int re, float* const* bins,
                     float* const* band, int64_t pair_base, int64_t pair_stride, cudaStream_t st) {
  const int K2 = (K + 1) / 2 * 2;
  const int Npad = (p.N + kLtI - 1) / kLtI * kLtI;
  const size_t nops = (size_t)nbb * K2 * Npad;
  const size_t need = 2 * nops * sizeof(uint4) + (size_t)nbb * p.N * sizeof(float2);
  if (need > p.lag_bytes) {
    if (p.lag_ops) cudaFreeAsync(p.lag_ops, st);
    if (cudaMallocAsync(&p.lag_ops, need, st) != cudaSuccess) {
      p.lag_ops = nullptr;
      p.lag_bytes = 0;
      cs_set_error("device allocation failed (phase-lag operands %zu bytes)", need);
      return false;
    }
    p.lag_bytes = need;
  }
  uint4* GA = (uint4*)p.lag_ops;
  uint4* GB = GA + nops;
  float2* nf = (float2*)(GB + nops);
  {
    PhaseMark ph(p, "lag_prep", st);
    dim3 grid((Npad + 127) / 128, K2, nbb);
    k_lagtc_prep<<<grid, 128, 0, st>>>(p.X64, slots, K, K2, p.N, Npad, p.nb, bin_lo, p.scale, p.nscale, p.mag,
                                       p.psd, p.dc_local, p.nyq_local, GA, GB, nf);
  }
  LtArgs a{};
  a.N = p.N; a.K = K; a.K2 = K2; a.Npad = Npad; a.nbb = nbb; a.bin_lo = bin_lo;
  a.i_lo = rb * kTile;
  a.i_hi = re * kTile < p.N ? re * kTile : p.N;
  const int nt64 = (p.N + kLtJ - 1) / kLtJ;
  int64_t n_tiles = 0;
  a.tiles = tc_tile_list(p, a.i_lo, a.i_hi, nt64, &n_tiles, st);
  if (!a.tiles) return false;
  int nsm = 148;
  cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, p.device);
  {  // bin split for small pair spaces: rounds x (unit overhead ~1 bin + bins per unit)
    int nbc = 1;
    double best = 1e300;
    for (int c = 1; c <= nbb && n_tiles > 0; ++c) {
      const int bpc = (nbb + c - 1) / c, chunks = (nbb + bpc - 1) / bpc;
      if (chunks != c) continue;
      const double cost = (double)((n_tiles * chunks + nsm - 1) / nsm) * (1.0 + bpc);
      if (cost < best) {
        best = cost;
        nbc = c;
      }
    }
    static const int force_nbc = getenv("CSCONN_K3_NBC") ? atoi(getenv("CSCONN_K3_NBC")) : 0;
    if (force_nbc) nbc = force_nbc < 1 ? 1 : (force_nbc > nbb ? nbb : force_nbc);
    a.bpc = (nbb + nbc - 1) / nbc;
    a.nbc = (nbb + a.bpc - 1) / a.bpc;
  }
  a.n_units = (int)(n_tiles * a.nbc);
  a.nf = nf;
  a.GA = GA;
  a.GB = GB;
  a.pair_base = pair_base; a.pair_stride = pair_stride;
  unsigned need_st = 0;
  for (int m = 0; m < 5; ++m) {
    a.bins[m] = bins[m];
    a.band[m] = band[m];
    const bool w = bins[m] || band[m];
    if (w && (m == 1 || m == 2)) need_st |= kLtSign;
    if (w && (m == 0 || m == 3 || m == 4)) need_st |= kLtSum;
    if (w && (m == 3 || m == 4)) need_st |= kLtAbs;
  }
  a.g = 1.5f * (11.4f + 8.f) * 5.9604645e-8f;
  a.flags = p.flags;
  a.counters = p.counters;
  a.flag_cap = p.flag_cap;
  if (a.nbc > 1)
    for (int m = 0; m < 5; ++m)
      if (band[m]) cudaMemsetAsync(band[m], 0, pair_stride * sizeof(float), st);
  const size_t smem = lagtc_smem_bytes();
  PhaseMark ph(p, "pairs_lag", st);
  if (a.n_units == 0) return true;
  const unsigned grid = (unsigned)(a.n_units < nsm ? a.n_units : nsm);
#define CS_LT(SS)                                                            \
  do {                                                                       \
    CS_SMEM_ONCE(k_pairs_lagtc<SS>, smem);                                  \
    k_pairs_lagtc<SS><<<grid, kLtThreads, smem, st>>>(a);            \
  } while (0)
  switch (need_st) {
    case kLtSign: CS_LT(kLtSign); break;
    case kLtSum: CS_LT(kLtSum); break;
    case kLtSign | kLtSum: CS_LT(kLtSign | kLtSum); break;
    case kLtSum | kLtAbs: CS_LT(kLtSum | kLtAbs); break;
    default: CS_LT(kLtAll); break;
  }
#undef CS_LT
  return true;
}

}  // namespace cs
