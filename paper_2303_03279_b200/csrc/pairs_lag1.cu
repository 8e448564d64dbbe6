// K3: the phase-lag family (PLI, USPLI, WPLI, DSWPLI) + IMAGCOHY (+ multitaper PLV) on the
// FP32/ALU pipes, with a TMA producer and an mbarrier ring instead of CTA-wide barriers.
//
// Reference: spectral.py:216-241 (_fold_csd: Im flush, sign(Im), |Im|, Im sums),
// metrics.py:49-86 (imagcohy / pli / uspli / wpli / dswpli), metrics.py:115-134
// and core.py:208-215 (band mean).
//
// CTA = 64 x 64 node tile x all bins of the band (small pair spaces: a bin chunk).  16
// compute warps (512 threads, each 4 x 2 pairs: i = ty + 16 r, j = tx + 32 c; common.cuh
// kGuardTR x kGuardTC); single taper adds a producer warpgroup whose first thread issues the
// TMA loads (multitaper: warp 0 lane 0).  The packed trial-pair operands (k_lag_prep: float4
// (re_a, re_b, im_a, im_b), J side with Im negated) are streamed by 2D TMA boxes of 64 nodes
// x up to 26 rows into a 2-stage ring; consumers wait on the stage's full barrier and release
// it with one arrive per warp.  Per trial pair and pair of nodes: FMUL2 + FFMA2 (t = Im X_i
// conj X_j for two trials), 2 FADD |.| (sum |t|), PRMT + 1/2 IADD3 (packed #(t < 0)),
// FMNMX3 (min |t|, the exact-sign guard of pairs_lag.cu) and, unless the tensor-core kernel
// hands IMAGCOHY over, FADD2 (sum t).
#include <type_traits>

#include "common.cuh"
#include "ptx.cuh"

namespace cs {

#ifndef CS_K3_ROWS
#define CS_K3_ROWS 26
#endif
#ifndef CS_K3_STAGES
#define CS_K3_STAGES 2
#endif
constexpr int k1Rows = CS_K3_ROWS;       // max operand rows (trial pair x taper) per stage
constexpr int k1Stages = CS_K3_STAGES;   // (build-time overrides for stage sweeps)
constexpr int k1TR = kGuardTR, k1TC = kGuardTC;  // pairs per thread (rows x cols; common.cuh)
constexpr int k1TY = kTile / k1TR, k1TX = kTile / k1TC;
constexpr int k1NP = k1TR * k1TC;
constexpr int k1Warps = k1TY * k1TX / 32;  // compute warps
constexpr int k1Threads = k1Warps * 32;        // multitaper: lane 0 of warp 0 also issues the TMA loads
constexpr int k1Quads = k1NP / 4;              // float4 band slots per thread and metric
constexpr int k1RowsPerQuad = 4 / k1TC;        // tile rows of a band slot's four pairs
constexpr int k1LanesPerRow = k1TX < 32 ? k1TX : 32;
// single taper: plus a producer warpgroup (the first producer warp issues the TMA loads, the
// others idle) whose registers go to the compute warps with setmaxnreg: the launch gives every
// thread k1RegLaunch registers, the producers drop to 24 and the compute warps rise to
// k1RegCompute (4 x 4 pairs, 8 compute warps: 384 x 168 = 128 x 24 + 256 x 240)
constexpr int k1ThreadsP = k1Threads + 128;
constexpr int k1RegLaunch = ((65536 / k1ThreadsP) & ~7) > 255 ? 248 : ((65536 / k1ThreadsP) & ~7);
constexpr int k1RegProducer = 24;
constexpr int k1RegCompute0 = ((k1ThreadsP * k1RegLaunch - 128 * k1RegProducer) / k1Threads) & ~7;
constexpr int k1RegCompute = k1RegCompute0 > 240 ? 240 : k1RegCompute0;
static_assert(k1TC == 2 || k1TC == 4, "band slots hold 4 pairs: 2 rows x 2 or 1 row x 4");
constexpr int k1StageF4 = k1Rows * kTile;  // float4 per side per stage
constexpr float k1Phantom = 9.765625e-4f;  // 2^-10 (see k_lag_prep)

// Exact-sign guard work list.  A warp whose (pair, bin) entries are flagged reserves
// list slots with one atomic; when the list is full it instead appends one record
// (row of its first pair, tile column base, bin, 256-bit mask over its 4 x 2 x 32 pairs)
// to a record list sized for every (tile, bin, warp) of the call, so no flagged entry is
// ever dropped (k_lag_fallback processes both).  counters: [0] flagged entries,
// [1] list overflowed, [2] records.
__device__ __noinline__ void guard_push(int4* flags, int4* recs, int* counters, int cap, unsigned fl,
                                        int iBase, int jBase, int ty, int tx, int lane, int bl) {
  const int n = __popc(fl);
  int incl = n;
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    const int v = __shfl_up_sync(0xffffffffu, incl, o);
    if (lane >= o) incl += v;
  }
  const int total = __shfl_sync(0xffffffffu, incl, 31);
  int base = 0;
  if (lane == 31) base = atomicAdd(&counters[0], total);
  base = __shfl_sync(0xffffffffu, base, 31);
  if (base + total <= cap) {
    int s = base + incl - n;
#pragma unroll
    for (int r = 0; r < k1TR; ++r)
#pragma unroll
      for (int c = 0; c < k1TC; ++c)
        if ((fl >> (r * k1TC + c)) & 1u)
          flags[s++] = make_int4(iBase + ty + k1TY * r, jBase + tx + k1TX * c, bl, 0);
    return;
  }
  // slots this warp reserved below the capacity stay unused: mark them empty
  for (int s = base + lane; s < min(cap, base + total); s += 32) flags[s] = make_int4(-1, -1, 0, 0);
  unsigned m[k1NP];
#pragma unroll
  for (int q = 0; q < k1NP; ++q) m[q] = __ballot_sync(0xffffffffu, (fl >> q) & 1u);
  if (lane == 0) {  // lane 0 holds tx = 0 and the warp's first row ty
    const int rec = atomicAdd(&counters[2], 1);
    recs[kGuardRecI4 * rec] = make_int4(iBase + ty, jBase, bl, k1LanesPerRow);
#pragma unroll
    for (int w4 = 0; w4 < k1Quads; ++w4)
      recs[kGuardRecI4 * rec + 1 + w4] =
          make_int4((int)m[4 * w4], (int)m[4 * w4 + 1], (int)m[4 * w4 + 2], (int)m[4 * w4 + 3]);
    counters[1] = 1;
  }
}
static_assert(k1NP == kGuardNP && k1Warps == kGuardWarps && k1TY == kGuardRowStep && k1TX == kGuardColStep &&
                  k1TC == kGuardTC && k1NP <= 32,
              "guard record layout (common.cuh)");

// first pair index of row i minus one, i (N - 1) - i (i - 1) / 2 - i - 1, mod 2^32: the FULL
// path's per-bin offsets are host-checked < 2^32, so unsigned wrap-around is exact
__device__ __forceinline__ uint32_t row_off32(uint32_t i, uint32_t N) {
  const uint32_t tri = (i & 1u) ? i * ((i - 1u) >> 1) : (i >> 1) * (i - 1u);
  return i * (N - 1u) - tri - i - 1u;
}

struct Lag1Args {
  int N, N64, K, Kp, bin_lo, nbb;
  int bpc, nbc;              // bins per CTA, bin chunks per tile (small pair spaces split bins)
  const float* psd;
  const float* mag;
  int real0, real1, nt, row_begin;
  int64_t pair_base, pair_stride;
  float* bins[5];
  float* band[5];
  float* plv_bins;           // multitaper: PLV of the taper-mean CSD (PLVK instantiation)
  float* plv_band;
  float g;
  int4* flags;
  int4* recs;
  int* counters;
  int flag_cap;
  bool wide;                 // K >= 2^17: sign counts decoded per stage (see neg[] below)
  const float* imag_in;      // IMAGIN: IMAGCOHY per bin from the tensor-core kernel, [nbb][pair_stride]
  float imag_tau;            // IMAGIN: its error bound (entries below it went to the fp64 fallback)
  const float4* nf;          // [nbb][N64] node factors {M', rsqrt(psd) / s, rsqrt(psd), M' 2^-10}
                             // (k_lag_prep; M' = 0 on exactly-real bins, s = the fp16 operand scale):
                             // the FULL epilogue's per-node inputs
};


// L == 1 uses a dedicated producer warpgroup (20 warps; setmaxnreg gives the 16 compute
// warps 112 registers and the producers 24); L > 1 needs 128 registers, so 16 warps
// with the TMA issued from warp 0.
// STATS: which per-pair trial statistics the requested metrics need (the exact-sign
// guard min |t| is always kept): 1 = #(t < 0) (PLI, USPLI), 2 = sum t (IMAGCOHY, WPLI,
// DSWPLI), 4 = sum |t| (WPLI, DSWPLI).  Single taper only; multitaper runs all.
constexpr unsigned kStSign = 1, kStSum = 2, kStAbs = 4, kStAll = 7;
// FULL: every per-bin and band output is requested (the fused all-metrics call), so the
// epilogue needs no per-store pointer checks.
// WIDE: K >= 2^17 trials, where the two 16-bit sign-count fields could wrap: the
// packed counts are decoded into plain 32-bit counters after every stage.
// IMAGIN: the tensor-core kernel already wrote the per-bin IMAGCOHY for this call (its
// D_im is sum Im; this kernel still forms the band mean); sum t is not accumulated here -- WPLI's numerator is IMAGCOHY sqrt(psd_i psd_j)
// -- which takes the FADD2 out of the trial loop (see run_lag_family).
template <int L, bool PLVK, unsigned STATS = kStAll, bool FULL = false, bool WIDE = false, bool IMAGIN = false>
__global__ void __launch_bounds__(L == 1 ? k1ThreadsP : k1Threads, 1)
k_pairs_lag1(const __grid_constant__ CUtensorMap mapI, const __grid_constant__ CUtensorMap mapJ, const Lag1Args a) {
  constexpr int KCL = k1Rows / L;  // max trial pairs per stage
  constexpr int NM = PLVK ? 6 : 5;
  extern __shared__ __align__(128) unsigned char lag1_smem[];
  float4* XI = (float4*)lag1_smem;                       // [stages][KC][64]
  float4* XJ = XI + k1Stages * k1StageF4;                // [stages][KC][64]
  float* band_s = (float*)(XJ + k1Stages * k1StageF4);  // [NM][64][64]
  // FULL single-taper epilogue (kF): band_s holds per-thread band sums instead, float4
  // [metric][pair half][compute thread] (80 KB), then IMAGCOHY staging [pair][thread]
  // (16 KB); nf_s: the bin's node factors [bin % 3][I 64 | J 64], bulk-copied by the
  // producer with the bin's last stage
  constexpr bool kF = FULL && L == 1;
  float4* band4 = (float4*)band_s;
  float* imv_s = band_s + 5 * kTile * kTile;
  float4* nf_s = (float4*)(band_s + 6 * kTile * kTile);
  uint64_t* full = (uint64_t*)(nf_s + 3 * 2 * kTile);
  uint64_t* empty = full + k1Stages;

  int I, J;
  const int bchunk = blockIdx.x % a.nbc;
  decode_tile(blockIdx.x / a.nbc, a.nt, a.row_begin, I, J);
  const int bl0 = bchunk * a.bpc;                      // first bin (of the call's nbb) of this CTA
  const int nbl = min(a.bpc, a.nbb - bl0);
  const int iBase = I * kTile, jBase = J * kTile;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const bool interior = iBase + kTile <= jBase && jBase + kTile <= a.N;  // every i < j < N

  unsigned bin_mask = 0, band_mask = 0;
#pragma unroll
  for (int m = 0; m < 5; ++m) {
    bin_mask |= (a.bins[m] != nullptr) << m;
    band_mask |= (a.band[m] != nullptr) << m;
  }
  if (PLVK) {
    bin_mask |= (a.plv_bins != nullptr) << 5;
    band_mask |= (a.plv_band != nullptr) << 5;
  }
  if (FULL) {  // IMAGIN: the per-bin IMAGCOHY is the tensor-core kernel's, its band mean is summed here
    bin_mask = IMAGIN ? 30u : 31u;
    band_mask = 31u;
  }
  const int n_stage = (a.Kp + KCL - 1) / KCL;
  int kc = (a.Kp + n_stage - 1) / n_stage;         // balanced stage size (<= KCL trial pairs)
  if (L == 1 && (kc & 1) && kc < KCL) ++kc;        // even stages: the 2-unrolled loop has no remainder
  const int total = n_stage * nbl;
  constexpr bool kDedicated = L == 1;
  // single taper: the producer thread (warp 16, lane 0) issues stage t
  const bool producer = kDedicated && warp == k1Warps && lane == 0;
  auto produce = [&](int t) {
    const int s = t % k1Stages;
    mbar_wait_backoff(&empty[s], ((t / k1Stages) & 1) ^ 1);
    const int bl = bl0 + t / n_stage, st = t % n_stage;
    const int row = (bl * a.Kp + st * kc) * L;
    const bool nf_now = kF && st == n_stage - 1;  // the bin's node factors ride on its last stage
    mbar_expect_tx(&full[s], 2 * (k1Rows / L) * L * kTile * 16 + (nf_now ? 2 * kTile * 16 : 0));
    tma_load_2d(XI + s * k1StageF4, &mapI, &full[s], iBase * 4, row);
    tma_load_2d(XJ + s * k1StageF4, &mapJ, &full[s], jBase * 4, row);
    if (nf_now) {
      float4* dst = nf_s + (bl % 3) * 2 * kTile;
      bulk_load_1d(dst, a.nf + (int64_t)bl * a.N64 + iBase, kTile * 16, &full[s]);
      bulk_load_1d(dst + kTile, a.nf + (int64_t)bl * a.N64 + jBase, kTile * 16, &full[s]);
    }
  };
  // the barriers are initialised by the thread that issues the TMA loads, which then starts
  // the first stages at once, so their latency overlaps the band zeroing and the CTA barrier
  if (threadIdx.x == (kDedicated ? k1Warps * 32 : 0)) {
    for (int s = 0; s < k1Stages; ++s) {
      mbar_init(&full[s], 1);
      mbar_init(&empty[s], k1Warps);
    }
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    if (kDedicated)
      for (int t = 0; t < min(k1Stages, total); ++t) produce(t);
  }
  if (band_mask)
    for (int e = threadIdx.x; e < NM * kTile * kTile; e += blockDim.x) band_s[e] = 0.f;
  __syncthreads();

  // multitaper TMA issue (warp 0, lane 0): stage t into slot t % stages once every warp has
  // released that slot's previous use.  16 warps = 4 per SMSP keep 128 registers
  // per thread available (a 17th producer warp would cap them at 96).
  auto issue = [&](int t) {
    if (!kDedicated && warp == 0 && lane == 0 && t < total) {
      const int s = t % k1Stages;
      mbar_wait(&empty[s], ((t / k1Stages) & 1) ^ 1);
      const int bl = bl0 + t / n_stage, st = t % n_stage;
      const int row = (bl * a.Kp + st * kc) * L;
      mbar_expect_tx(&full[s], 2 * (k1Rows / L) * L * kTile * 16);  // exactly the two TMA boxes
      tma_load_2d(XI + s * k1StageF4, &mapI, &full[s], iBase * 4, row);
      tma_load_2d(XJ + s * k1StageF4, &mapJ, &full[s], jBase * 4, row);
    }
  };
  if (kDedicated) {
    if (warp >= k1Warps) {  // producer warpgroup: 24 registers; warp 16 lane 0 issues the stages
      asm volatile("setmaxnreg.dec.sync.aligned.u32 %0;" ::"n"(k1RegProducer));
      if (producer)
        for (int t = k1Stages; t < total; ++t) produce(t);
      return;
    }
    asm volatile("setmaxnreg.inc.sync.aligned.u32 %0;" ::"n"(k1RegCompute));
  } else {
    for (int t = 0; t < k1Stages - 1; ++t) issue(t);
  }

  // ------------------------------------------------------------ compute warps
  const int tid = threadIdx.x, tx = tid % k1TX, ty = tid / k1TX;
  const bool odd = a.K & 1;
  const float invK = 1.f / (float)a.K;
  const float uspA = a.K > 1 ? (float)a.K / (float)(a.K - 1) : 0.f;
  const float uspB = a.K > 1 ? 1.f / (float)(a.K - 1) : 0.f;

  f2 sim[k1NP];
  float sabs[k1NP], mn[k1NP];
  // #(t < 0), two trials per PRMT: the sign bytes of (t_a, t_b) replicated into
  // 0x0000FFFF [t_a < 0] + 0xFFFF0000 [t_b < 0]; two trial pairs are added with one
  // IADD3 (3 instructions per 4 trials instead of 4 LEA.HI).  Decoded exactly in
  // the epilogue: A = -acc mod 2^16, B = (65535 A - acc) >> 16 (counts < 2^16).
  unsigned neg[k1NP], ntmp[k1NP], negw[WIDE ? k1NP : 1];
  f2 pvr[PLVK ? k1NP : 1], pvi[PLVK ? k1NP : 1];
#pragma unroll
  for (int p = 0; p < k1NP; ++p) {
    sim[p] = 0ull;
    sabs[p] = 0.f;
    mn[p] = 3.0e38f;
    neg[p] = 0u;
    ntmp[p] = 0u;
    if (WIDE) negw[p] = 0u;
    if (PLVK) pvr[p] = pvi[p] = 0ull;
  }

  int bl = bl0, st = -1;  // bin and stage-in-bin of step t, advanced incrementally (no divisions)
  for (int t = 0; t < total; ++t) {
    issue(t + k1Stages - 1);
    if (++st == n_stage) {
      st = 0;
      ++bl;
    }
    const int s = t % k1Stages;
    if (kF && IMAGIN && st == n_stage - 1) {
      // the bin's tensor-core IMAGCOHY of this thread's pairs, copied while the last stage runs
      const uint32_t bin_off = (uint32_t)bl * (uint32_t)a.pair_stride;
#pragma unroll
      for (int r = 0; r < k1TR; ++r) {
        const uint32_t i = (uint32_t)(iBase + ty + k1TY * r);
        const uint32_t ro = row_off32(i, (uint32_t)a.N) - (uint32_t)a.pair_base + bin_off;
#pragma unroll
        for (int c = 0; c < k1TC; ++c) {
          const int j = jBase + tx + k1TX * c;
          if ((int)i < j && j < a.N)
            cp_async_4(smem_u32(imv_s + (r * k1TC + c) * k1Threads + tid), a.imag_in + (ro + (uint32_t)j));
        }
      }
    }
    mbar_wait(&full[s], (t / k1Stages) & 1);
    const float4* sI = XI + s * k1StageF4;
    const float4* sJ = XJ + s * k1StageF4;
    const int nkp = min(kc, a.Kp - st * kc);
    auto stats = [&](int p, f2 tt, int odd) {
      if (STATS & kStSum) sim[p] = fadd2(sim[p], tt);
      const float tl = lo_of(tt), th = hi_of(tt);
      if (STATS & kStAbs) {
        sabs[p] += fabsf(tl);
        sabs[p] += fabsf(th);
      }
      if (!(STATS & kStSign)) {
      } else if (L == 1) {
        unsigned r;
        asm("prmt.b32 %0, %1, %2, 0xFFBB;" : "=r"(r) : "r"(__float_as_uint(tl)), "r"(__float_as_uint(th)));
        if (odd) neg[p] += ntmp[p] + r;
        else ntmp[p] = r;
      } else {  // multitaper: registers are tighter, plain counts (LEA.HI)
        neg[p] += __float_as_uint(tl) >> 31;
        neg[p] += __float_as_uint(th) >> 31;
      }
      mn[p] = fminf(mn[p], fminf(fabsf(tl), fabsf(th)));
    };
    auto body = [&](int kp) {
      if (L == 1) {
        float4 xi[k1TR], xj[k1TC];
#pragma unroll
        for (int r = 0; r < k1TR; ++r) xi[r] = sI[kp * kTile + ty + k1TY * r];
#pragma unroll
        for (int c = 0; c < k1TC; ++c) xj[c] = sJ[kp * kTile + tx + k1TX * c];
#pragma unroll
        for (int r = 0; r < k1TR; ++r) {
          const f2 ir = pk(xi[r].x, xi[r].y), ii = pk(xi[r].z, xi[r].w);
#pragma unroll
          for (int c = 0; c < k1TC; ++c) {
            const f2 jr = pk(xj[c].x, xj[c].y), jn = pk(xj[c].z, xj[c].w);
            stats(r * k1TC + c, ffma2(ii, jr, fmul2(ir, jn)), kp & 1);  // Im(X_i conj X_j), trials a, b
          }
        }
      } else {
        // multitaper: t = sum_l Im(X_il conj X_jl) (the 1/L of the taper mean cancels)
        float4 xj[L][k1TC];
#pragma unroll
        for (int l = 0; l < L; ++l)
#pragma unroll
          for (int c = 0; c < k1TC; ++c) xj[l][c] = sJ[(kp * L + l) * kTile + tx + k1TX * c];
#pragma unroll
        for (int r = 0; r < k1TR; ++r) {
          float4 xi[L];
#pragma unroll
          for (int l = 0; l < L; ++l) xi[l] = sI[(kp * L + l) * kTile + ty + k1TY * r];
#pragma unroll
          for (int c = 0; c < k1TC; ++c) {
            const int p = r * k1TC + c;
            f2 tt = 0ull, re1 = 0ull, re2 = 0ull;
#pragma unroll
            for (int l = 0; l < L; ++l) {
              const f2 ir = pk(xi[l].x, xi[l].y), ii = pk(xi[l].z, xi[l].w);
              const f2 jr = pk(xj[l][c].x, xj[l][c].y), jn = pk(xj[l][c].z, xj[l][c].w);
              tt = ffma2(ii, jr, ffma2(ir, jn, tt));
              if (PLVK) {  // Re = sum ir jr + ii ji = re1 - re2 with re2 = sum ii (-ji)
                re1 = ffma2(ir, jr, re1);
                re2 = ffma2(ii, jn, re2);
              }
            }
            stats(p, tt, kp & 1);
            if (PLVK) {  // unit phasor of the trial's taper-mean CSD
              f2 re;
              asm("sub.rn.f32x2 %0, %1, %2;" : "=l"(re) : "l"(re1), "l"(re2));
              // |CSD|^2 clamped to FLT_MIN: a zero CSD (dead node) then adds 0 * 2^63 = 0,
              // and the MUFU needs no denormal fix-up (scaled spectra are O(1))
              const f2 m2 = ffma2(tt, tt, fmul2(re, re));
              const float ml = fmaxf(lo_of(m2), 1.17549435e-38f), mh = fmaxf(hi_of(m2), 1.17549435e-38f);
              const f2 rs = pk(rsqrt_approx(ml), rsqrt_approx(mh));
              pvr[p] = ffma2(re, rs, pvr[p]);
              pvi[p] = ffma2(tt, rs, pvi[p]);
            }
          }
        }
      }
    };
    constexpr int kUnroll = L == 1 ? 2 : 1;  // multitaper: one trial pair at a time (registers)
#pragma unroll kUnroll
    for (int kp = 0; kp < nkp; ++kp) body(kp);
    if (L == 1 && (STATS & kStSign) && (nkp & 1)) {  // the stage's last trial pair had no partner
#pragma unroll
      for (int p = 0; p < k1NP; ++p) neg[p] += ntmp[p];
    }
    if (WIDE && L == 1 && (STATS & kStSign)) {  // < 2^16 per field within one stage
#pragma unroll
      for (int p = 0; p < k1NP; ++p) {
        const unsigned nA = (0u - neg[p]) & 0xFFFFu, nB = ((65535u * nA - neg[p]) >> 16) & 0xFFFFu;
        negw[p] += nA + nB;
        neg[p] = 0u;
      }
    }
    __syncwarp();
    if (lane == 0) mbar_arrive(&empty[s]);
    if (st + 1 < n_stage) continue;

    if constexpr (kF) {
      // ---- FULL epilogue for bin bl: node factors and IMAGCOHY already staged in shared
      // memory, 32-bit per-bin offsets, one store address per (row, metric) (the c = 1 pair is
      // +32 floats), band sums in this thread's own float4 slots, predicated stores
      const float4* nfs = nf_s + (bl % 3) * 2 * kTile;
      const uint32_t bin_off = (uint32_t)bl * (uint32_t)a.pair_stride;
      float4 fI[k1TR], fJ[k1TC];  // {M', rsqrt(psd) / s, rsqrt(psd), M' 2^-10}
#pragma unroll
      for (int r = 0; r < k1TR; ++r) fI[r] = nfs[ty + k1TY * r];
#pragma unroll
      for (int c = 0; c < k1TC; ++c) fJ[c] = nfs[kTile + tx + k1TX * c];
      if (IMAGIN) cp_async_wait_all();
      const float tau = IMAGIN ? a.imag_tau : 0.f;
      unsigned fl = 0;
      // kFast: an interior tile (every i < j < N) whose nodes all have non-zero spectra in
      // this bin (warp-uniform): no validity or dead-node predicates per pair
      auto pairs = [&](auto fast_tag) {
        constexpr bool kFast = decltype(fast_tag)::value;
#pragma unroll
        for (int h = 0; h < k1Quads; ++h) {  // pairs 4h .. 4h + 3 (k1RowsPerQuad rows)
          float bsum[5][4];
#pragma unroll
          for (int m = 0; m < 5; ++m) {
            const float4 q = band4[(m * k1Quads + h) * k1Threads + tid];
            bsum[m][0] = q.x; bsum[m][1] = q.y; bsum[m][2] = q.z; bsum[m][3] = q.w;
          }
#pragma unroll
          for (int rr = 0; rr < k1RowsPerQuad; ++rr) {
            const int r = k1RowsPerQuad * h + rr;
            const int i = iBase + ty + k1TY * r;
            // offset of the last column's pair (i, jBase + tx + k1TX (k1TC - 1)): exact whenever
            // any pair of the row is valid (the c = 0 offset wraps below 0 for i = 0, tx = 0);
            // column c stores k1TX (k1TC - 1 - c) floats before it
            const uint32_t ro = row_off32((uint32_t)i, (uint32_t)a.N) - (uint32_t)a.pair_base + bin_off +
                                (uint32_t)(jBase + tx + k1TX * (k1TC - 1));
            float* pb[5];
#pragma unroll
            for (int m = IMAGIN ? 1 : 0; m < 5; ++m) pb[m] = a.bins[m] + ro;
            const float phI = odd ? fI[r].w : 0.f;
            const float gMi = a.g * fI[r].x;
#pragma unroll
            for (int c = 0; c < k1TC; ++c) {
              const int p = r * k1TC + c;
              const int j = jBase + tx + k1TX * c;
              const bool valid = kFast || ((i < j) && (j < a.N));
              const bool dead = !kFast && fI[r].x * fJ[c].x == 0.f;
              const float tph = phI * fJ[c].w;
              const float rr2 = fI[r].z * fJ[c].z;
              const float s_abs = dead ? 0.f : sabs[p] - tph;
              float s_im, v0;
              bool flagged;
              if (IMAGIN) {
                const float im = imv_s[p * k1Threads + tid];
                s_im = (dead || (!kFast && rr2 == 0.f)) ? 0.f : im * rcp_approx(rr2);
                v0 = dead ? 0.f : im;
                flagged = valid && !dead && (mn[p] <= gMi * fJ[c].x || tau > 1e-4f * rr2 * s_abs);
              } else {
                s_im = dead ? 0.f : (lo_of(sim[p]) + hi_of(sim[p])) - tph;
                v0 = s_im * rr2;
                flagged = valid && !dead && mn[p] <= gMi * fJ[c].x;
              }
              fl |= (unsigned)flagged << p;
              const unsigned nA = (0u - neg[p]) & 0xFFFFu, nB = ((65535u * nA - neg[p]) >> 16) & 0xFFFFu;
              const int pli_sum = dead ? 0 : a.K - 2 * (int)(nA + nB);
              const float pli = fabsf((float)pli_sum) * invK;
              const float w = s_abs > 0.f ? fminf(fabsf(s_im) * rcp_approx(s_abs), 1.f) : 0.f;
              const float v[5] = {v0, pli, pli * pli * uspA - uspB, w, w * w};
              const bool ok = valid && !flagged;
#pragma unroll
              for (int m = 0; m < 5; ++m) {
                if (m > 0 || !IMAGIN) {
                  if (ok) __stcs(pb[m] - k1TX * (k1TC - 1 - c), v[m]);  // streaming: keep the operands in L2
                }
                bsum[m][rr * k1TC + c] += ok ? v[m] : 0.f;
              }
              sim[p] = 0ull;
              sabs[p] = 0.f;
              mn[p] = 3.0e38f;
              neg[p] = 0u;
            }
          }
#pragma unroll
          for (int m = 0; m < 5; ++m)
            band4[(m * k1Quads + h) * k1Threads + tid] = make_float4(bsum[m][0], bsum[m][1], bsum[m][2], bsum[m][3]);
        }
      };
      bool fast = interior;
#pragma unroll
      for (int r = 0; r < k1TR; ++r) fast = fast && fI[r].x != 0.f;
#pragma unroll
      for (int c = 0; c < k1TC; ++c) fast = fast && fJ[c].x != 0.f;
      if (__all_sync(0xffffffffu, fast))
        pairs(std::true_type{});
      else
        pairs(std::false_type{});
      if (__any_sync(0xffffffffu, fl)) guard_push(a.flags, a.recs, a.counters, a.flag_cap, fl, iBase, jBase, ty, tx, lane, bl);
      continue;
    }

    // ---- epilogue for bin bl ----
    // per-node factors first (6 nodes per thread), then ~30 instructions per pair
    const int b = a.bin_lo + bl;
    const bool real_bin = (b == a.real0) || (b == a.real1);
    float Mi[k1TR], gMi[k1TR], rPi[k1TR], phI[k1TR];
    float Mj[k1TC], rPj[k1TC], phJ[k1TC];
#pragma unroll
    for (int r = 0; r < k1TR; ++r) {
      const int i = iBase + ty + k1TY * r;
      const float m = (i < a.N && !real_bin) ? a.mag[(int64_t)bl * a.N + i] : 0.f;
      const float pw = i < a.N ? a.psd[(int64_t)bl * a.N + i] : 0.f;
      Mi[r] = m;
      gMi[r] = a.g * m;
      rPi[r] = pw > 0.f ? rsqrt_approx(pw) : 0.f;
      phI[r] = odd ? m * k1Phantom : 0.f;
    }
#pragma unroll
    for (int c = 0; c < k1TC; ++c) {
      const int j = jBase + tx + k1TX * c;
      const float m = (j < a.N && !real_bin) ? a.mag[(int64_t)bl * a.N + j] : 0.f;
      const float pw = j < a.N ? a.psd[(int64_t)bl * a.N + j] : 0.f;
      Mj[c] = m;
      rPj[c] = pw > 0.f ? rsqrt_approx(pw) : 0.f;
      phJ[c] = m * k1Phantom;
    }
    const int64_t bin_off = (int64_t)bl * a.pair_stride;
    unsigned fl = 0;  // exact-sign guard: this thread's entries the fp64 fallback writes
    float imv[IMAGIN ? k1NP : 1];
    if (IMAGIN) {  // issued with the node-factor loads above, so their latencies overlap
#pragma unroll
      for (int r = 0; r < k1TR; ++r) {
        const int i = iBase + ty + k1TY * r;
        const int64_t rowoff = (int64_t)i * (a.N - 1) - (int64_t)i * (i - 1) / 2 - i - 1 - a.pair_base + bin_off;
#pragma unroll
        for (int c = 0; c < k1TC; ++c) {
          const int j = jBase + tx + k1TX * c;
          imv[r * k1TC + c] = (i < j && j < a.N) ? __ldcs(&a.imag_in[rowoff + j]) : 0.f;
        }
      }
    }
#pragma unroll
    for (int r = 0; r < k1TR; ++r) {
      const int li = ty + k1TY * r, i = iBase + li;
      const int64_t rowoff = (int64_t)i * (a.N - 1) - (int64_t)i * (i - 1) / 2 - i - 1 - a.pair_base + bin_off;
#pragma unroll
      for (int c = 0; c < k1TC; ++c) {
        const int p = r * k1TC + c;
        const int lj = tx + k1TX * c, j = jBase + lj;
        const bool valid = (i < j) && (j < a.N);
        // dead: a node with a zero spectrum in this bin (or DC / Nyquist): all Im are 0
        const bool dead = Mi[r] * Mj[c] == 0.f;
        const float tph = phI[r] * phJ[c];  // odd-K phantom trial (0 when K is even)
        float s_im;
        bool flagged;
        if (IMAGIN) {
          const float rr = rPi[r] * rPj[c];
          s_im = (dead || rr == 0.f) ? 0.f : imv[p] * rcp_approx(rr);
          // re-folded in fp64 (IMAGCOHY included): a sign within the fp32 guard (this also
          // catches the reference's exact zeros: every trial's |Im| is below the guard), or a
          // sum |Im| too small for WPLI's numerator error tau / (rPi rPj)
          flagged = valid && !dead && (mn[p] <= gMi[r] * Mj[c] || a.imag_tau > 1e-4f * rr * (sabs[p] - tph));
        } else {
          s_im = dead ? 0.f : (lo_of(sim[p]) + hi_of(sim[p])) - tph;
          flagged = valid && !dead && mn[p] <= gMi[r] * Mj[c];
        }
        fl |= (unsigned)flagged << p;
        const float s_abs = dead ? 0.f : sabs[p] - tph;
        const unsigned nA = (0u - neg[p]) & 0xFFFFu, nB = ((65535u * nA - neg[p]) >> 16) & 0xFFFFu;
        const int n_neg = WIDE ? (int)negw[p] : L == 1 ? (int)(nA + nB) : (int)neg[p];
        const int pli_sum = dead ? 0 : a.K - 2 * n_neg;
        float v[5];
        v[0] = s_im * rPi[r] * rPj[c];
        const float pli = fabsf((float)pli_sum) * invK;
        v[1] = pli;
        v[2] = pli * pli * uspA - uspB;
        const float w = s_abs > 0.f ? fminf(fabsf(s_im) * rcp_approx(s_abs), 1.f) : 0.f;
        v[3] = w;
        v[4] = w * w;
        if (PLVK && valid) {  // PLV is continuous: written even for guard-flagged entries
          // the odd-K phantom contributed the unit phasor (0, 1) to the PLV sums
          const float pr = lo_of(pvr[p]) + hi_of(pvr[p]);
          const float pim = lo_of(pvi[p]) + hi_of(pvi[p]) - (odd ? 1.f : 0.f);
          // a real bin (Nyquist) still has phases 0 / pi: only a zero spectrum makes PLV 0
          const bool dead_plv = rPi[r] * rPj[c] == 0.f;
          const float plv = dead_plv ? 0.f : sqrt_approx(pr * pr + pim * pim) * invK;
          if (bin_mask & 32u) __stcs(&a.plv_bins[rowoff + j], plv);  // streaming: keep the operands in L2
          if (band_mask & 32u) band_s[(5 * kTile + li) * kTile + lj] += plv;
          pvr[p] = pvi[p] = 0ull;
        }
        if (valid && !flagged) {
          float* bs = band_s + li * kTile + lj;
#pragma unroll
          for (int m = 0; m < 5; ++m) {
            if (bin_mask & (1u << m)) {
              if (FULL)  // host-checked: every per-bin index < 2^32 -> one IMAD.WIDE.U32 per address
                __stcs(&a.bins[m][(uint32_t)(rowoff + j)], v[m]);
              else
                __stcs(&a.bins[m][rowoff + j], v[m]);
            }
            if (band_mask & (1u << m)) bs[m * kTile * kTile] += v[m];
          }
        }
        sim[p] = 0ull;
        sabs[p] = 0.f;
        mn[p] = 3.0e38f;
        neg[p] = 0u;
        if (WIDE) negw[p] = 0u;
      }
    }
    if (__any_sync(0xffffffffu, fl)) guard_push(a.flags, a.recs, a.counters, a.flag_cap, fl, iBase, jBase, ty, tx, lane, bl);
  }

  if (kF) {
    // FULL: each thread writes its own band sums (no barrier); per (row, column half)
    // a warp covers 32 contiguous pair columns
    const float inv = 1.f / (float)a.nbb;
#pragma unroll
    for (int r = 0; r < k1TR; ++r) {
      const int i = iBase + ty + k1TY * r;
      const int64_t rowoff = (int64_t)i * (a.N - 1) - (int64_t)i * (i - 1) / 2 - i - 1 - a.pair_base;
#pragma unroll
      for (int m = 0; m < 5; ++m) {
        const float4 q = band4[(m * k1Quads + r / k1RowsPerQuad) * k1Threads + tid];
#pragma unroll
        for (int c = 0; c < k1TC; ++c) {
          const int j = jBase + tx + k1TX * c;
          const int e = (r % k1RowsPerQuad) * k1TC + c;
          const float v = (e == 0 ? q.x : e == 1 ? q.y : e == 2 ? q.z : q.w) * inv;
          if (i < j && j < a.N) {
            if (a.nbc > 1)
              atomicAdd(a.band[m] + rowoff + j, v);  // bins split over CTAs: band zeroed by the host
            else
              __stcs(a.band[m] + rowoff + j, v);
          }
        }
      }
    }
  } else if (band_mask) {
    // band write-out by rows: the compute warps' band slots are complete after one
    // named barrier (the producer warp has left); warp w writes rows w, w + 16, ...
    // of every requested metric, lanes over 64 contiguous pair columns.
    asm volatile("bar.sync 1, %0;" ::"n"(k1Threads) : "memory");
    const float inv = 1.f / (float)a.nbb;
    for (int li = warp; li < kTile; li += k1Warps) {
      const int i = iBase + li;
      if (i >= a.N) break;
      const int64_t rowoff = (int64_t)i * (a.N - 1) - (int64_t)i * (i - 1) / 2 - i - 1 - a.pair_base;
#pragma unroll
      for (int m = 0; m < NM; ++m) {
        if (!(band_mask & (1u << m))) continue;
        float* dst = (m < 5 ? a.band[m] : a.plv_band) + rowoff + jBase;
        const float* bs = band_s + (m * kTile + li) * kTile;
#pragma unroll
        for (int c = 0; c < 2; ++c) {
          const int lj = lane + 32 * c, j = jBase + lj;
          if (i < j && j < a.N) {
            const float v = bs[lj] * inv;
            if (a.nbc > 1)
              atomicAdd(dst + lj, v);  // bins split over CTAs: band zeroed by the host
            else
              __stcs(dst + lj, v);
          }
        }
      }
    }
  }
}

bool launch_lag1(const float4* PkI, const float4* PkJ, int N, int N64, int K, int Kp, int bin_lo, int nbb,
                 const float* psd, const float* mag, int real0, int real1, int nt, int row_begin,
                 int64_t pair_base, int64_t pair_stride, float* const* bins, float* const* band, float g,
                 int4* flags, int4* recs, int* counters, int flag_cap, int64_t n_tiles, int nbc,
                 int L, float* plv_bins, float* plv_band, const float* imag_in, float imag_tau, const float4* nf,
                 cudaStream_t st) {
  EncodeTiledFn enc = get_encode();
  if (!enc) {
    cs_set_error("cuTensorMapEncodeTiled unavailable");
    return false;
  }
  CUtensorMap mI, mJ;
  cuuint64_t dims[2] = {(cuuint64_t)N64 * 4, (cuuint64_t)nbb * Kp * L};
  cuuint64_t strides[1] = {(cuuint64_t)N64 * 16};
  cuuint32_t box[2] = {(cuuint32_t)kTile * 4, (cuuint32_t)((k1Rows / L) * L)};
  cuuint32_t estr[2] = {1, 1};
  CUresult r = enc(&mI, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 2, (void*)PkI, dims, strides, box, estr,
                   CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                   CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  if (r == CUDA_SUCCESS)
    r = enc(&mJ, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 2, (void*)PkJ, dims, strides, box, estr,
            CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
            CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  if (r != CUDA_SUCCESS) {
    cs_set_error("cuTensorMapEncodeTiled failed (%d)", (int)r);
    return false;
  }
  Lag1Args a{};
  a.N = N; a.N64 = N64; a.K = K; a.Kp = Kp; a.bin_lo = bin_lo; a.nbb = nbb;
  a.nbc = nbc;
  a.bpc = (nbb + nbc - 1) / nbc;
  a.psd = psd; a.mag = mag; a.real0 = real0; a.real1 = real1; a.nt = nt; a.row_begin = row_begin;
  a.pair_base = pair_base; a.pair_stride = pair_stride;
  for (int m = 0; m < 5; ++m) {
    a.bins[m] = bins[m];
    a.band[m] = band[m];
  }
  a.g = g; a.flags = flags; a.recs = recs; a.counters = counters; a.flag_cap = flag_cap;
  a.plv_bins = plv_bins;
  a.plv_band = plv_band;
  a.imag_in = imag_in;
  a.imag_tau = imag_tau;
  a.nf = nf;
  const size_t smem = (size_t)2 * k1Stages * k1StageF4 * 16 + 6 * kTile * kTile * 4 + 3 * 2 * kTile * 16 +
                     2 * k1Stages * 8;
  const unsigned grid = (unsigned)(n_tiles * nbc);
  const bool plvk = plv_bins || plv_band;
#define CS_LAG1S(LL, PV, SS)                                                                           \
  do {                                                                                                   \
    CS_SMEM_ONCE((k_pairs_lag1<LL, PV, SS>), smem);                                                     \
    k_pairs_lag1<LL, PV, SS><<<grid, LL == 1 ? k1ThreadsP : k1Threads, smem, st>>>(mI, mJ, a);    \
  } while (0)
#define CS_LAG1(LL, PV)                                                                              \
  do {                                                                                                   \
    CS_SMEM_ONCE((k_pairs_lag1<LL, PV>), smem);                                                         \
    k_pairs_lag1<LL, PV><<<grid, LL == 1 ? k1ThreadsP : k1Threads, smem, st>>>(mI, mJ, a);     \
  } while (0)
  if (imag_in) {  // IMAGCOHY from the tensor-core kernel (run_lag_family checked the shape)
    CS_SMEM_ONCE((k_pairs_lag1<1, false, kStSign | kStAbs, true, false, true>), smem);
    k_pairs_lag1<1, false, kStSign | kStAbs, true, false, true><<<grid, k1ThreadsP, smem, st>>>(mI, mJ, a);
  } else if (L == 1 && Kp >= 65536) {  // a 16-bit sign-count field could wrap: per-stage decode
    CS_SMEM_ONCE((k_pairs_lag1<1, false, kStAll, false, true>), smem);
    k_pairs_lag1<1, false, kStAll, false, true><<<grid, k1ThreadsP, smem, st>>>(mI, mJ, a);
  } else if (L == 1) {
    // statistics the requested outputs need (bins / band pointers: IMAG, PLI, USPLI, WPLI, DSWPLI)
    auto want = [&](int m) { return bins[m] || band[m]; };
    const unsigned need = ((want(1) || want(2)) ? kStSign : 0u) | ((want(0) || want(3) || want(4)) ? kStSum : 0u) |
                          ((want(3) || want(4)) ? kStAbs : 0u);
    switch (need) {
      case kStSign: CS_LAG1S(1, false, kStSign); break;
      case kStSum: CS_LAG1S(1, false, kStSum); break;
      case kStSign | kStSum: CS_LAG1S(1, false, kStSign | kStSum); break;
      case kStSum | kStAbs: CS_LAG1S(1, false, kStSum | kStAbs); break;
      default: {
        bool full = (uint64_t)nbb * (uint64_t)pair_stride + kTile < (1ull << 32);  // 32-bit per-bin offsets
        for (int m = 0; m < 5; ++m) full = full && bins[m] && band[m];
        if (full) {
          CS_SMEM_ONCE((k_pairs_lag1<1, false, kStAll, true>), smem);
          k_pairs_lag1<1, false, kStAll, true><<<grid, k1ThreadsP, smem, st>>>(mI, mJ, a);
        } else {
          CS_LAG1(1, false);
        }
        break;
      }
    }
  } else if (L == 2) {
    if (plvk) CS_LAG1(2, true);
    else CS_LAG1(2, false);
  } else if (L == 3) {
    if (plvk) CS_LAG1(3, true);
    else CS_LAG1(3, false);
  } else {
    if (plvk) CS_LAG1(4, true);
    else CS_LAG1(4, false);
  }
#undef CS_LAG1
#undef CS_LAG1S
  return true;
}

}  // namespace cs
