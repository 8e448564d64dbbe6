// K2: the coherency family (COH, COHY, PLV; IMAGCOHY from D_im) as complex-as-real
// tcgen05 tensor-core contractions over trials, per frequency bin, on 128 x 64 node tiles
// (one CTA) or 256 x 64 tiles (a CTA pair, cta_group::2) of the upper-triangular pair space.
//
// Reference: spectral.py:204-241 (CSD = X_i conj X_j and unit phasor sums),
// metrics.py:32-56 (cohy/coh/plv finalisers), metrics.py:115-134 (band mean).
//
// Per bin b and tile (I, J) the kernel accumulates, in TMEM (fp32),
//   D_re = sum_k Re X_i Re X_j + Im X_i Im X_j      D_im = sum_k Im X_i Re X_j - Re X_i Im X_j
// for X (pass 0: cross-spectra) and for the unit phasors U = X/|X| (pass 1: PLV).
// Operands are fp16 hi/lo splits (x = h + l, |x| <= 1 after a per-node-bin power
// of two) so each real product is h*h + h*l + l*h: ~22-bit products on the f16
// tensor path (the plain fp16/bf16/tf32 product misses the 1e-4 COH tolerance;
// SURVEY.md section 7, hard part 2).  Single CTA: the subtraction in D_im uses the
// instruction descriptor's A-negate bit; CTA pair: the peer's B half is the -Im plane.
//
// Pipeline (warp specialised, persistent CTAs / CTA pairs, all bins and both passes of a
// tile per work unit):
//   warp 0: TMA producer (cp.async.bulk.tensor, 64B swizzle) into a 3-stage ring
//   warp 1: tcgen05.mma issuer (pair: the leader CTA's), tcgen05.commit to mbarriers
//   warp 2: TMEM allocator (512 columns: up to three 128-column accumulator regions
//           round-robin over the (bin, pass) sequence, band-mean accumulators)
//   warps 4-19: epilogue (tcgen05.ld/st 32x32b.x8; TMEM lane quadrant = warp % 4,
//           four warps per quadrant split the 64 columns; 112 registers each after
//           setmaxnreg), per-bin values leave through a shared-memory transpose buffer
//           as coalesced row stores; band means accumulate in TMEM across bins.
// The (bin, pass) units use rotating TMEM regions, so the epilogue of one overlaps the
// MMAs of the next ones.
#include <cuda.h>
#include <cuda_fp16.h>

#include <cstdlib>
#include <vector>

#include "common.cuh"
#include "ptx.cuh"

namespace cs {

constexpr int kTcTile = 128;          // i rows per tile (UMMA M)
constexpr int kTcTileJ = 64;          // j columns per tile (UMMA N)
constexpr int kTcChunk = 32;          // trials per stage (64-byte fp16 rows)
constexpr int kTcStages = 3;
constexpr int kTcPlaneA = kTcTile * kTcChunk * 2;       // 8 KB
constexpr int kTcPlaneB = kTcTileJ * kTcChunk * 2;      // 4 KB
constexpr int kTcStageBytes = 4 * kTcPlaneA + 4 * kTcPlaneB;  // 48 KB
constexpr int kTcXStride = kTcTileJ + 1;                // transpose buffer row stride (float2)
constexpr int kTcEpiWarps = 16;   // 4 per TMEM lane quadrant
constexpr int kTcThreads = (4 + kTcEpiWarps) * 32;  // warps 0-3: TMA, MMA, TMEM alloc, spare; 4-19: epilogue
constexpr int kTcColsPerWarp = kTcTileJ / (kTcEpiWarps / 4);  // TMEM-phase columns per epilogue warp (16)
constexpr int kTcRowsPerWarp = kTcTile / kTcEpiWarps;         // store-phase rows per epilogue warp (8)
// TMEM columns: [0,128) pass-0 accumulators (re | im), [128,256) pass-1,
// [256,512) band sums: COH, PLV, COHY re, COHY im (64 each)
constexpr int kTmBand = 256;

#ifdef CS_TC_ABLATION
#define TC_ABL(bit) (a.dbg & (bit))
#else
#define TC_ABL(bit) 0
#endif

struct TcArgs {
  int N, K, K_pad, nbb;
  int i_lo, i_hi;            // row range [i_lo, i_hi) of pairs computed (shard)
  int tile_row0, n_tiles;    // first 128-row tile and number of tiles in the launch
  const int2* tiles;         // (I, J) per tile, L2-friendly grouped order
  int bpc, nbc;              // bins per CTA and bin chunks per tile (small pair spaces split bins)
  int nt;                    // 64-node column tiles over N
  const float* psd;          // [nbb][N] plan-scaled sum_k |X|^2
  const float* nscale;       // [nbb][N] per-node-bin power of two used for the fp16 split
  float invK;
  int64_t pair_base, pair_stride;
  float* coh_bins;  float* coh_band;
  float2* cohy_bins; float2* cohy_band;
  float* plv_bins;  float* plv_band;
  float* imag_bins; float* imag_band;   // IMAGCOHY from D_im (the phase-lag kernel then reads it for WPLI)
  int do_x, do_u;
  // IMAGCOHY produced here (no sign-based metric asked): entries with |IMAG| < imag_tau
  // (above the tensor-core error bound) go to the fp64 fallback list, so values that
  // are exactly 0 in the reference (zero-lag copies) come out exact, not ~1e-9
  int4* flags;
  int* counters;
  int flag_cap;
  float imag_tau;
  int dbg;   // ablation bits (builds with -DCS_TC_ABLATION only): 1 per-bin stores, 2 TMEM-phase
             // math, 4 band phase, 8 MMAs, 16 TMA loads are skipped (timing experiments).  With
             // CTA pairs, 16 takes the peer's loads out of the leader's stage barrier, so with
             // 1 | 8 as well the leader can lap the peer's producer by two phases (a hang the
             // watchdog traps); with the loads on, the peer's bytes keep the pair in step.
};

// 16 consecutive fp32 columns of this thread's TMEM lane
__device__ __forceinline__ void tmem_ld16(uint32_t taddr, float* v) {
  uint32_t r[16];
  asm volatile(
      "tcgen05.ld.sync.aligned.32x32b.x16.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15}, [%16];"
      : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]), "=r"(r[7]),
        "=r"(r[8]), "=r"(r[9]), "=r"(r[10]), "=r"(r[11]), "=r"(r[12]), "=r"(r[13]), "=r"(r[14]), "=r"(r[15])
      : "r"(taddr));
  asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
#pragma unroll
  for (int q = 0; q < 16; ++q) v[q] = __uint_as_float(r[q]);
}
// two 16-column loads under one tcgen05.wait::ld
__device__ __forceinline__ void tmem_ld16x2(uint32_t ta, float* v, uint32_t tb, float* w) {
  uint32_t r[16], s[16];
  asm volatile(
      "tcgen05.ld.sync.aligned.32x32b.x16.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15}, [%16];"
      : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]), "=r"(r[7]),
        "=r"(r[8]), "=r"(r[9]), "=r"(r[10]), "=r"(r[11]), "=r"(r[12]), "=r"(r[13]), "=r"(r[14]), "=r"(r[15])
      : "r"(ta));
  asm volatile(
      "tcgen05.ld.sync.aligned.32x32b.x16.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15}, [%16];"
      : "=r"(s[0]), "=r"(s[1]), "=r"(s[2]), "=r"(s[3]), "=r"(s[4]), "=r"(s[5]), "=r"(s[6]), "=r"(s[7]),
        "=r"(s[8]), "=r"(s[9]), "=r"(s[10]), "=r"(s[11]), "=r"(s[12]), "=r"(s[13]), "=r"(s[14]), "=r"(s[15])
      : "r"(tb));
  asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
#pragma unroll
  for (int q = 0; q < 16; ++q) {
    v[q] = __uint_as_float(r[q]);
    w[q] = __uint_as_float(s[q]);
  }
}

// K-major operand tile [128 rows x 32 fp16] written by TMA with SWIZZLE_64B:
// 64-byte rows, 8-row core groups 512 B apart (SBO), LBO unused, descriptor version 1.
__device__ __forceinline__ uint64_t umma_desc_sw64(uint32_t smem_addr) {
  uint64_t d = 0;
  d |= (uint64_t)((smem_addr >> 4) & 0x3FFF);        // start address
  d |= (uint64_t)1 << 16;                             // LBO (ignored for swizzled K-major)
  d |= (uint64_t)(512 >> 4) << 32;                    // SBO
  d |= (uint64_t)1 << 46;                             // version (Blackwell)
  d |= (uint64_t)4 << 61;                             // SWIZZLE_64B
  return d;
}
// kind::f16 instruction descriptor: fp16 x fp16 -> fp32, K-major A and B, M x N
__host__ __device__ constexpr uint32_t idesc_f16(bool neg_a, int M = kTcTile, int N = kTcTileJ) {
  return (1u << 4)                     // D format f32
         | (0u << 7) | (0u << 10)      // A, B format f16
         | ((neg_a ? 1u : 0u) << 13)   // negate A
         | ((uint32_t)(N >> 3) << 17)  // N >> 3
         | ((uint32_t)(M >> 4) << 24); // M >> 4
}

// ---------------------------------------------------------------- the kernel
// Tile (I, J): rows i in [128 I, 128 I + 128), columns j in [64 J, 64 J + 64),
// J >= 2 I (upper triangle).  decode over the row range starting at tile_row0.
__device__ __forceinline__ void decode_tc_tile(int64_t t, int nt64, int row0, int& I, int& J) {
  int r = row0;
  int64_t left = t;
  while (left >= nt64 - 2 * r) {
    left -= nt64 - 2 * r;
    ++r;
  }
  I = r;
  J = 2 * r + (int)left;
}

__device__ __forceinline__ void tmem_st16(uint32_t taddr, const float* v) {
  asm volatile(
      "tcgen05.st.sync.aligned.32x32b.x16.b32 [%0], {%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,%16};"
      ::"r"(taddr), "r"(__float_as_uint(v[0])), "r"(__float_as_uint(v[1])), "r"(__float_as_uint(v[2])),
      "r"(__float_as_uint(v[3])), "r"(__float_as_uint(v[4])), "r"(__float_as_uint(v[5])),
      "r"(__float_as_uint(v[6])), "r"(__float_as_uint(v[7])), "r"(__float_as_uint(v[8])),
      "r"(__float_as_uint(v[9])), "r"(__float_as_uint(v[10])), "r"(__float_as_uint(v[11])),
      "r"(__float_as_uint(v[12])), "r"(__float_as_uint(v[13])), "r"(__float_as_uint(v[14])),
      "r"(__float_as_uint(v[15])));
}
__device__ __forceinline__ void epi_bar() {  // the epilogue warps only
  asm volatile("bar.sync 1, %0;" ::"n"(kTcEpiWarps * 32) : "memory");
}

// PAIR: a CTA pair (cluster of 2, cta_group::2) works on a 256 x 64 tile: CTA r holds
// rows [256 I + 128 r, +128) as A and one half of the stacked B' = [B1 | B2] (N = 128), so
// one M = 256 x N = 128 MMA gives both CTAs' D_re (columns 0-63) and D_im (64-127):
//   A = Re_i^a : B' = [Re_j^b | -Im_j^b]     A = Im_i^a : B' = [Im_j^b | Re_j^b]
// (rank 0's B slots hold re_h re_l im_h im_l, rank 1's -im_h -im_l re_h re_l).  Six MMAs
// per 16-trial step instead of 2 x 12 single-CTA 128 x 64 MMAs, each SM reading the same
// 6 KB of operands per MMA for twice the products (the single-CTA N = 64 MMA is bound by
// the shared-memory read port, 48 of 32 cycles: tools/ubench/mma_rate.cu).  The leader's
// MMA warp issues; both CTAs' TMA loads complete on the leader's stage barrier; commits
// multicast to both CTAs; both CTAs' epilogue warps release a TMEM region on the leader.
template <bool PAIR>
__global__ void __launch_bounds__(kTcThreads, 1)
k_pairs_tc(const __grid_constant__ CUtensorMap mapA, const __grid_constant__ CUtensorMap mapB, const TcArgs a) {
  // dynamic shared memory starts at the (1024-aligned) base of the CTA's window: no
  // static __shared__ in this kernel.  Indexing the extern array directly keeps every
  // epilogue access in the shared state space (LDS/STS, not generic LD/ST).
  extern __shared__ __align__(1024) unsigned char smem[];
  float2* xbuf = (float2*)(smem + kTcStages * kTcStageBytes);          // [128][65] transpose buffer
  float* colfac = (float*)(xbuf + kTcTile * kTcXStride);               // [64] psd_j * s_j^2
  int64_t* rowoff_s = (int64_t*)(colfac + kTcTileJ);                   // [128] output row offsets
  uint64_t* full = (uint64_t*)(rowoff_s + kTcTile);
  uint64_t* empty = full + kTcStages;
  uint64_t* tfull = empty + kTcStages;   // [3] per accumulator region
  uint64_t* tempty = tfull + 3;          // [3]
  uint32_t* tmem_slot = (uint32_t*)(tempty + 3);

  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  // persistent CTAs (PAIR: CTA pairs): work unit u = (tile u / nbc, bin chunk u % nbc),
  // strided by the grid; the smem ring and TMEM phases carry over between units, so the
  // next unit's loads and MMAs overlap this unit's epilogue
  const int n_units = a.n_tiles * a.nbc;
  const uint32_t rank = PAIR ? cluster_ctarank() : 0u;
  const int u0 = PAIR ? (int)(blockIdx.x >> 1) : (int)blockIdx.x;
  const int ustep = PAIR ? (int)(gridDim.x >> 1) : (int)gridDim.x;
  constexpr int kUnitRows = PAIR ? 2 * kTcTile : kTcTile;  // tile rows per unit

  if (threadIdx.x == 0) {
    if (smem_u32(smem) & 1023) __trap();  // swizzled TMA/UMMA tiles need 1024-byte alignment
    for (int s = 0; s < kTcStages; ++s) {
      mbar_init(&full[s], 1);
      mbar_init(&empty[s], 1);
    }
    for (int r = 0; r < 3; ++r) {
      mbar_init(&tfull[r], 1);
      mbar_init(&tempty[r], (PAIR ? 2 : 1) * kTcEpiWarps);  // one arrive per epilogue warp (of both CTAs)
    }
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  if (warp == 2) {
    if (PAIR) {
      asm volatile("tcgen05.alloc.cta_group::2.sync.aligned.shared::cta.b32 [%0], 512;" ::"r"(smem_u32(tmem_slot)));
      asm volatile("tcgen05.relinquish_alloc_permit.cta_group::2.sync.aligned;");
    } else {
      asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 512;" ::"r"(smem_u32(tmem_slot)));
      asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
    }
  }
  tc_fence_before();
  if (PAIR)
    cluster_sync();  // the peer signals the leader's barriers only after they exist
  else
    __syncthreads();
  tc_fence_after();
  const uint32_t tmem = *tmem_slot;

  const int n_chunk = (a.K_pad + kTcChunk - 1) / kTcChunk;
  const int npass = a.do_x + a.do_u;
  const int pass0 = a.do_x ? 0 : 1;
  // accumulator regions of 128 TMEM columns, used round-robin by the (bin, pass) sequence
  // so the MMAs can run ahead of the epilogue: [0,128), [128,256) and, when the band sums
  // need only [256,384) (no COHY / IMAGCOHY band), a third at [384,512)
  const int nreg = (a.cohy_band || a.imag_band) ? 2 : 3;

  // register budgets: warps 0-3 (TMA, MMA, TMEM allocator, spare) drop to 32, the
  // epilogue warps rise to 112 (launch pool 640 x 96 = 128 x 32 + 512 x 112)
  if (warp < 4) {
  asm volatile("setmaxnreg.dec.sync.aligned.u32 32;");
  if (warp == 0) {
    // ------------------------------------------------------------ TMA producer
    if (lane == 0) {
      int stage = 0;
      uint32_t phase = 0;
      // PAIR: every load completes on the leader's stage barrier (which expects both CTAs' bytes)
      const uint32_t full0 = PAIR ? mapa_u32(smem_u32(full), 0) : 0u;
      constexpr int bplane_peer[4] = {4, 5, 0, 1};  // rank 1's B slots: -im_h, -im_l, re_h, re_l
      for (int u = u0; u < n_units; u += ustep) {
        const int2 tij = a.tiles[u / a.nbc];
        const int bl0 = (u % a.nbc) * a.bpc, bl1 = min(a.nbb, bl0 + a.bpc);
        const int iBase = tij.x * kUnitRows + (int)rank * kTcTile, jBase = tij.y * kTcTileJ;
      for (int bl = bl0; bl < bl1; ++bl)
        for (int ps = 0; ps < npass; ++ps) {
          const int pass = pass0 + ps;
          for (int c = 0; c < n_chunk; ++c) {
            mbar_wait(&empty[stage], phase ^ 1);
            unsigned char* st = smem + stage * kTcStageBytes;
            if (TC_ABL(16)) {
              mbar_arrive(&full[stage]);
              if (++stage == kTcStages) { stage = 0; phase ^= 1; }
              continue;
            }
            if (!PAIR) {
              mbar_expect_tx(&full[stage], kTcStageBytes);
              for (int pl = 0; pl < 4; ++pl) {
                const int z = (bl * 2 + pass) * kTcPlanes + pl;
                tma_load_3d(st + pl * kTcPlaneA, &mapA, &full[stage], c * kTcChunk, iBase, z);
                tma_load_3d(st + 4 * kTcPlaneA + pl * kTcPlaneB, &mapB, &full[stage], c * kTcChunk, jBase, z);
              }
            } else {
              if (rank == 0) mbar_expect_tx(&full[stage], 2 * kTcStageBytes);
              const uint32_t fb = full0 + (uint32_t)stage * 8u;
              for (int pl = 0; pl < 4; ++pl) {
                const int z = (bl * 2 + pass) * kTcPlanes;
                tma_load_3d_cg2(st + pl * kTcPlaneA, &mapA, fb, c * kTcChunk, iBase, z + pl);
                tma_load_3d_cg2(st + 4 * kTcPlaneA + pl * kTcPlaneB, &mapB, fb, c * kTcChunk, jBase,
                                z + (rank ? bplane_peer[pl] : pl));
              }
            }
            if (++stage == kTcStages) { stage = 0; phase ^= 1; }
          }
        }
      }
      // drain: every stage's last use released, so no MMA commit (PAIR: multicast from the
      // leader) can still be in flight to this CTA's barriers when it exits
      for (int i = 0; i < kTcStages; ++i) {
        mbar_wait(&empty[stage], phase ^ 1);
        if (++stage == kTcStages) { stage = 0; phase ^= 1; }
      }
    }
  } else if (warp == 1) {
    // ------------------------------------------------------------ MMA issuer
    // the whole warp runs the (uniform) loop so descriptors stay in uniform registers;
    // one elected lane issues each tcgen05.mma / commit
    // (A plane, B plane) for D_re then D_im; planes: 0 re_h, 1 re_l, 2 im_h, 3 im_l;
    // the first three D_im products are -(Re_i Im_j) via the A-negate bit
    // (D_im: the -Re_i Im_j products first, the order of the CTA-pair kernel's N = 128 MMAs)
    constexpr int prod_a[12] = {0, 0, 1, 2, 2, 3, 0, 0, 1, 2, 2, 3};
    constexpr int prod_b[12] = {0, 1, 0, 2, 3, 2, 2, 3, 2, 0, 1, 0};
    constexpr uint32_t id_pos = idesc_f16(false), id_neg = idesc_f16(true);
    // PAIR: (A plane, B slot) per MMA: A = re_h re_h re_l against B' = [Re | -Im] (slots 0, 1),
    // A = im_h im_h im_l against B' = [Im | Re] (slots 2, 3); all into one N = 128 D
    constexpr int pa2[6] = {0, 0, 1, 2, 2, 3};
    constexpr int pb2[6] = {0, 1, 0, 2, 3, 2};
    constexpr uint32_t id_pair = idesc_f16(false, 2 * kTcTile, 2 * kTcTileJ);
    int stage = 0;
    uint32_t phase = 0;
    uint32_t tuse = 0;  // bit r: phase of TMEM region r
    int seq = 0;        // region of the next (bin, pass): round-robin over nreg
    const uint64_t desc0 = umma_desc_sw64(smem_u32(smem));
    if (PAIR && rank != 0) {
      // the peer's MMA warp idles: the leader issues for both CTAs
    } else
    for (int u = u0; u < n_units; u += ustep) {
      const int bl0 = (u % a.nbc) * a.bpc, bl1 = min(a.nbb, bl0 + a.bpc);
      for (int bl = bl0; bl < bl1; ++bl)
        for (int ps = 0; ps < npass; ++ps) {
          const int reg = seq;
          seq = seq + 1 == nreg ? 0 : seq + 1;
          mbar_wait(&tempty[reg], ((tuse >> reg) & 1) ^ 1);
          tuse ^= 1u << reg;
          tc_fence_after();
          const uint32_t d_re = tmem + (reg == 2 ? 384 : reg * 128), d_im = d_re + 64;
          for (int c = 0; c < n_chunk; ++c) {
            mbar_wait(&full[stage], phase);
            tc_fence_after();
            const uint64_t sd = desc0 + (uint64_t)((stage * kTcStageBytes) >> 4);
            const int n_steps = TC_ABL(8) ? 0 : min(kTcChunk / 16, (a.K_pad - c * kTcChunk) / 16);
#pragma unroll
            for (int s = 0; s < kTcChunk / 16; ++s) {
                if (PAIR && s < n_steps) {
#pragma unroll
                for (int q = 0; q < 6; ++q) {
                  const uint64_t ad = sd + (uint64_t)((pa2[q] * kTcPlaneA + s * 32) >> 4);
                  const uint64_t bd = sd + (uint64_t)((4 * kTcPlaneA + pb2[q] * kTcPlaneB + s * 32) >> 4);
                  tc_mma2_elect(d_re, ad, bd, id_pair, (c == 0 && s == 0 && q == 0) ? 0u : 1u);
                }
              } else if (s < n_steps) {
#pragma unroll
                for (int q = 0; q < 12; ++q) {
                  const uint64_t ad = sd + (uint64_t)((prod_a[q] * kTcPlaneA + s * 32) >> 4);
                  const uint64_t bd = sd + (uint64_t)((4 * kTcPlaneA + prod_b[q] * kTcPlaneB + s * 32) >> 4);
                  const bool first = (c == 0 && s == 0 && (q == 0 || q == 6));
                  tc_mma_elect(q < 6 ? d_re : d_im, ad, bd, (q >= 6 && q < 9) ? id_neg : id_pos, first ? 0u : 1u);
                }
              }
            }
            // frees the smem stage (PAIR: in both CTAs) when these MMAs finish
            if (PAIR) tc_commit2_elect(&empty[stage]);
            else tc_commit_elect(&empty[stage]);
            if (++stage == kTcStages) { stage = 0; phase ^= 1; }
          }
          if (PAIR) tc_commit2_elect(&tfull[reg]);  // accumulators of (bin, pass) complete
          else tc_commit_elect(&tfull[reg]);
        }
    }
  }
  } else {
    asm volatile("setmaxnreg.inc.sync.aligned.u32 112;");
    // ------------------------------------------------------------ epilogue
    // warp e = warp - 4: TMEM lane quadrant q = warp % 4 (hardware rule), column group h
    const int e = warp - 4, q = warp & 3, h = e >> 2;
    const int r = q * 32 + lane;             // tile row owned in the TMEM phase
    const int cb = h * kTcColsPerWarp;       // first tile column owned in the TMEM phase
    const float inv_nb = 1.f / (float)a.nbb;
    const uint32_t lane_addr = (uint32_t)(q * 32) << 16;
    const int et = e * 32 + lane;            // 0..255 within the epilogue group
    const uint32_t xb = smem_u32(xbuf), cfb = smem_u32(colfac), rob = smem_u32(rowoff_s);
    const uint32_t xrow = xb + (uint32_t)(r * kTcXStride) * 8u;  // this thread's transpose row
    const bool cohy = a.cohy_bins || a.cohy_band;
    uint32_t tuse = 0;  // bit r: phase of TMEM region r
    int seq = 0;        // region of the next (bin, pass), as in the MMA warp
    const uint32_t tempty0 = PAIR ? mapa_u32(smem_u32(tempty), 0) : 0u;  // the leader's region barriers
    for (int u = u0; u < n_units; u += ustep) {
    const int2 tij = a.tiles[u / a.nbc];
    const int bl0 = (u % a.nbc) * a.bpc, bl1 = min(a.nbb, bl0 + a.bpc);
    const int iBase = tij.x * kUnitRows + (int)rank * kTcTile, jBase = tij.y * kTcTileJ;
    const int i = iBase + r;
    const int chi = a.N - jBase;             // valid tile columns: c < chi (and c > i - jBase)
    // every (row, column) of the tile is a stored pair (strictly above the diagonal, inside N
    // and the row range): the per-bin stores need no predicates (warp-uniform)
    const bool full_tile = iBase + kTcTile <= jBase && jBase + kTcTileJ <= a.N && iBase >= a.i_lo &&
                           iBase + kTcTile <= a.i_hi;
    // (the previous unit's last epi_bar ordered its rowoff_s reads before these writes)
    if (et < kTcTile) {
      const int ii = iBase + et;
      const bool ok = ii >= a.i_lo && ii < a.i_hi && ii < a.N;
      // pair (ii, j) -> rowoff + j; row 0 legitimately has offset -1, so INT64_MIN marks skipped rows
      rowoff_s[et] = ok ? (int64_t)ii * (a.N - 1) - (int64_t)ii * (ii - 1) / 2 - ii - 1 - a.pair_base : INT64_MIN;
    }
    for (int bl = bl0; bl < bl1; ++bl) {
      const bool acc_band = bl != bl0;  // first bin of the chunk initialises the TMEM band sums
      const int64_t bo = (int64_t)bl * a.pair_stride;
      float rsi = 0.f;                  // 1/sqrt(psd_i s_i^2), 0 for a dead node
      if (a.do_x) {
        if (et < kTcTileJ) {
          const int j = jBase + et;
          float f = 0.f;
          if (j < a.N) {
            const float sj = a.nscale[(int64_t)bl * a.N + j];
            f = a.psd[(int64_t)bl * a.N + j] * sj * sj;
          }
          colfac[et] = f > 0.f ? rsqrtf(f) : 0.f;
        }
        if (i < a.N) {
          const float si = a.nscale[(int64_t)bl * a.N + i];
          const float pi = a.psd[(int64_t)bl * a.N + i] * si * si;
          rsi = pi > 0.f ? rsqrtf(pi) : 0.f;
        }
      }
      epi_bar();
      for (int ps = 0; ps < npass; ++ps) {
        const int pass = pass0 + ps;
        const int reg = seq;
        seq = seq + 1 == nreg ? 0 : seq + 1;
        mbar_wait(&tfull[reg], (tuse >> reg) & 1);
        tuse ^= 1u << reg;
        tc_fence_after();
        const uint32_t t_acc = tmem + lane_addr + (reg == 2 ? 384 : reg * 128);
#pragma unroll
        for (int c1 = 0; c1 < kTcColsPerWarp; c1 += 8) {
          const int c0 = cb + c1;
          float vr[8], vi[8];
          tmem_ld8x2(t_acc + c0, vr, t_acc + 64 + c0, vi);
          if (TC_ABL(2)) { sts_f2(xrow + c0 * 8u, vr[3], vi[5]); continue; }
          if (pass == 0) {
#pragma unroll
            for (int u4 = 0; u4 < 8; u4 += 4) {
              const float4 cf = lds_f4(cfb + (uint32_t)(c0 + u4) * 4u);
              const float rs[4] = {rsi * cf.x, rsi * cf.y, rsi * cf.z, rsi * cf.w};
#pragma unroll
              for (int u = 0; u < 4; ++u) {
                vr[u4 + u] *= rs[u];
                vi[u4 + u] *= rs[u];
              }
              if (a.flags) {
#pragma unroll
                for (int u = 0; u < 4; ++u) {
                  const int j = jBase + c0 + u4 + u;
                  if (rs[u] > 0.f && i < j && j < a.N && i >= a.i_lo && i < a.i_hi &&
                      fabsf(vi[u4 + u]) < a.imag_tau) {
                    const int slot = atomicAdd(&a.counters[0], 1);
                    if (slot < a.flag_cap) {
                      a.flags[slot] = make_int4(i, j, bl, 0);
                      vi[u4 + u] = 0.f;  // out of the band sum; the fallback adds the fp64 value
                    } else {
                      a.counters[1] = 1;  // list full: keep the tensor-core value (|err| < imag_tau)
                    }
                  }
                }
              }
            }
            if (a.coh_band || !cohy) {
              float m[8];
#pragma unroll
              for (int u = 0; u < 8; ++u) m[u] = sqrt_approx(vr[u] * vr[u] + vi[u] * vi[u]);
              if (!cohy)
#pragma unroll
                for (int u = 0; u < 8; ++u) sts_f2(xrow + (uint32_t)(c0 + u) * 8u, m[u], vi[u]);
              if (a.coh_band) {
                float b[8];
                if (acc_band) tmem_ld8(tmem + lane_addr + kTmBand + c0, b);
#pragma unroll
                for (int u = 0; u < 8; ++u) b[u] = acc_band ? fmaf(m[u], inv_nb, b[u]) : m[u] * inv_nb;
                tmem_st8(tmem + lane_addr + kTmBand + c0, b);
              }
            }
            if (a.imag_band && !a.cohy_band) {  // IMAGCOHY band mean in the COHY-im columns
              float bi[8];
              if (acc_band) tmem_ld8(tmem + lane_addr + kTmBand + 192 + c0, bi);
#pragma unroll
              for (int u = 0; u < 8; ++u) bi[u] = acc_band ? fmaf(vi[u], inv_nb, bi[u]) : vi[u] * inv_nb;
              tmem_st8(tmem + lane_addr + kTmBand + 192 + c0, bi);
            }
            if (cohy) {
#pragma unroll
              for (int u = 0; u < 8; ++u) sts_f2(xrow + (uint32_t)(c0 + u) * 8u, vr[u], vi[u]);
              if (a.cohy_band) {
                float br[8], bi[8];
                if (acc_band) tmem_ld8x2(tmem + lane_addr + kTmBand + 128 + c0, br, tmem + lane_addr + kTmBand + 192 + c0, bi);
#pragma unroll
                for (int u = 0; u < 8; ++u) {
                  br[u] = acc_band ? fmaf(vr[u], inv_nb, br[u]) : vr[u] * inv_nb;
                  bi[u] = acc_band ? fmaf(vi[u], inv_nb, bi[u]) : vi[u] * inv_nb;
                }
                tmem_st8(tmem + lane_addr + kTmBand + 128 + c0, br);
                tmem_st8(tmem + lane_addr + kTmBand + 192 + c0, bi);
              }
            }
          } else {
#pragma unroll
            for (int u = 0; u < 8; ++u) {
              vr[u] = sqrt_approx(vr[u] * vr[u] + vi[u] * vi[u]) * a.invK;
              sts_f32(xrow + (uint32_t)(c0 + u) * 8u, vr[u]);
            }
            if (a.plv_band) {
              float b[8];
              if (acc_band) tmem_ld8(tmem + lane_addr + kTmBand + 64 + c0, b);
#pragma unroll
              for (int u = 0; u < 8; ++u) b[u] = acc_band ? fmaf(vr[u], inv_nb, b[u]) : vr[u] * inv_nb;
              tmem_st8(tmem + lane_addr + kTmBand + 64 + c0, b);
            }
          }
        }
        // accumulators drained: hand the region back to the MMA warp
        asm volatile("tcgen05.wait::st.sync.aligned;" ::: "memory");
        tc_fence_before();
        __syncwarp();
        if (lane == 0) {
          if (PAIR) mbar_arrive_cluster_relaxed(tempty0 + (uint32_t)reg * 8u);
          else mbar_arrive(&tempty[reg]);
        }
        epi_bar();
        // per-bin outputs: warp e stores rows [8 e, 8 e + 8), 64 contiguous pairs each;
        // four rows per group, all shared loads of a group issued before its stores
        if (!TC_ABL(1)) {
          float* const px = pass == 0 ? a.coh_bins : a.plv_bins;   // .x: COH (or |COHY|) / PLV
          float* const py = pass == 0 ? a.imag_bins : nullptr;     // .y: IMAGCOHY
          float2* const pc = (pass == 0 && cohy) ? a.cohy_bins : nullptr;
          const bool magx = pass == 0 && cohy;                     // buffer holds COHY: COH = |.|
          if (full_tile && !pc && px) {
            // interior tile, every row in range, no COHY: no per-store predicates, one
            // 64-bit address per row (the c = 32 half is +32 floats)
            float* const pxb = px + bo + jBase + lane;
            float* const pyb = py ? py + bo + jBase + lane : nullptr;
#pragma unroll
            for (int g = 0; g < kTcRowsPerWarp; g += 4) {
              long long ro[4];
              float2 v0[4], v1[4];
#pragma unroll
              for (int t = 0; t < 4; ++t) {
                const int row = e * kTcRowsPerWarp + g + t;
                ro[t] = lds_s64(rob + (uint32_t)row * 8u);
                const uint32_t xa = xb + (uint32_t)(row * kTcXStride + lane) * 8u;
                v0[t] = lds_f2(xa);
                v1[t] = lds_f2(xa + 256u);
              }
#pragma unroll
              for (int t = 0; t < 4; ++t) {
                __stcs(pxb + ro[t], v0[t].x);  // streaming stores: keep the operands in L2
                __stcs(pxb + ro[t] + 32, v1[t].x);
                if (pyb) {
                  __stcs(pyb + ro[t], v0[t].y);
                  __stcs(pyb + ro[t] + 32, v1[t].y);
                }
              }
            }
          } else
          for (int g = 0; g < kTcRowsPerWarp; g += 4) {
            long long ro[4];
            float2 v0[4], v1[4];
#pragma unroll
            for (int t = 0; t < 4; ++t) {
              const int row = e * kTcRowsPerWarp + g + t;
              ro[t] = lds_s64(rob + (uint32_t)row * 8u);
              const uint32_t xa = xb + (uint32_t)(row * kTcXStride + lane) * 8u;
              v0[t] = lds_f2(xa);
              v1[t] = lds_f2(xa + 256u);
            }
#pragma unroll
            for (int t = 0; t < 4; ++t) {
              const int row = e * kTcRowsPerWarp + g + t;
              const int clo = iBase + row + 1 - jBase;
              const bool live = ro[t] != INT64_MIN;
              const bool ok0 = live && lane >= clo && lane < chi;
              const bool ok1 = live && lane + 32 >= clo && lane + 32 < chi;
              const int64_t off = bo + ro[t] + jBase + lane;
              if (px) {
                const float x0 = magx ? sqrt_approx(v0[t].x * v0[t].x + v0[t].y * v0[t].y) : v0[t].x;
                const float x1 = magx ? sqrt_approx(v1[t].x * v1[t].x + v1[t].y * v1[t].y) : v1[t].x;
                if (ok0) __stcs(px + off, x0);  // streaming stores: keep the operands in L2
                if (ok1) __stcs(px + off + 32, x1);
              }
              if (py) {
                if (ok0) __stcs(py + off, v0[t].y);
                if (ok1) __stcs(py + off + 32, v1[t].y);
              }
              if (pc) {
                if (ok0) __stcs(pc + off, v0[t]);
                if (ok1) __stcs(pc + off + 32, v1[t]);
              }
            }
          }
        }
        epi_bar();
      }
    }
    // band means: TMEM -> transpose buffer -> coalesced stores
    if (!TC_ABL(4) && (a.coh_band || a.plv_band || a.cohy_band || a.imag_band)) {
      asm volatile("tcgen05.wait::st.sync.aligned;" ::: "memory");
      for (int kind = 0; kind < 4; ++kind) {
        if ((kind == 0 && !a.coh_band) || (kind == 1 && !a.plv_band) || (kind == 2 && !a.cohy_band) ||
            (kind == 3 && (!a.imag_band || a.cohy_band)))
          continue;
#pragma unroll
        for (int c1 = 0; c1 < kTcColsPerWarp; c1 += 8) {
          const int c0 = cb + c1;
          float b0[8], b1[8];
          const uint32_t col = kTmBand + (kind >= 2 ? (kind == 3 ? 192 : 128) : kind * 64) + c0;
          if (kind == 2) tmem_ld8x2(tmem + lane_addr + col, b0, tmem + lane_addr + kTmBand + 192 + c0, b1);
          else tmem_ld8(tmem + lane_addr + col, b0);
#pragma unroll
          for (int u = 0; u < 8; ++u) sts_f2(xrow + (uint32_t)(c0 + u) * 8u, b0[u], kind == 2 ? b1[u] : 0.f);
        }
        epi_bar();
        float* dst1 = kind == 0 ? a.coh_band : (kind == 1 ? a.plv_band : a.imag_band);
        for (int rr = 0; rr < kTcRowsPerWarp; ++rr) {
          const int row = e * kTcRowsPerWarp + rr;
          const long long ro = lds_s64(rob + (uint32_t)row * 8u);
          if (ro == INT64_MIN) continue;
          const int clo = iBase + row + 1 - jBase;
#pragma unroll
          for (int hh = 0; hh < 2; ++hh) {
            const int c = lane + 32 * hh;
            if (c < clo || c >= chi) continue;
            const float2 v = lds_f2(xb + (uint32_t)(row * kTcXStride + c) * 8u);
            const int64_t o = ro + jBase + c;
            if (a.nbc > 1) {  // bins split over CTAs: the host zeroed the band outputs
              if (kind == 2) {
                atomicAdd(&a.cohy_band[o].x, v.x);
                atomicAdd(&a.cohy_band[o].y, v.y);
              } else {
                atomicAdd(&dst1[o], v.x);
              }
            } else if (kind == 2) {
              a.cohy_band[o] = v;
            } else {
              dst1[o] = v.x;
            }
            if (kind == 2 && a.imag_band) {  // IMAGCOHY band = Im of the COHY band mean
              if (a.nbc > 1) atomicAdd(&a.imag_band[o], v.y);
              else a.imag_band[o] = v.y;
            }
          }
        }
        epi_bar();
      }
    }
    }  // units
  }

  tc_fence_before();
  if (PAIR)
    cluster_sync();  // neither CTA frees TMEM while the pair's MMAs / epilogues may use it
  else
    __syncthreads();
  tc_fence_after();
  if (warp == 2) {
    if (PAIR) asm volatile("tcgen05.dealloc.cta_group::2.sync.aligned.b32 %0, 512;" ::"r"(tmem));
    else asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 512;" ::"r"(tmem));
  }
}

// ---------------------------------------------------------------- operand prep
// G[z = (bl*2 + pass)*kTcPlanes + plane][n][k] fp16, k < K_pad (zero padded):
//   pass 0: X * 2^-e(n,b) (|.| <= 1), pass 1: U = X/|X|; planes re_h, re_l, im_h, im_l, -im_h, -im_l.
__global__ void k_tc_prep(const float2* __restrict__ X32, const int* __restrict__ slots, int K, int K_pad,
                          int N, int nb, int L, int bin_lo, int nbb, const float* __restrict__ nscale,
                          __half* __restrict__ G, int neg_planes) {
  const int k = blockIdx.x * 32 + threadIdx.x;
  const int n = blockIdx.y * 8 + threadIdx.y;
  const int bl = blockIdx.z;
  if (n >= N || k >= K_pad) return;
  float xr = 0.f, xi = 0.f;
  if (k < K) {  // contraction index k = trial * L + taper (multitaper: CSD summed over tapers)
    const float2 v = X32[(((int64_t)slots[k / L] * L + k % L) * nb + bin_lo + bl) * N + n];
    const float s = nscale[(int64_t)bl * N + n];
    xr = v.x * s;
    xi = v.y * s;
  }
  const float m2 = xr * xr + xi * xi;
  const float inv = m2 > 0.f ? rsqrtf(m2) : 0.f;
  float vals[2][2] = {{xr, xi}, {xr * inv, xi * inv}};
  const size_t plane = (size_t)N * K_pad;
#pragma unroll
  for (int pass = 0; pass < 2; ++pass)
#pragma unroll
    for (int c = 0; c < 2; ++c) {
      const float v = vals[pass][c];
      const __half h = __float2half_rn(v);
      const __half l = __float2half_rn(v - __half2float(h));
      const size_t z = ((size_t)bl * 2 + pass) * kTcPlanes + c * 2;
      G[(z + 0) * plane + (size_t)n * K_pad + k] = h;
      G[(z + 1) * plane + (size_t)n * K_pad + k] = l;
      if (c == 1 && neg_planes) {  // -im_h, -im_l (exact negations; the CTA-pair kernel's B halves)
        G[(z + 2) * plane + (size_t)n * K_pad + k] = __hneg(h);
        G[(z + 3) * plane + (size_t)n * K_pad + k] = __hneg(l);
      }
    }
}

// ---------------------------------------------------------------- host side
size_t tc_smem_bytes() {
  return (size_t)kTcStages * kTcStageBytes + (size_t)kTcTile * kTcXStride * sizeof(float2) + kTcTileJ * 4 +
         kTcTile * 8 + 256;
}

// Tile list (I, J), J >= 2 I, of 128 x 64 tiles over the row range [i_lo, i_hi), in a
// grouped order: bands of 8 row tiles swept column by column, so the CTAs resident at
// once touch ~8 x 128 + 18 x 64 nodes of operands (L2 resident).  Built once per row
// range and cached in the plan (a blocking upload: first call for that range only).
// rmul = 2: 128-row tiles (J >= 2 I); rmul = 1: 64 x 64 tiles (J >= I) over row tiles [tile_row0, tile_row1)
const int2* tile_list(Plan& p, int tile_row0, int tile_row1, int nt64, int rmul, int64_t* n_tiles, cudaStream_t st) {
  const uint64_t key = ((uint64_t)tile_row0 << 40) ^ ((uint64_t)tile_row1 << 20) ^ (uint64_t)nt64 ^ ((uint64_t)rmul << 56);
  Plan::TileList* tle = nullptr;
  for (auto& e : p.tc_tiles)
    if (e.key == key && e.ptr) tle = &e;
  if (!tle) {
    std::vector<int2> tl;
    constexpr int GR = 8;
    for (int b0 = tile_row0; b0 < tile_row1; b0 += GR)
      for (int J = 0; J < nt64; ++J)
        for (int I = b0; I < b0 + GR && I < tile_row1; ++I)
          if (J >= rmul * I) tl.push_back(make_int2(I, J));
    tle = &p.tc_tiles[p.tc_tiles_next];
    p.tc_tiles_next = (p.tc_tiles_next + 1) % Plan::kTileCache;
    if (tle->ptr) {
      cudaStreamSynchronize(st);  // the evicted list may still be read by queued work
      cudaFree(tle->ptr);
    }
    tle->ptr = nullptr;
    tle->key = key;
    tle->n = (int64_t)tl.size();
    const size_t bytes = (tl.empty() ? 1 : tl.size()) * sizeof(int2);
    if (cudaMalloc(&tle->ptr, bytes) != cudaSuccess) {
      tle->ptr = nullptr;
      cs_set_error("device allocation failed (tile list)");
      return nullptr;
    }
    if (!tl.empty()) cudaMemcpy(tle->ptr, tl.data(), tl.size() * sizeof(int2), cudaMemcpyHostToDevice);
  }
  *n_tiles = tle->n;
  return (const int2*)tle->ptr;
}

// fp16 hi/lo split operands of the call (k_tc_prep) in the plan's buffer: [nbb][pass][plane][N][K_pad]
__half* tc_prep_ops(Plan& p, const int* slots, int K, int bin_lo, int nbb, const float* nscale, cudaStream_t st,
                    int* K_pad_out, bool neg_planes) {
  const int Kc = K * p.L;                       // contraction length: trials x tapers
  const int K_pad = (Kc + 15) / 16 * 16;        // UMMA K granularity; the last TMA box is zero-filled
  const size_t need = (size_t)nbb * 2 * kTcPlanes * p.N * K_pad * sizeof(__half);
  if (need > p.tc_bytes) {
    if (p.tc_ops) cudaFreeAsync(p.tc_ops, st);
    if (cudaMallocAsync(&p.tc_ops, need, st) != cudaSuccess) {
      cs_set_error("device allocation failed (tensor-core operands %zu bytes)", need);
      p.tc_ops = nullptr;
      p.tc_bytes = 0;
      return nullptr;
    }
    p.tc_bytes = need;
  }
  __half* G = (__half*)p.tc_ops;
  if (!p.reuse_prep || (neg_planes && !p.tc_neg_planes)) {
    p.tc_neg_planes = neg_planes;
    PhaseMark ph(p, "tc_prep", st);
    dim3 grid((K_pad + 31) / 32, (p.N + 7) / 8, nbb);
    k_tc_prep<<<grid, dim3(32, 8), 0, st>>>(p.X32, slots, Kc, K_pad, p.N, p.nb, p.L, bin_lo, nbb, nscale, G,
                                            neg_planes ? 1 : 0);
  }
  *K_pad_out = K_pad;
  return G;
}

bool run_pairs_tc(Plan& p, const int* slots, int K, int bin_lo, int nbb, int rb, int re, bool do_x, bool do_u,
                  bool do_imag, const cs_outputs* out, const float* nscale, cudaStream_t st, bool handoff) {
  EncodeTiledFn enc = get_encode();
  if (!enc) {
    cs_set_error("cuTensorMapEncodeTiled unavailable");
    return false;
  }
  int nsm = 148;
  cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, p.device);
  // CTA pairs (256 x 64 tiles, cta_group::2) when the row range gives every pair of SMs at
  // least two tiles and no more masked rows than single-CTA 128 x 64 tiles would (a shard
  // whose row range is not 256-aligned computes the rows outside it for nothing: at 8 ranks
  // of cfg5 the busiest rank would run 1.22x the single-CTA work); small pair spaces keep
  // single CTAs and bin splitting.  Both kernels issue the same products in the same order
  // per element, so the choice never changes a result bit (tests/test_gpu_pair.py).
  const char* pair_s = getenv("CSCONN_K2_PAIR");  // A/B and test override: 0 single CTAs, 1 CTA pairs
  const int pair_env = pair_s ? atoi(pair_s) : -1;
  const int nt64 = (p.N + kTcTileJ - 1) / kTcTileJ;
  const int r_lo = rb * kTile, r_hi = re * kTile < p.N ? re * kTile : p.N;
  auto unit_tiles = [&](int rows) {  // tiles of `rows` x 64 over [r_lo, r_hi), J >= rows / 64 * I
    int64_t n = 0;
    for (int I = r_lo / rows; I < (r_hi + rows - 1) / rows; ++I) n += nt64 - rows / kTcTileJ * I > 0 ? nt64 - rows / kTcTileJ * I : 0;
    return n;
  };
  const int64_t t128 = unit_tiles(kTcTile), t256 = unit_tiles(2 * kTcTile);
  const bool pair = pair_env >= 0 ? pair_env > 0 : (t256 >= nsm && 2 * t256 <= t128 + t128 / 50);
  int K_pad = 0;
  __half* G = tc_prep_ops(p, slots, K, bin_lo, nbb, nscale, st, &K_pad, pair);
  if (!G) return false;
  const int Kc = K * p.L;
  CUtensorMap mapA, mapB;
  cuuint64_t dims[3] = {(cuuint64_t)K_pad, (cuuint64_t)p.N, (cuuint64_t)nbb * 2 * kTcPlanes};
  cuuint64_t strides[2] = {(cuuint64_t)K_pad * 2, (cuuint64_t)p.N * K_pad * 2};
  cuuint32_t boxA[3] = {(cuuint32_t)kTcChunk, (cuuint32_t)kTcTile, 1};
  cuuint32_t boxB[3] = {(cuuint32_t)kTcChunk, (cuuint32_t)kTcTileJ, 1};
  cuuint32_t estr[3] = {1, 1, 1};
  CUresult r = enc(&mapA, CU_TENSOR_MAP_DATA_TYPE_FLOAT16, 3, G, dims, strides, boxA, estr,
                   CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_64B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                   CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  if (r == CUDA_SUCCESS)
    r = enc(&mapB, CU_TENSOR_MAP_DATA_TYPE_FLOAT16, 3, G, dims, strides, boxB, estr, CU_TENSOR_MAP_INTERLEAVE_NONE,
            CU_TENSOR_MAP_SWIZZLE_64B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  if (r != CUDA_SUCCESS) {
    cs_set_error("cuTensorMapEncodeTiled failed (%d)", (int)r);
    return false;
  }
  TcArgs a{};
  a.N = p.N; a.K = Kc; a.K_pad = K_pad; a.nbb = nbb;
  a.i_lo = rb * kTile;
  a.i_hi = re * kTile < p.N ? re * kTile : p.N;
  a.nt = (p.N + kTcTileJ - 1) / kTcTileJ;
  const int unit_rows = pair ? 2 * kTcTile : kTcTile;
  a.tile_row0 = a.i_lo / unit_rows;
  int64_t n_tiles = 0;
  a.tiles = tile_list(p, a.i_lo / unit_rows, (a.i_hi + unit_rows - 1) / unit_rows, a.nt, unit_rows / kTcTileJ,
                      &n_tiles, st);
  if (!a.tiles) return false;
  a.n_tiles = (int)n_tiles;
  if (pair) {
    a.bpc = nbb;
    a.nbc = 1;
  } else {  // small pair spaces: split bins over CTAs.  Persistent CTAs overlap most of a
     // work unit's fixed cost, so the time is ~ rounds x (unit overhead + bins x
     // per-bin cost) with the overhead ~2 bins (cfg1/2/4 sweeps); pick the split
     // minimising rounds * (2 + bins per unit).
    int nbc = 1;
    double best = 1e300;
    for (int c = 1; c <= nbb && n_tiles > 0; ++c) {
      const int bpc = (nbb + c - 1) / c, chunks = (nbb + bpc - 1) / bpc;
      if (chunks != c) continue;
      const double cost = (double)((n_tiles * chunks + nsm - 1) / nsm) * (2.0 + bpc);
      if (cost < best) {
        best = cost;
        nbc = c;
      }
    }
    static const int force_nbc = getenv("CSCONN_K2_NBC") ? atoi(getenv("CSCONN_K2_NBC")) : 0;  // sweep override
    if (force_nbc) nbc = force_nbc < 1 ? 1 : (force_nbc > nbb ? nbb : force_nbc);
    a.bpc = (nbb + nbc - 1) / nbc;
    a.nbc = (nbb + a.bpc - 1) / a.bpc;
  }
  a.psd = p.psd; a.nscale = nscale;
  a.invK = 1.f / (float)K;
  a.pair_base = out->pair_base; a.pair_stride = out->pair_stride;
  a.cohy_bins = do_x ? (float2*)out->bins[0] : nullptr;
  a.cohy_band = do_x ? (float2*)out->band[0] : nullptr;
  a.coh_bins = do_x ? (float*)out->bins[1] : nullptr;
  a.coh_band = do_x ? (float*)out->band[1] : nullptr;
  a.plv_bins = do_u ? (float*)out->bins[3] : nullptr;
  a.plv_band = do_u ? (float*)out->band[3] : nullptr;
  a.imag_bins = do_imag ? (float*)out->bins[2] : nullptr;
  // hand-off: per-bin IMAGCOHY only (the phase-lag kernel forms the band mean and flags)
  a.imag_band = do_imag && !handoff ? (float*)out->band[2] : nullptr;
  a.do_x = do_x; a.do_u = do_u;
  if (do_imag && !handoff && (a.imag_bins || a.imag_band)) {
    a.flags = p.flags;
    a.counters = p.counters;
    a.flag_cap = p.flag_cap;
    a.imag_tau = 1e-5f + 6e-8f * (float)Kc;  // > fp16-split + fp32-accumulation error of D_im / norm
    cudaMemsetAsync(p.counters, 0, 2 * sizeof(int), st);
  }
#ifdef CS_TC_ABLATION
  { const char* d = getenv("CSCONN_TC_DBG"); a.dbg = d ? atoi(d) : 0; }
#endif
  const size_t smem = tc_smem_bytes();
  CS_SMEM_ONCE(k_pairs_tc<false>, smem);
  CS_SMEM_ONCE(k_pairs_tc<true>, smem);
  {
    PhaseMark ph(p, "pairs_tc", st);
    if (a.nbc > 1) {
      if (a.coh_band) cudaMemsetAsync(a.coh_band, 0, a.pair_stride * sizeof(float), st);
      if (a.plv_band) cudaMemsetAsync(a.plv_band, 0, a.pair_stride * sizeof(float), st);
      if (a.cohy_band) cudaMemsetAsync(a.cohy_band, 0, a.pair_stride * sizeof(float2), st);
      if (a.imag_band) cudaMemsetAsync(a.imag_band, 0, a.pair_stride * sizeof(float), st);
    }
    if (n_tiles > 0 && !pair) {  // persistent: one CTA per SM (210 KB smem), units strided over the grid
      const int64_t units = n_tiles * a.nbc;
      const int64_t grid = units < nsm ? units : nsm;
      k_pairs_tc<false><<<(unsigned)grid, kTcThreads, smem, st>>>(mapA, mapB, a);
    } else if (n_tiles > 0) {  // persistent CTA pairs (clusters of 2: the two SMs of a TPC)
      const int64_t units = n_tiles;
      const int64_t pairs = units < nsm / 2 ? units : nsm / 2;
      cudaLaunchConfig_t cfg = {};
      cfg.gridDim = dim3((unsigned)(2 * pairs));
      cfg.blockDim = dim3(kTcThreads);
      cfg.dynamicSmemBytes = smem;
      cfg.stream = st;
      cudaLaunchAttribute at[1];
      at[0].id = cudaLaunchAttributeClusterDimension;
      at[0].val.clusterDim.x = 2;
      at[0].val.clusterDim.y = 1;
      at[0].val.clusterDim.z = 1;
      cfg.attrs = at;
      cfg.numAttrs = 1;
      const cudaError_t e = cudaLaunchKernelEx(&cfg, k_pairs_tc<true>, mapA, mapB, a);
      if (e != cudaSuccess) {
        cs_set_error("k_pairs_tc (CTA pairs) launch failed: %s", cudaGetErrorString(e));
        return false;
      }
    }
  }
  return true;
}

}  // namespace cs
