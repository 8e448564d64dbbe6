// Network post-processing on the device: normalisation by the
// maximum |weight| (core.py:168-181) and the top-ceil(f P) threshold by |weight|
// with ascending-(i, j) tie-break (core.py:184-205), without host copies of the
// P-edge arrays.
//
// Threshold = radix select + order-preserving compaction.  Keys are the |w|
// float bits (monotone for non-negative floats).  Four 8-bit MSB-first passes
// find the keep-th largest key tau and how many of the tau ties are kept; the
// ties kept are the lowest pair indices (edges are in triu order, so ascending
// pair index = ascending (i, j)).  The compaction writes the kept pair indices in
// ascending order: per-block counts of (|w| > tau) and ties, an exclusive scan,
// then every block places its elements.  No host synchronisation.
#include <algorithm>

#include "common.cuh"

namespace cs {

__device__ __forceinline__ uint32_t absbits(float v) { return __float_as_uint(v) & 0x7fffffffu; }

__global__ void k_absmax(const float* __restrict__ w, int64_t n, unsigned* __restrict__ out) {
  unsigned m = 0;
  for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < n; e += (int64_t)gridDim.x * blockDim.x)
    m = max(m, absbits(w[e]));
  for (int o = 16; o > 0; o >>= 1) m = max(m, __shfl_xor_sync(0xffffffffu, m, o));
  if ((threadIdx.x & 31) == 0) atomicMax(out, m);
}

__global__ void k_scale(float* __restrict__ w, float2* __restrict__ cw, int64_t n, const unsigned* __restrict__ mx) {
  const float m = __uint_as_float(*mx);
  if (m == 0.f) return;  // an all-zero network is returned unchanged (core.py:176-177)
  for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < n; e += (int64_t)gridDim.x * blockDim.x) {
    w[e] = w[e] / m;
    if (cw) cw[e] = make_float2(cw[e].x / m, cw[e].y / m);
  }
}

// select state: [0] prefix bits, [1] prefix mask, [2] remaining rank k (1-based),
// [3] number of keys > tau (after the last pass), [4] ties kept
struct SelState {
  unsigned prefix, mask;
  long long k, n_gt, ties;
};

__global__ void k_hist(const float* __restrict__ w, int64_t n, const SelState* __restrict__ s, int shift,
                       unsigned long long* __restrict__ hist) {
  __shared__ unsigned h[256];
  for (int i = threadIdx.x; i < 256; i += blockDim.x) h[i] = 0;
  __syncthreads();
  const unsigned prefix = s->prefix, mask = s->mask;
  for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < n; e += (int64_t)gridDim.x * blockDim.x) {
    const unsigned key = absbits(w[e]);
    if ((key & mask) == prefix) atomicAdd(&h[(key >> shift) & 255u], 1u);
  }
  __syncthreads();
  for (int i = threadIdx.x; i < 256; i += blockDim.x)
    if (h[i]) atomicAdd(&hist[i], (unsigned long long)h[i]);
}

// 256 threads, one digit each: the count of keys in digits above d is a scan from
// the top; the thread whose digit holds the k-th largest key updates the state,
// and every thread clears its histogram bin.
__global__ void __launch_bounds__(256) k_pick(SelState* __restrict__ s, int shift,
                                              unsigned long long* __restrict__ hist) {
  __shared__ long long wsum[8];
  const int d = 255 - (int)threadIdx.x;  // thread 0 holds the top digit
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const long long c = (long long)hist[d];
  long long x = c;  // inclusive scan in thread order = count of keys in digits >= d
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    const long long y = __shfl_up_sync(0xffffffffu, x, o);
    if (lane >= o) x += y;
  }
  if (lane == 31) wsum[warp] = x;
  const long long k = s->k;
  __syncthreads();
  for (int i = 0; i < warp; ++i) x += wsum[i];
  const long long above = x - c;  // keys in digits > d
  // the digit holding rank k; digit 0 takes whatever is left (as the serial scan did)
  if ((above < k && x >= k && d > 0) || (d == 0 && above < k)) {
    s->prefix |= (unsigned)d << shift;
    s->mask |= 255u << shift;
    s->n_gt += above;
    s->k = k - above;
  }
  hist[d] = 0;
}

constexpr int kSelBlock = 256, kSelItems = 16;  // 4096 elements per compaction block

__global__ void k_count(const float* __restrict__ w, int64_t n, const SelState* __restrict__ s,
                        long long* __restrict__ cnt_gt, long long* __restrict__ cnt_tie) {
  const unsigned tau = s->prefix;
  const int64_t base = (int64_t)blockIdx.x * kSelBlock * kSelItems;
  int gt = 0, tie = 0;
  for (int q = 0; q < kSelItems; ++q) {
    const int64_t e = base + (int64_t)q * kSelBlock + threadIdx.x;
    if (e < n) {
      const unsigned key = absbits(w[e]);
      gt += key > tau;
      tie += key == tau;
    }
  }
  for (int o = 16; o > 0; o >>= 1) {
    gt += __shfl_xor_sync(0xffffffffu, gt, o);
    tie += __shfl_xor_sync(0xffffffffu, tie, o);
  }
  __shared__ int sg[kSelBlock / 32], st[kSelBlock / 32];
  if ((threadIdx.x & 31) == 0) {
    sg[threadIdx.x >> 5] = gt;
    st[threadIdx.x >> 5] = tie;
  }
  __syncthreads();
  if (threadIdx.x == 0) {
    long long a = 0, b = 0;
    for (int i = 0; i < kSelBlock / 32; ++i) {
      a += sg[i];
      b += st[i];
    }
    cnt_gt[blockIdx.x] = a;
    cnt_tie[blockIdx.x] = b;
  }
}

// exclusive scan of the per-block counts (one CTA; nblk is small: P / 4096)
__global__ void k_scan(long long* __restrict__ cnt_gt, long long* __restrict__ cnt_tie, int nblk) {
  __shared__ long long carry_g, carry_t;
  __shared__ long long wg[32], wt[32];
  if (threadIdx.x == 0) carry_g = carry_t = 0;
  __syncthreads();
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  for (int b0 = 0; b0 < nblk; b0 += blockDim.x) {
    const int b = b0 + threadIdx.x;
    long long g = b < nblk ? cnt_gt[b] : 0, t = b < nblk ? cnt_tie[b] : 0;
    long long ig = g, it = t;  // inclusive warp scan
    for (int o = 1; o < 32; o <<= 1) {
      const long long yg = __shfl_up_sync(0xffffffffu, ig, o), yt = __shfl_up_sync(0xffffffffu, it, o);
      if (lane >= o) {
        ig += yg;
        it += yt;
      }
    }
    if (lane == 31) {
      wg[warp] = ig;
      wt[warp] = it;
    }
    __syncthreads();
    if (warp == 0) {
      long long xg = lane < (int)(blockDim.x >> 5) ? wg[lane] : 0, xt = lane < (int)(blockDim.x >> 5) ? wt[lane] : 0;
      for (int o = 1; o < 32; o <<= 1) {
        const long long yg = __shfl_up_sync(0xffffffffu, xg, o), yt = __shfl_up_sync(0xffffffffu, xt, o);
        if (lane >= o) {
          xg += yg;
          xt += yt;
        }
      }
      wg[lane] = xg;  // inclusive warp totals
      wt[lane] = xt;
    }
    __syncthreads();
    const long long offg = carry_g + (warp ? wg[warp - 1] : 0) + ig - g;
    const long long offt = carry_t + (warp ? wt[warp - 1] : 0) + it - t;
    if (b < nblk) {
      cnt_gt[b] = offg;
      cnt_tie[b] = offt;
    }
    __syncthreads();
    if (threadIdx.x == 0) {
      carry_g += wg[(blockDim.x >> 5) - 1];
      carry_t += wt[(blockDim.x >> 5) - 1];
    }
    __syncthreads();
  }
}

// exclusive block-wide scan of one int per thread (kSelBlock threads)
__device__ __forceinline__ int block_excl_scan(int v, int* wsum) {
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  int x = v;
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    const int y = __shfl_up_sync(0xffffffffu, x, o);
    if (lane >= o) x += y;
  }
  if (lane == 31) wsum[warp] = x;
  __syncthreads();
  int before = 0;
#pragma unroll
  for (int i = 0; i < kSelBlock / 32; ++i) before += i < warp ? wsum[i] : 0;
  __syncthreads();  // wsum reusable
  return before + x - v;
}

// Thread t of block b owns the 16 consecutive elements b*4096 + 16t .. +15 (same
// block ranges as k_count): one vector load, the ties before it from a block scan,
// its kept elements decided in order, their output slots from a second scan.
__global__ void __launch_bounds__(kSelBlock) k_compact(const float* __restrict__ w, int64_t n,
                                                       const SelState* __restrict__ s,
                                                       const long long* __restrict__ off_gt,
                                                       const long long* __restrict__ off_tie,
                                                       int64_t* __restrict__ out) {
  __shared__ int wsum[kSelBlock / 32];
  const unsigned tau = s->prefix;
  const long long ties_kept = s->k;  // the tau ties kept (lowest indices first)
  const int64_t base = (int64_t)blockIdx.x * kSelBlock * kSelItems + (int64_t)threadIdx.x * kSelItems;
  unsigned key[kSelItems];
  if (base + kSelItems <= n && ((reinterpret_cast<uintptr_t>(w) & 15) == 0)) {
#pragma unroll
    for (int q = 0; q < kSelItems / 4; ++q) {
      const float4 v = __ldcs(reinterpret_cast<const float4*>(w + base) + q);
      key[4 * q] = absbits(v.x);
      key[4 * q + 1] = absbits(v.y);
      key[4 * q + 2] = absbits(v.z);
      key[4 * q + 3] = absbits(v.w);
    }
  } else {
#pragma unroll
    for (int q = 0; q < kSelItems; ++q) key[q] = base + q < n ? absbits(w[base + q]) : 0u;
  }
  int nt = 0;
#pragma unroll
  for (int q = 0; q < kSelItems; ++q) nt += (base + q < n) && key[q] == tau;
  long long tie = off_tie[blockIdx.x] + block_excl_scan(nt, wsum);
  unsigned sel = 0;
#pragma unroll
  for (int q = 0; q < kSelItems; ++q) {
    const bool in = base + q < n;
    bool keep = in && key[q] > tau;
    if (in && key[q] == tau) keep = tie++ < ties_kept;
    sel |= (unsigned)keep << q;
  }
  const long long blk_sel = off_gt[blockIdx.x] + min(off_tie[blockIdx.x], ties_kept);
  long long pos = blk_sel + block_excl_scan(__popc(sel), wsum);
  while (sel) {
    const int q = __ffs(sel) - 1;
    sel &= sel - 1;
    out[pos++] = base + q;
  }
}

}  // namespace cs

extern "C" {

int cs_net_normalize(float* w, void* cw, int64_t n, void* stream) {
  if (!w || n < 1) { cs_set_error("cannot normalize a network without edges"); return CS_EPARAM; }
  cudaStream_t st = (cudaStream_t)stream;
  unsigned* mx = nullptr;
  if (cudaMallocAsync(&mx, sizeof(unsigned), st) != cudaSuccess) { cs_set_error("device allocation failed"); return CS_ENOMEM; }
  cudaMemsetAsync(mx, 0, sizeof(unsigned), st);
  const int grid = (int)std::min<int64_t>((n + 255) / 256, 148 * 8);
  cs::k_absmax<<<grid, 256, 0, st>>>(w, n, mx);
  cs::k_scale<<<grid, 256, 0, st>>>(w, (float2*)cw, n, mx);
  cudaFreeAsync(mx, st);
  return cudaPeekAtLastError() == cudaSuccess ? CS_OK : CS_ECUDA;
}

int cs_net_threshold(const float* w, int64_t n, int64_t keep, int64_t* out_idx, void* stream) {
  if (!w || !out_idx || n < 1) { cs_set_error("cs_net_threshold: null argument"); return CS_EPARAM; }
  if (keep < 1 || keep > n) { cs_set_error("keep count %lld outside [1, %lld]", (long long)keep, (long long)n); return CS_EPARAM; }
  cudaStream_t st = (cudaStream_t)stream;
  const int nblk = (int)((n + cs::kSelBlock * cs::kSelItems - 1) / (cs::kSelBlock * cs::kSelItems));
  const size_t bytes = sizeof(cs::SelState) + 256 * sizeof(unsigned long long) + 2 * (size_t)nblk * sizeof(long long);
  unsigned char* ws = nullptr;
  if (cudaMallocAsync(&ws, bytes, st) != cudaSuccess) { cs_set_error("device allocation failed"); return CS_ENOMEM; }
  cs::SelState* s = (cs::SelState*)ws;
  unsigned long long* hist = (unsigned long long*)(ws + sizeof(cs::SelState));
  long long* cg = (long long*)(hist + 256);
  long long* ct = cg + nblk;
  cs::SelState init{0u, 0u, (long long)keep, 0, 0};
  cudaMemcpyAsync(s, &init, sizeof(init), cudaMemcpyHostToDevice, st);
  cudaMemsetAsync(hist, 0, 256 * sizeof(unsigned long long), st);
  const int grid = (int)std::min<int64_t>((n + 255) / 256, 148 * 8);
  for (int shift = 24; shift >= 0; shift -= 8) {
    cs::k_hist<<<grid, 256, 0, st>>>(w, n, s, shift, hist);
    cs::k_pick<<<1, 256, 0, st>>>(s, shift, hist);
  }
  cs::k_count<<<nblk, cs::kSelBlock, 0, st>>>(w, n, s, cg, ct);
  cs::k_scan<<<1, 1024, 0, st>>>(cg, ct, nblk);
  cs::k_compact<<<nblk, cs::kSelBlock, 0, st>>>(w, n, s, cg, ct, out_idx);
  cudaFreeAsync(ws, st);
  return cudaPeekAtLastError() == cudaSuccess ? CS_OK : CS_ECUDA;
}

}  // extern "C"
