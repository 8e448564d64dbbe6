// Probe for a tensor-core phase-lag kernel: per-trial t = Im(X_i conj X_j) from
// fp16 hi/lo operands with kind::f16 tcgen05.mma, no-swizzle K-major layouts.
//   A (M = 128 rows i, K = 16 = two trials x 8 entries)   core (g, h) at g*128 + h*2048
//   B block-diagonal (N = 128 = (j, trial), K = 16)       [k0 1 KB][zeros 1 KB][k1 1 KB]
//   B' (N = 64 rows j, K = 16)                            same bytes, K-stride 2048
// Checks the descriptor convention (which field strides K) and measures the error of
// the tensor-core sum against the exact (double) sum of the same fp16 products and
// against the exact t of the fp32 inputs, in units of 2^-24 M_i M_j.
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o tc_lag_probe tc_lag_probe.cu -lcuda
#include <cuda.h>
#include <cuda_fp16.h>
#include <cuda_runtime.h>

#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <random>
#include <vector>

__device__ __forceinline__ uint32_t su32(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }
__device__ __forceinline__ uint64_t desc_none(uint32_t addr, uint32_t lbo, uint32_t sbo) {
  uint64_t d = 0;
  d |= (uint64_t)((addr >> 4) & 0x3FFF);
  d |= (uint64_t)((lbo >> 4) & 0x3FFF) << 16;
  d |= (uint64_t)((sbo >> 4) & 0x3FFF) << 32;
  d |= (uint64_t)1 << 46;
  return d;
}
__host__ __device__ constexpr uint32_t idesc(int M, int N) {
  return (1u << 4) | ((uint32_t)(N >> 3) << 17) | ((uint32_t)(M >> 4) << 24);
}

// in: A 4096 B, B 3072 B (zeros included); out: [128][192] f32 (D_t 128 cols, D_s 64 cols)
__global__ void k_probe(const uint4* A, const uint4* B, float* out, int swap) {
  extern __shared__ __align__(1024) uint4 dyn[];  // 64 KB: a wrong stride reads zeros, not out of range
  uint4* sA = dyn;
  uint4* sB = dyn + 512;
  uint64_t& bar = *(uint64_t*)(dyn + 4000);
  uint32_t& tslot = *(uint32_t*)(dyn + 4001);
  for (int e = threadIdx.x; e < 4096; e += blockDim.x) dyn[e] = make_uint4(0, 0, 0, 0);
  __syncthreads();
  for (int e = threadIdx.x; e < 256; e += blockDim.x) sA[e] = A[e];
  for (int e = threadIdx.x; e < 192; e += blockDim.x) sB[e] = B[e];
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  if (threadIdx.x == 0) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(su32(&bar)));
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  if (warp == 0) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 256;" ::"r"(su32(&tslot)));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
  const uint32_t tmem = tslot;
  if (threadIdx.x == 0) {
    // K-direction core stride kA / kB, M/N-direction 128 B
    const uint32_t a_k = 2048, bt_k = 1024, bs_k = 2048, mn = 128;
    const uint64_t da = swap ? desc_none(su32(sA), mn, a_k) : desc_none(su32(sA), a_k, mn);
    const uint64_t dbt = swap ? desc_none(su32(sB), mn, bt_k) : desc_none(su32(sB), bt_k, mn);
    const uint64_t dbs = swap ? desc_none(su32(sB), mn, bs_k) : desc_none(su32(sB), bs_k, mn);
    asm volatile("tcgen05.mma.cta_group::1.kind::f16 [%0], %1, %2, %3, 0;" ::"r"(tmem), "l"(da), "l"(dbt),
                 "r"(idesc(128, 128)));
    asm volatile("tcgen05.mma.cta_group::1.kind::f16 [%0], %1, %2, %3, 0;" ::"r"(tmem + 128), "l"(da), "l"(dbs),
                 "r"(idesc(128, 64)));
    asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(su32(&bar))
                 : "memory");
  }
  __syncwarp();
  {
    uint32_t done = 0;
    while (!done)
      asm volatile("{\n\t.reg .pred P1;\n\tmbarrier.try_wait.parity.shared::cta.b64 P1, [%1], 0;\n\tselp.u32 %0, 1, 0, P1;\n\t}"
                   : "=r"(done) : "r"(su32(&bar)) : "memory");
  }
  asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
  const int row = warp * 32 + lane;
  for (int c0 = 0; c0 < 192; c0 += 8) {
    uint32_t r[8];
    asm volatile("tcgen05.ld.sync.aligned.32x32b.x8.b32 {%0,%1,%2,%3,%4,%5,%6,%7}, [%8];"
                 : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]), "=r"(r[7])
                 : "r"(tmem + ((uint32_t)(warp * 32) << 16) + c0));
    asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
    for (int q = 0; q < 8; ++q) out[row * 192 + c0 + q] = __uint_as_float(r[q]);
  }
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  __syncthreads();
  if (warp == 0) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 256;" ::"r"(tmem));
}


// round-trip latency: MMA(s) + commit + mbarrier wait, repeated (one thread issues, all wait)
__global__ void k_lat(float* out, int reps, int nmma) {
  extern __shared__ __align__(1024) uint4 dyn[];
  uint4* sA = dyn;
  uint4* sB = dyn + 512;
  uint64_t& bar = *(uint64_t*)(dyn + 4000);
  uint32_t& tslot = *(uint32_t*)(dyn + 4001);
  for (int e = threadIdx.x; e < 4096; e += blockDim.x) dyn[e] = make_uint4(0x3c003c00u, 0, 0, 0);
  __syncthreads();
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
  const int warp = threadIdx.x >> 5;
  if (threadIdx.x == 0) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(su32(&bar)));
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  if (warp == 0) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 256;" ::"r"(su32(&tslot)));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
  const uint32_t tmem = tslot;
  const uint64_t da = desc_none(su32(sA), 2048, 128), dbt = desc_none(su32(sB), 1024, 128);
  long long t0 = clock64();
  for (int r = 0; r < reps; ++r) {
    if (threadIdx.x == 0) {
      for (int m = 0; m < nmma; ++m)
        asm volatile("tcgen05.mma.cta_group::1.kind::f16 [%0], %1, %2, %3, 0;" ::"r"(tmem), "l"(da), "l"(dbt),
                     "r"(idesc(128, 128)));
      asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(su32(&bar))
                   : "memory");
    }
    uint32_t done = 0;
    while (!done)
      asm volatile("{\n\t.reg .pred P1;\n\tmbarrier.try_wait.parity.shared::cta.b64 P1, [%1], %2;\n\tselp.u32 %0, 1, 0, P1;\n\t}"
                   : "=r"(done) : "r"(su32(&bar)), "r"((uint32_t)(r & 1)) : "memory");
    asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
  }
  long long t1 = clock64();
  if (threadIdx.x == 0) out[0] = (float)(t1 - t0) / reps;
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  __syncthreads();
  if (warp == 0) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 256;" ::"r"(tmem));
}

static void split(float x, __half& h, __half& l) {
  h = __float2half_rn(x);
  l = __float2half_rn(x - __half2float(h));
}

int main() {
  {
    float* d; cudaMalloc(&d, 4);
    cudaFuncSetAttribute(k_lat, cudaFuncAttributeMaxDynamicSharedMemorySize, 65536);
    for (int nm : {1, 2, 4, 16}) for (int thr : {32, 512}) {
      k_lat<<<1, thr, 65536>>>(d, 1000, nm);
      float c; cudaMemcpy(&c, d, 4, cudaMemcpyDeviceToHost);
      printf("MMA x%d + commit + wait round trip (%d threads waiting): %.0f cycles (%s)\n", nm, thr, c, cudaGetErrorString(cudaGetLastError()));
    }
  }
  std::mt19937 rng(7);
  std::uniform_real_distribution<float> U(-1.f, 1.f);
  double worst_acc = 0, worst_tot = 0, worst_guard = 0;
  int bad_layout[2] = {0, 0};
  for (int rep = 0; rep < 2000; ++rep) {
    // nodes: i 128, j 64, trials 2; magnitudes spread over decades, max |x| in (0.5, 1]
    float xi[2][128][2], xj[2][64][2];
    double Mi[128] = {0}, Mj[64] = {0};
    for (int k = 0; k < 2; ++k)
      for (int n = 0; n < 128; ++n) {
        const float s = powf(2.f, -(float)(rng() % 12));
        xi[k][n][0] = U(rng) * s; xi[k][n][1] = U(rng) * s;
      }
    for (int k = 0; k < 2; ++k)
      for (int n = 0; n < 64; ++n) {
        const float s = powf(2.f, -(float)(rng() % 12));
        xj[k][n][0] = U(rng) * s; xj[k][n][1] = U(rng) * s;
      }
    if (rep % 3 == 0)  // near-cancelling pairs: j = i (rows 0..63) with a tiny phase shift in trial 1
      for (int n = 0; n < 64; ++n) {
        xj[0][n][0] = xi[0][n][0]; xj[0][n][1] = xi[0][n][1];
        xj[1][n][0] = xi[1][n][0] * (1.f + 1e-6f * U(rng)); xj[1][n][1] = xi[1][n][1];
      }
    for (int n = 0; n < 128; ++n) for (int k = 0; k < 2; ++k) Mi[n] = fmax(Mi[n], hypot(xi[k][n][0], xi[k][n][1]));
    for (int n = 0; n < 64; ++n) for (int k = 0; k < 2; ++k) Mj[n] = fmax(Mj[n], hypot(xj[k][n][0], xj[k][n][1]));
    // per-node power-of-two scale: max |x| in (0.5, 1] (as the kernel's operand prep does)
    for (int n = 0; n < 128; ++n) {
      const double s = ldexp(1.0, -(int)ceil(log2(Mi[n])));
      for (int k = 0; k < 2; ++k) { xi[k][n][0] *= s; xi[k][n][1] *= s; }
      Mi[n] *= s;
    }
    for (int n = 0; n < 64; ++n) {
      const double s = ldexp(1.0, -(int)ceil(log2(Mj[n])));
      for (int k = 0; k < 2; ++k) { xj[k][n][0] *= s; xj[k][n][1] *= s; }
      Mj[n] *= s;
    }
    // encodings: A = [Im_h, Im_l, Im_h, Im_l, -Re_h, -Re_l, -Re_h, -Re_l],
    //            B = [Re_h, Re_h, Re_l, Re_l, Im_h, Im_h, Im_l, Im_l]
    std::vector<__half> hA(2048), hB(1536, __float2half_rn(0.f));
    float ea[2][128][8], eb[2][64][8];
    for (int k = 0; k < 2; ++k) {
      for (int n = 0; n < 128; ++n) {
        __half rh, rl, ih, il;
        split(xi[k][n][0], rh, rl);
        split(xi[k][n][1], ih, il);
        __half e[8] = {ih, il, ih, il, __hneg(rh), __hneg(rl), __hneg(rh), __hneg(rl)};
        for (int c = 0; c < 8; ++c) { hA[k * 1024 + n * 8 + c] = e[c]; ea[k][n][c] = __half2float(e[c]); }
      }
      for (int n = 0; n < 64; ++n) {
        __half rh, rl, ih, il;
        split(xj[k][n][0], rh, rl);
        split(xj[k][n][1], ih, il);
        __half e[8] = {rh, rh, rl, rl, ih, ih, il, il};
        for (int c = 0; c < 8; ++c) { hB[k * 1024 + n * 8 + c] = e[c]; eb[k][n][c] = __half2float(e[c]); }
      }
    }
    uint4 *dA, *dB;
    float* dO;
    cudaMalloc(&dA, 4096); cudaMalloc(&dB, 3072); cudaMalloc(&dO, 128 * 192 * 4);
    cudaMemcpy(dA, hA.data(), 4096, cudaMemcpyHostToDevice);
    cudaMemcpy(dB, hB.data(), 3072, cudaMemcpyHostToDevice);
    std::vector<float> o(128 * 192);
    for (int swap = 0; swap < 2; ++swap) {
      if (rep > 0 && swap == 1) break;
      cudaFuncSetAttribute(k_probe, cudaFuncAttributeMaxDynamicSharedMemorySize, 65536);
      k_probe<<<1, 128, 65536>>>(dA, dB, dO, swap);
      cudaError_t err = cudaDeviceSynchronize();
      if (err != cudaSuccess) { printf("launch error %s\n", cudaGetErrorString(err)); return 1; }
      cudaMemcpy(o.data(), dO, o.size() * 4, cudaMemcpyDeviceToHost);
      for (int i = 0; i < 128; ++i)
        for (int j = 0; j < 64; ++j) {
          double tsp[2], tex[2];
          for (int k = 0; k < 2; ++k) {
            double s = 0;
            for (int c = 0; c < 8; ++c) s += (double)ea[k][i][c] * (double)eb[k][j][c];
            tsp[k] = s;
            tex[k] = (double)xi[k][i][1] * xj[k][j][0] - (double)xi[k][i][0] * xj[k][j][1];
          }
          const double mm = Mi[i] * Mj[j];
          const double d0 = o[i * 192 + j], d1 = o[i * 192 + 64 + j], ds = o[i * 192 + 128 + j];
          const double e_acc = fmax(fabs(d0 - tsp[0]), fmax(fabs(d1 - tsp[1]), fabs(ds - tsp[0] - tsp[1]) / 2)) / mm;
          const double e_tot = fmax(fabs(d0 - tex[0]), fabs(d1 - tex[1])) / mm;
          if (e_tot > 1e-3) bad_layout[swap]++;
          if (rep == 0 && i == 5 && j < 3) printf("swap %d i %d j %d: D0 %g (want %g) D1 %g (want %g) Ds %g\n", swap, i, j, d0, tex[0], d1, tex[1], ds);
          if (swap == 0 || rep == 0) {
            if (swap == 0) {
              worst_acc = fmax(worst_acc, e_acc);
              worst_tot = fmax(worst_tot, e_tot);
            }
          }
          // error of the fp32 SIMT formula (FMUL + FFMA) for reference
          const float f = fmaf(xi[0][i][1], xj[0][j][0], -(xi[0][i][0] * xj[0][j][1]));
          worst_guard = fmax(worst_guard, fabs((double)f - tex[0]) / mm);
        }
    }
    cudaFree(dA); cudaFree(dB); cudaFree(dO);
  }
  printf("layout errors (e_tot > 1e-3): lbo=K-stride %d, swapped %d (of %d entries in rep 0)\n", bad_layout[0],
         bad_layout[1], 128 * 64);
  printf("tensor-core accumulation error  max %.3f x 2^-24 M_i M_j\n", worst_acc * 16777216.0);
  printf("tensor-core t vs exact fp32-in  max %.3f x 2^-24 M_i M_j\n", worst_tot * 16777216.0);
  printf("fp32 FMUL+FFMA t vs exact       max %.3f x 2^-24 M_i M_j\n", worst_guard * 16777216.0);
  return 0;
}
