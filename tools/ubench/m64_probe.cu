// Probe: one tcgen05.mma kind::f16 with M = 64, N = 64, K = 16, both operands K-major
// 16-half (32-byte) rows written by TMA with SWIZZLE_32B.  Checks the SW32 smem
// descriptor (layout type 6, SBO = 8 rows x 32 B) and where the 64 accumulator rows land
// in TMEM (dumps all 128 lanes x 64 columns and tests two placements).
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o m64_probe m64_probe.cu -lcuda
#include <cuda.h>
#include <cuda_fp16.h>
#include <cuda_runtime.h>

#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <random>
#include <vector>

__device__ __forceinline__ uint32_t su32(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }
__device__ __forceinline__ uint64_t desc_sw32(uint32_t addr) {
  uint64_t d = 0;
  d |= (uint64_t)((addr >> 4) & 0x3FFF);
  d |= (uint64_t)1 << 16;               // LBO (ignored, swizzled K-major)
  d |= (uint64_t)(256 >> 4) << 32;      // SBO: 8-row groups of 32-byte rows
  d |= (uint64_t)1 << 46;               // version
  d |= (uint64_t)6 << 61;               // SWIZZLE_32B
  return d;
}
__host__ __device__ constexpr uint32_t idesc(int M, int N) {
  return (1u << 4) | ((uint32_t)(N >> 3) << 17) | ((uint32_t)(M >> 4) << 24);
}

__global__ void k_probe(const __grid_constant__ CUtensorMap mA, const __grid_constant__ CUtensorMap mB, float* out,
                        float* out2) {
  extern __shared__ __align__(1024) unsigned char sm[];
  unsigned char* sA = sm;          // 64 x 32 B
  unsigned char* sB = sm + 2048;   // 64 x 32 B
  uint64_t* bar = (uint64_t*)(sm + 4096);
  uint64_t* mbar = bar + 1;
  uint32_t* tslot = (uint32_t*)(bar + 2);
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  if (threadIdx.x == 0) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(su32(bar)));
    asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(su32(mbar)));
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  if (warp == 0) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 128;" ::"r"(su32(tslot)));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
  const uint32_t tmem = *tslot;
  // zero the 128 lanes x 64 columns first (so unwritten lanes read 0)
  {
    uint32_t z = 0;
    for (int c = 0; c < 64; ++c)
      asm volatile("tcgen05.st.sync.aligned.32x32b.x1.b32 [%0], {%1};" ::"r"(tmem + ((uint32_t)(warp * 32) << 16) + c), "r"(z));
    asm volatile("tcgen05.wait::st.sync.aligned;" ::: "memory");
  }
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
  if (threadIdx.x == 0) {
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(su32(bar)), "r"(4096) : "memory");
    asm volatile("cp.async.bulk.tensor.2d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%3, %4}], [%2];"
                 ::"r"(su32(sA)), "l"((uint64_t)&mA), "r"(su32(bar)), "r"(0), "r"(0) : "memory");
    asm volatile("cp.async.bulk.tensor.2d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%3, %4}], [%2];"
                 ::"r"(su32(sB)), "l"((uint64_t)&mB), "r"(su32(bar)), "r"(0), "r"(0) : "memory");
    uint32_t done = 0;
    while (!done)
      asm volatile("{\n\t.reg .pred P1;\n\tmbarrier.try_wait.parity.shared::cta.b64 P1, [%1], 0;\n\tselp.u32 %0, 1, 0, P1;\n\t}"
                   : "=r"(done) : "r"(su32(bar)) : "memory");
    asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
    asm volatile("tcgen05.mma.cta_group::1.kind::f16 [%0], %1, %2, %3, 0;" ::"r"(tmem), "l"(desc_sw32(su32(sA))),
                 "l"(desc_sw32(su32(sB))), "r"(idesc(64, 64)));
    asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(su32(mbar))
                 : "memory");
  }
  __syncwarp();
  {
    uint32_t done = 0;
    while (!done)
      asm volatile("{\n\t.reg .pred P1;\n\tmbarrier.try_wait.parity.shared::cta.b64 P1, [%1], 0;\n\tselp.u32 %0, 1, 0, P1;\n\t}"
                   : "=r"(done) : "r"(su32(mbar)) : "memory");
  }
  asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
  const int row = warp * 32 + lane;
  for (int c = 0; c < 64; ++c) {
    uint32_t v;
    asm volatile("tcgen05.ld.sync.aligned.32x32b.x1.b32 {%0}, [%1];" : "=r"(v) : "r"(tmem + ((uint32_t)(warp * 32) << 16) + c));
    asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
    out[row * 64 + c] = __uint_as_float(v);
  }
  // unique values lane * 1000 + column, then read back with 16x256b.x2
  for (int c = 0; c < 64; ++c) {
    const float v = (float)(row * 1000 + c);
    asm volatile("tcgen05.st.sync.aligned.32x32b.x1.b32 [%0], {%1};" ::"r"(tmem + ((uint32_t)(warp * 32) << 16) + c),
                 "r"(__float_as_uint(v)));
  }
  asm volatile("tcgen05.wait::st.sync.aligned;" ::: "memory");
  {  // 16x256b.x2: 16 lanes x 16 columns per warp, 8 registers per thread
    uint32_t r[8];
    asm volatile("tcgen05.ld.sync.aligned.16x256b.x2.b32 {%0,%1,%2,%3,%4,%5,%6,%7}, [%8];"
                 : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]), "=r"(r[7])
                 : "r"(tmem + ((uint32_t)(warp * 32) << 16)));
    asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
    for (int q = 0; q < 8; ++q) out2[(warp * 32 + lane) * 8 + q] = __uint_as_float(r[q]);
  }
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
  if (warp == 0) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 128;" ::"r"(tmem));
}

int main() {
  std::mt19937 rng(5);
  std::uniform_int_distribution<int> d(-3, 3);
  std::vector<__half> A(64 * 16), B(64 * 16);
  std::vector<float> Af(64 * 16), Bf(64 * 16);
  for (int e = 0; e < 64 * 16; ++e) {
    Af[e] = (float)d(rng);
    Bf[e] = (float)d(rng);
    A[e] = __float2half(Af[e]);
    B[e] = __float2half(Bf[e]);
  }
  __half *dA, *dB;
  float* dO;
  float* dO2;
  cudaMalloc(&dO2, 128 * 8 * 4);
  cudaMalloc(&dA, A.size() * 2);
  cudaMalloc(&dB, B.size() * 2);
  cudaMalloc(&dO, 128 * 64 * 4);
  cudaMemcpy(dA, A.data(), A.size() * 2, cudaMemcpyHostToDevice);
  cudaMemcpy(dB, B.data(), B.size() * 2, cudaMemcpyHostToDevice);
  CUtensorMap mA, mB;
  cuuint64_t dims[2] = {16, 64};
  cuuint64_t str[1] = {32};
  cuuint32_t box[2] = {16, 64};
  cuuint32_t es[2] = {1, 1};
  CUresult r1 = cuTensorMapEncodeTiled(&mA, CU_TENSOR_MAP_DATA_TYPE_FLOAT16, 2, dA, dims, str, box, es,
                                       CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_32B,
                                       CU_TENSOR_MAP_L2_PROMOTION_NONE, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  CUresult r2 = cuTensorMapEncodeTiled(&mB, CU_TENSOR_MAP_DATA_TYPE_FLOAT16, 2, dB, dims, str, box, es,
                                       CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_32B,
                                       CU_TENSOR_MAP_L2_PROMOTION_NONE, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  printf("encode %d %d\n", (int)r1, (int)r2);
  cudaFuncSetAttribute(k_probe, cudaFuncAttributeMaxDynamicSharedMemorySize, 8192);
  k_probe<<<1, 128, 8192>>>(mA, mB, dO, dO2);
  cudaError_t e = cudaDeviceSynchronize();
  printf("kernel %s\n", cudaGetErrorString(e));
  std::vector<float> O(128 * 64);
  cudaMemcpy(O.data(), dO, O.size() * 4, cudaMemcpyDeviceToHost);
  auto ref = [&](int m, int n) {
    float s = 0;
    for (int k = 0; k < 16; ++k) s += Af[m * 16 + k] * Bf[n * 16 + k];
    return s;
  };
  double e1 = 0, e2 = 0;
  for (int m = 0; m < 64; ++m)
    for (int n = 0; n < 64; ++n) {
      e1 = fmax(e1, fabs(O[m * 64 + n] - ref(m, n)));
      const int l2 = 32 * (m / 16) + (m % 16);
      e2 = fmax(e2, fabs(O[l2 * 64 + n] - ref(m, n)));
    }
  printf("H1 lane = m: max err %g\nH2 lane = 32 (m / 16) + m %% 16: max err %g\n", e1, e2);
  for (int l = 0; l < 128; l += 8) {
    printf("lane %3d:", l);
    for (int c = 0; c < 4; ++c) printf(" %6.1f", O[l * 64 + c]);
    printf("   ref rows:");
    for (int m = 0; m < 64; m += 16) printf(" %6.1f", ref(m, 0));
    printf("\n");
  }
  // 16x256b.x2 mapping: register value = lane * 1000 + column
  std::vector<float> O2(128 * 8);
  cudaMemcpy(O2.data(), dO2, O2.size() * 4, cudaMemcpyDeviceToHost);
  for (int t = 0; t < 32; ++t) {
    printf("warp0 thread %2d:", t);
    for (int q = 0; q < 8; ++q) printf(" (l%d,c%d)", (int)O2[t * 8 + q] / 1000, (int)O2[t * 8 + q] % 1000);
    printf("\n");
  }
  return 0;
}
