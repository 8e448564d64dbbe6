// fp64 mma.sync m8n8k4 (DMMA) vs DFMA throughput probe on sm_100a.
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o dmma_rate dmma_rate.cu
#include <cstdio>
#include <cuda_runtime.h>

__global__ void k_dmma(double* out, int iters) {
  double a = threadIdx.x * 1e-3, b = 1.0 + threadIdx.x * 1e-4;
  double c[4][2] = {};
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int q = 0; q < 4; ++q)
      asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};"
                   : "+d"(c[q][0]), "+d"(c[q][1]) : "d"(a), "d"(b));
  }
  double s = 0;
  for (int q = 0; q < 4; ++q) s += c[q][0] + c[q][1];
  if (s == 12345.678) out[0] = s;
}
__global__ void k_dfma(double* out, int iters) {
  double a = threadIdx.x * 1e-3, b = 1.0 + threadIdx.x * 1e-4;
  double c[8] = {};
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int q = 0; q < 8; ++q) c[q] = fma(a, b, c[q]);
  }
  double s = 0;
  for (int q = 0; q < 8; ++q) s += c[q];
  if (s == 12345.678) out[0] = s;
}
// both pipes at once: even warps DMMA, odd warps DFMA (or every warp interleaving both)
__global__ void k_mixed(double* out, int iters, int mode, int dfma_per_dmma) {
  double a = threadIdx.x * 1e-3, b = 1.0 + threadIdx.x * 1e-4;
  double c[4][2] = {}, f[8] = {};
  const bool dm = mode == 0 ? ((threadIdx.x >> 5) & 1) == 0 : true;
  const bool df = mode == 0 ? !dm : true;
  for (int it = 0; it < iters; ++it) {
    if (dm) {
#pragma unroll
      for (int q = 0; q < 4; ++q)
        asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};"
                     : "+d"(c[q][0]), "+d"(c[q][1]) : "d"(a), "d"(b));
    }
    if (df) {
      for (int r = 0; r < dfma_per_dmma; ++r) {
#pragma unroll
        for (int q = 0; q < 8; ++q) f[q] = fma(a, b, f[q]);
      }
    }
  }
  double s = 0;
  for (int q = 0; q < 4; ++q) s += c[q][0] + c[q][1];
  for (int q = 0; q < 8; ++q) s += f[q];
  if (s == 12345.678) out[0] = s;
}
int main() {
  double* d;
  cudaMalloc(&d, 8);
  int nsm = 148, iters = 20000;
  for (int warps = 4; warps <= 32; warps *= 2) {
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0); cudaEventCreate(&e1);
    k_dmma<<<nsm, warps * 32>>>(d, 100);
    cudaEventRecord(e0);
    k_dmma<<<nsm, warps * 32>>>(d, iters);
    cudaEventRecord(e1);
    cudaEventSynchronize(e1);
    float ms; cudaEventElapsedTime(&ms, e0, e1);
    double fmas = (double)nsm * warps * iters * 4 * 256;
    printf("DMMA warps/SM=%d: %.2f T FMA/s\n", warps, fmas / (ms * 1e-3) / 1e12);
    k_dfma<<<nsm, warps * 32>>>(d, 100);
    cudaEventRecord(e0);
    k_dfma<<<nsm, warps * 32>>>(d, iters);
    cudaEventRecord(e1);
    cudaEventSynchronize(e1);
    cudaEventElapsedTime(&ms, e0, e1);
    fmas = (double)nsm * warps * 32 * iters * 8;
    printf("DFMA warps/SM=%d: %.2f T FMA/s\n", warps, fmas / (ms * 1e-3) / 1e12);
  }
  for (int mode = 0; mode < 2; ++mode)
    for (int rep = 1; rep <= 4; rep *= 2)
      for (int warps = 8; warps <= 16; warps *= 2) {
        cudaEvent_t e0, e1;
        cudaEventCreate(&e0); cudaEventCreate(&e1);
        k_mixed<<<nsm, warps * 32>>>(d, 100, mode, rep);
        cudaEventRecord(e0);
        k_mixed<<<nsm, warps * 32>>>(d, iters, mode, rep);
        cudaEventRecord(e1);
        cudaEventSynchronize(e1);
        float ms; cudaEventElapsedTime(&ms, e0, e1);
        const double dw = mode == 0 ? warps / 2 : warps;  // warps issuing each kind
        const double dm = (double)nsm * dw * iters * 4 * 256, dfm = (double)nsm * dw * 32 * iters * 8 * rep;
        printf("MIXED mode=%d (%s) dfma_x=%d warps/SM=%d: DMMA %.2f + DFMA %.2f = %.2f T FMA/s\n", mode,
               mode ? "interleaved" : "split warps", rep, warps, dm / (ms * 1e-3) / 1e12, dfm / (ms * 1e-3) / 1e12,
               (dm + dfm) / (ms * 1e-3) / 1e12);
      }
  printf("%s\n", cudaGetErrorString(cudaDeviceSynchronize()));
  return 0;
}
