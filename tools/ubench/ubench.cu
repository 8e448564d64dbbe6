// Pipe-throughput microbenchmarks for sizing the phase-lag (K3) kernel:
// scalar FFMA vs packed fma.rn.f32x2, DFMA, and a K3-shaped update body.
#include <cstdio>
#include <cuda_runtime.h>
#define ITERS 4096
__global__ void k_ffma(float* out, float a, float b) {
  float x[8];
  for (int i = 0; i < 8; i++) x[i] = threadIdx.x + i;
  for (int it = 0; it < ITERS; it++) {
#pragma unroll
    for (int i = 0; i < 8; i++) x[i] = fmaf(x[i], a, b);
  }
  float s = 0; for (int i = 0; i < 8; i++) s += x[i];
  if (s == 12345.f) out[0] = s;
}
__device__ __forceinline__ unsigned long long f2pack(float lo, float hi) {
  unsigned long long r; asm("mov.b64 %0, {%1,%2};" : "=l"(r) : "f"(lo), "f"(hi)); return r; }
__global__ void k_ffma2(float* out, float a, float b) {
  unsigned long long x[8];
  for (int i = 0; i < 8; i++) x[i] = f2pack(threadIdx.x + i, i);
  unsigned long long A = f2pack(a, a), B = f2pack(b, b);
  for (int it = 0; it < ITERS; it++) {
#pragma unroll
    for (int i = 0; i < 8; i++) asm volatile("fma.rn.f32x2 %0, %0, %1, %2;" : "+l"(x[i]) : "l"(A), "l"(B));
  }
  unsigned long long s = 0; for (int i = 0; i < 8; i++) s ^= x[i];
  if (s == 12345ull) out[0] = 1;
}
__global__ void k_dfma(double* out, double a, double b) {
  double x[8];
  for (int i = 0; i < 8; i++) x[i] = threadIdx.x + i;
  for (int it = 0; it < ITERS; it++) {
#pragma unroll
    for (int i = 0; i < 8; i++) x[i] = fma(x[i], a, b);
  }
  double s = 0; for (int i = 0; i < 8; i++) s += x[i];
  if (s == 12345.0) out[0] = s;
}
// K3-shaped body: t = ai*br - ar*bi ; abs += |t| ; im += t ; neg += t<0 ; mn = min(mn,|t|)
__global__ void k_k3(float* out, const float4* __restrict__ src) {
  float4 xi[4], xj[4];
  for (int i = 0; i < 4; i++) { xi[i] = src[threadIdx.x % 32 + i]; xj[i] = src[threadIdx.x % 32 + 8 + i]; }
  float ab[16], im[16], mn[16]; int ng[16];
  for (int p = 0; p < 16; p++) { ab[p] = 0; im[p] = 0; mn[p] = 1e30f; ng[p] = 0; }
  for (int it = 0; it < ITERS / 8; it++) {
#pragma unroll
    for (int a = 0; a < 4; a++)
#pragma unroll
      for (int b = 0; b < 4; b++) {
        int p = a * 4 + b;
        float t = fmaf(xi[a].y, xj[b].x, -xi[a].x * xj[b].y);
        ab[p] += fabsf(t); im[p] += t; mn[p] = fminf(mn[p], fabsf(t));
        ng[p] += __float_as_uint(t) >> 31;
      }
#pragma unroll
    for (int a = 0; a < 4; a++) { xi[a].x += 1.0f; xj[a].y += 0.5f; }
  }
  float s = 0; for (int p = 0; p < 16; p++) s += ab[p] + im[p] + mn[p] + ng[p];
  out[blockIdx.x * blockDim.x + threadIdx.x] = s;
}
// packed variant: two trials per f32x2 lane pair
__global__ void k_k3p(float* out, const float4* __restrict__ src) {
  float4 xi[4], xj[4];
  for (int i = 0; i < 4; i++) { xi[i] = src[threadIdx.x % 32 + i]; xj[i] = src[threadIdx.x % 32 + 8 + i]; }
  unsigned long long ab[16], im[16]; float mn[16]; int ng[16];
  for (int p = 0; p < 16; p++) { ab[p] = 0; im[p] = 0; mn[p] = 1e30f; ng[p] = 0; }
  for (int it = 0; it < ITERS / 16; it++) {
#pragma unroll
    for (int a = 0; a < 4; a++)
#pragma unroll
      for (int b = 0; b < 4; b++) {
        int p = a * 4 + b;
        // xi = (re_k, re_k1, im_k, im_k1)
        unsigned long long ir = f2pack(xi[a].x, xi[a].y), ii = f2pack(xi[a].z, xi[a].w);
        unsigned long long jr = f2pack(xj[b].x, xj[b].y), ji = f2pack(xj[b].z, xj[b].w);
        unsigned long long q, t;
        asm("mul.rn.f32x2 %0, %1, %2;" : "=l"(q) : "l"(ir), "l"(ji));
        asm("fma.rn.f32x2 %0, %1, %2, %3;" : "=l"(t) : "l"(ii), "l"(jr), "l"(q ^ 0x8000000080000000ull));
        asm("add.rn.f32x2 %0, %0, %1;" : "+l"(im[p]) : "l"(t));
        unsigned long long ta = t & 0x7fffffff7fffffffull;
        asm("add.rn.f32x2 %0, %0, %1;" : "+l"(ab[p]) : "l"(ta));
        unsigned lo = (unsigned)t, hi = (unsigned)(t >> 32);
        ng[p] += (lo >> 31) + (hi >> 31);
        mn[p] = fminf(mn[p], fminf(__uint_as_float(lo & 0x7fffffff), __uint_as_float(hi & 0x7fffffff)));
      }
#pragma unroll
    for (int a = 0; a < 4; a++) { xi[a].x += 1.0f; xj[a].y += 0.5f; }
  }
  float s = 0; for (int p = 0; p < 16; p++) s += __uint_as_float((unsigned)ab[p]) + __uint_as_float((unsigned)im[p]) + mn[p] + ng[p];
  out[blockIdx.x * blockDim.x + threadIdx.x] = s;
}
int main() {
  int nsm = 0; cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, 0);
  int clk = 0; cudaDeviceGetAttribute(&clk, cudaDevAttrClockRate, 0);
  printf("SMs %d clock %d kHz\n", nsm, clk);
  float* d; cudaMalloc(&d, 1 << 26); double* dd = (double*)d; float4* src; cudaMalloc(&src, 4096);
  cudaMemset(src, 0, 4096);
  cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
  int grid = nsm * 8, blk = 256; double thr = (double)grid * blk;
  for (int rep = 0; rep < 3; rep++) {
    float ms;
    cudaEventRecord(e0); k_ffma<<<grid, blk>>>(d, 1.0001f, 0.5f); cudaEventRecord(e1); cudaEventSynchronize(e1);
    cudaEventElapsedTime(&ms, e0, e1); printf("FFMA  : %.2f T fma-lane-ops/s\n", thr * ITERS * 8 / ms / 1e9);
    cudaEventRecord(e0); k_ffma2<<<grid, blk>>>(d, 1.0001f, 0.5f); cudaEventRecord(e1); cudaEventSynchronize(e1);
    cudaEventElapsedTime(&ms, e0, e1); printf("FFMA2 : %.2f T fma-lane-ops/s (2 per instr)\n", thr * ITERS * 8 * 2 / ms / 1e9);
    cudaEventRecord(e0); k_dfma<<<grid, blk>>>(dd, 1.0001, 0.5); cudaEventRecord(e1); cudaEventSynchronize(e1);
    cudaEventElapsedTime(&ms, e0, e1); printf("DFMA  : %.2f T dfma/s\n", thr * ITERS * 8 / ms / 1e9);
    cudaEventRecord(e0); k_k3<<<grid, blk>>>(d, src); cudaEventRecord(e1); cudaEventSynchronize(e1);
    cudaEventElapsedTime(&ms, e0, e1); printf("K3 scalar body: %.2f T updates/s\n", thr * (ITERS / 8) * 16 / ms / 1e9);
    cudaEventRecord(e0); k_k3p<<<grid, blk>>>(d, src); cudaEventRecord(e1); cudaEventSynchronize(e1);
    cudaEventElapsedTime(&ms, e0, e1); printf("K3 packed body: %.2f T updates/s\n", thr * (ITERS / 16) * 16 * 2 / ms / 1e9);
  }
  printf("err %s\n", cudaGetErrorString(cudaGetLastError()));
  return 0;
}
