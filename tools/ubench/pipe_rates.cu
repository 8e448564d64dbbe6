// Issue cost per SMSP of the instruction forms the phase-lag loop uses, one form at a
// time: 16 independent chains per thread, W warps per SM.  Prints SMSP cycles per warp
// instruction (1.0 = one per cycle; 2.0 = the pipe takes every other cycle).
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o pipe_rates pipe_rates.cu
#include <cstdio>
#include <cuda_runtime.h>
typedef unsigned long long u64;

template <int OP>
__global__ void k(u64* out, long long* cyc, int iters) {
  u64 r[16];
#pragma unroll
  for (int i = 0; i < 16; ++i) r[i] = 0x3f8000003f800000ull + threadIdx.x + i;
  const u64 c = 0x3f0000003f000000ull ^ (u64)blockIdx.x;
  __syncthreads();
  long long t0 = clock64();
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int i = 0; i < 16; ++i) {
      if (OP == 0) asm volatile("fma.rn.f32x2 %0, %0, %1, %1;" : "+l"(r[i]) : "l"(c));
      if (OP == 1) asm volatile("add.rn.f32x2 %0, %0, %1;" : "+l"(r[i]) : "l"(c));
      if (OP == 2) {  // |t| packed add: the abs of another chain's value (ptxas fuses it into FADD2 |R|)
        float a, b;
        asm("mov.b64 {%0,%1}, %2;" : "=f"(a), "=f"(b) : "l"(r[i ^ 1]));
        u64 p;
        asm("mov.b64 %0, {%1,%2};" : "=l"(p) : "f"(fabsf(a)), "f"(fabsf(b)));
        asm volatile("add.rn.f32x2 %0, %0, %1;" : "+l"(r[i]) : "l"(p));
      }
      if (OP == 9) asm volatile("add.rn.f32x2 %0, %0, %1;" : "+l"(r[i]) : "l"(r[i ^ 1]));  // same, no abs
      if (OP == 3) {  // scalar FADD with |x|
        float a;
        asm("mov.b32 %0, %1;" : "=f"(a) : "r"((unsigned)r[i]));
        asm volatile("add.rn.f32 %0, %0, %1;" : "+f"(a) : "f"(__uint_as_float((unsigned)c)));
        r[i] = (r[i] & ~0xffffffffull) | __float_as_uint(a);
      }
      if (OP == 4) {  // scalar FFMA 3-reg
        float a = __uint_as_float((unsigned)r[i]);
        asm volatile("fma.rn.f32 %0, %0, %1, %2;" : "+f"(a) : "f"(__uint_as_float((unsigned)c)), "f"(__uint_as_float((unsigned)(c >> 32))));
        r[i] = (r[i] & ~0xffffffffull) | __float_as_uint(a);
      }
      if (OP == 5) {  // 3-input float min
        float a = __uint_as_float((unsigned)r[i]);
        asm volatile("min.f32 %0, %0, %1, %2;" : "+f"(a) : "f"(__uint_as_float((unsigned)c)), "f"(__uint_as_float((unsigned)(c >> 32))));
        r[i] = (r[i] & ~0xffffffffull) | __float_as_uint(a);
      }
      if (OP == 6) {  // PRMT
        unsigned a = (unsigned)r[i];
        asm volatile("prmt.b32 %0, %0, %1, 0xFFBB;" : "+r"(a) : "r"((unsigned)c));
        r[i] = (r[i] & ~0xffffffffull) | a;
      }
      if (OP == 7) {  // IADD3
        unsigned a = (unsigned)r[i];
        asm volatile("add.u32 %0, %0, %1;" : "+r"(a) : "r"((unsigned)c));
        r[i] = (r[i] & ~0xffffffffull) | a;
      }
      if (OP == 8) asm volatile("mul.rn.f32x2 %0, %0, %1;" : "+l"(r[i]) : "l"(c));
    }
  }
  long long t1 = clock64();
  u64 s = 0;
#pragma unroll
  for (int i = 0; i < 16; ++i) s ^= r[i];
  out[blockIdx.x * blockDim.x + threadIdx.x] = s;
  if (threadIdx.x == 0) cyc[blockIdx.x] = t1 - t0;
}

template <int OP>
void run(const char* name, int warps) {
  const int blocks = 148, threads = warps * 32, iters = 4096;
  u64* out;
  long long* cyc;
  cudaMalloc(&out, sizeof(u64) * blocks * threads);
  cudaMalloc(&cyc, sizeof(long long) * blocks);
  k<OP><<<blocks, threads>>>(out, cyc, 64);
  k<OP><<<blocks, threads>>>(out, cyc, iters);
  cudaDeviceSynchronize();
  long long h[148];
  cudaMemcpy(h, cyc, sizeof(h), cudaMemcpyDeviceToHost);
  double avg = 0;
  for (int b = 0; b < blocks; ++b) avg += h[b];
  avg /= blocks;
  // warp-instructions per SMSP: warps/4 * iters * 16
  const double per = avg / ((warps / 4.0) * iters * 16.0);
  printf("%-26s warps/SM %2d: %.3f SMSP cycles per warp instruction\n", name, warps, per);
  cudaFree(out);
  cudaFree(cyc);
}

int main() {
  for (int w : {8, 16}) {
    run<4>("FFMA (3 reg)", w);
    run<0>("FFMA2", w);
    run<8>("FMUL2", w);
    run<1>("FADD2", w);
    run<2>("FADD2 |a| (reg operand)", w);
    run<9>("FADD2 (reg operand)", w);
    run<3>("FADD", w);
    run<5>("FMNMX3", w);
    run<6>("PRMT", w);
    run<7>("IADD3", w);
  }
  return 0;
}
