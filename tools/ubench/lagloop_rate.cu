// Throughput of the phase-lag inner loop's instruction mix without memory traffic:
// per pair and trial pair FMUL2 + FFMA2 (t), FADD2 (sum t), 2 FADD |t| (sum |t|),
// PRMT + IADD3/2 (sign counts), FMNMX3 (min |t|); 8 pairs per thread, 16 warps/SM.
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o lagloop_rate lagloop_rate.cu
#include <cstdio>
#include <cuda_runtime.h>
typedef unsigned long long f2;
__device__ __forceinline__ f2 pk(float a, float b) { f2 r; asm("mov.b64 %0, {%1,%2};" : "=l"(r) : "f"(a), "f"(b)); return r; }
__device__ __forceinline__ float lo(f2 v) { float a, b; asm("mov.b64 {%0,%1}, %2;" : "=f"(a), "=f"(b) : "l"(v)); return a; }
__device__ __forceinline__ float hi(f2 v) { float a, b; asm("mov.b64 {%0,%1}, %2;" : "=f"(a), "=f"(b) : "l"(v)); return b; }
__device__ __forceinline__ f2 fmul2(f2 a, f2 b) { f2 d; asm volatile("mul.rn.f32x2 %0, %1, %2;" : "=l"(d) : "l"(a), "l"(b)); return d; }
__device__ __forceinline__ f2 ffma2(f2 a, f2 b, f2 c) { f2 d; asm volatile("fma.rn.f32x2 %0, %1, %2, %3;" : "=l"(d) : "l"(a), "l"(b), "l"(c)); return d; }
__device__ __forceinline__ f2 fadd2(f2 a, f2 b) { f2 d; asm volatile("add.rn.f32x2 %0, %1, %2;" : "=l"(d) : "l"(a), "l"(b)); return d; }

template <int VAR>
__global__ void k(float* out, int iters) {
  f2 ir = pk(threadIdx.x * 1e-3f, 0.5f), ii = pk(0.25f, threadIdx.x * 2e-3f);
  f2 jr[8], jn[8];
  for (int p = 0; p < 8; ++p) { jr[p] = pk(p * 0.1f, 0.3f); jn[p] = pk(-0.2f, p * 0.05f); }
  f2 sim[8]; float sabs[8], mn[8]; unsigned neg[8], nt[8];
  for (int p = 0; p < 8; ++p) { sim[p] = 0; sabs[p] = 0; mn[p] = 1e30f; neg[p] = 0; nt[p] = 0; }
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int p = 0; p < 8; ++p) {
      const f2 tt = ffma2(ii, jr[p], fmul2(ir, jn[p]));
      if (VAR & 1) sim[p] = fadd2(sim[p], tt);
      const float tl = lo(tt), th = hi(tt);
      if (VAR & 2) { sabs[p] += fabsf(tl); sabs[p] += fabsf(th); }
      if (VAR & 4) {
        unsigned r; asm volatile("prmt.b32 %0, %1, %2, 0xFFBB;" : "=r"(r) : "r"(__float_as_uint(tl)), "r"(__float_as_uint(th)));
        if (it & 1) neg[p] += nt[p] + r; else nt[p] = r;
      }
      if (VAR & 8) mn[p] = fminf(mn[p], fminf(fabsf(tl), fabsf(th)));
      if (VAR & 16) { mn[p] = fminf(mn[p], fabsf(tl)); mn[p] = fminf(mn[p], fabsf(th)); }
      if (VAR & 32) {  // integer min over the |t| bit patterns
        unsigned m = __float_as_uint(mn[p]);
        m = min(m, __float_as_uint(tl) & 0x7fffffffu);
        m = min(m, __float_as_uint(th) & 0x7fffffffu);
        mn[p] = __uint_as_float(m);
      }
      if (VAR & 64) {  // packed |t| sum: clear both sign bits, one FADD2
        const f2 at = tt & 0x7fffffff7fffffffull;
        sim[p] = fadd2(sim[p], at);
      }
      if (VAR & 256) {  // guard on t^2 (packed square, plain mins)
        const f2 t2 = fmul2(tt, tt);
        mn[p] = fminf(mn[p], fminf(lo(t2), hi(t2)));
      }
      if (VAR & 512) {  // guard as a flag: any |t| below a per-pair threshold
        const float tau = 1e-7f;
        neg[p] |= (unsigned)(fabsf(tl) < tau) | (unsigned)(fabsf(th) < tau);
      }
      if (VAR & 128) {  // min via packed: min(|tl|,|th|) folded into one chain with FMNMX on the max-free path
        const float m2 = fminf(fabsf(tl), fabsf(th));
        mn[p] = fminf(mn[p], m2);
      }
    }
    ir = fadd2(ir, ii);  // vary the operands
  }
  float s = 0;
  for (int p = 0; p < 8; ++p) s += lo(sim[p]) + hi(sim[p]) + sabs[p] + mn[p] + neg[p];
  if (s == 1.2345f) out[0] = s;
}
template <int VAR>
void run(const char* name) {
  float* d; cudaMalloc(&d, 4);
  const int iters = 20000, nsm = 148, threads = 512;
  k<VAR><<<nsm, threads>>>(d, 100);
  cudaEvent_t a, b; cudaEventCreate(&a); cudaEventCreate(&b);
  cudaEventRecord(a); k<VAR><<<nsm, threads>>>(d, iters); cudaEventRecord(b); cudaEventSynchronize(b);
  float ms; cudaEventElapsedTime(&ms, a, b);
  const double warp_pair_tp = (double)nsm * (threads / 32) * iters * 8;   // per warp: 8 pairs x 1 trial pair per iter
  const double cyc = ms * 1e-3 * 1.965e9 * nsm * 4;                       // SMSP-cycles
  printf("%-32s %.2f SMSP-cycles per warp-pair-trialpair (%s)\n", name, cyc / warp_pair_tp, cudaGetErrorString(cudaGetLastError()));
}
int main() {
  run<0>("t only (FMUL2+FFMA2)");
  run<1>("+ sum t (FADD2)");
  run<3>("+ sum |t| (2 FADD)");
  run<7>("+ sign counts (PRMT, IADD3/2)");
  run<15>("+ min |t| (FMNMX3) = K3 loop");
  run<13>("K3 loop without sum |t|");
  run<7 | 16>("... min as 2 FMNMX");
  run<7 | 32>("... min as integer min on bits");
  run<1 | 4 | 8 | 64>("sum |t| as LOP3 + FADD2 (+ FMNMX3)");
  run<1 | 4 | 32 | 64>("sum |t| packed + integer min");
  run<7 | 128>("... min as FMNMX(FMNMX)");
  run<7 | 256>("... guard on packed t^2");
  run<7 | 512>("... guard as FSETP flags");
  return 0;
}
