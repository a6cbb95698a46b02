// FP32 pipe throughput on B200: FFMA, FADD, FFMA2, FADD2, and mixes (8 independent chains/thread).
#include <cstdint>
#include <cstdio>
__device__ __forceinline__ uint64_t P(float x, float y) { uint64_t r; asm("mov.b64 %0, {%1, %2};" : "=l"(r) : "f"(x), "f"(y)); return r; }
__device__ __forceinline__ float2 U(uint64_t r) { float2 v; asm("mov.b64 {%0, %1}, %2;" : "=f"(v.x), "=f"(v.y) : "l"(r)); return v; }
__device__ __forceinline__ uint64_t fma2(uint64_t a, uint64_t b, uint64_t c) { uint64_t r; asm volatile("fma.rn.f32x2 %0, %1, %2, %3;" : "=l"(r) : "l"(a), "l"(b), "l"(c)); return r; }
__device__ __forceinline__ uint64_t add2(uint64_t a, uint64_t b) { uint64_t r; asm volatile("add.rn.f32x2 %0, %1, %2;" : "=l"(r) : "l"(a), "l"(b)); return r; }
__device__ __forceinline__ float fadd(float a, float b) { float r; asm volatile("add.rn.f32 %0, %1, %2;" : "=f"(r) : "f"(a), "f"(b)); return r; }
__device__ __forceinline__ float ffma(float a, float b, float c) { float r; asm volatile("fma.rn.f32 %0, %1, %2, %3;" : "=f"(r) : "f"(a), "f"(b), "f"(c)); return r; }
template <int MODE> __global__ void k(float* out, int iters, float s) {
  uint64_t p[8]; float q[8];
  uint64_t m = P(s, s * 0.5f), c = P(1e-3f, 2e-3f);
  for (int i = 0; i < 8; ++i) { p[i] = P(threadIdx.x + i, i); q[i] = threadIdx.x * 0.5f + i; }
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int i = 0; i < 8; ++i) {
      if (MODE == 0) q[i] = ffma(q[i], s, 1e-3f);                 // FFMA
      if (MODE == 1) q[i] = fadd(q[i], s);                        // FADD
      if (MODE == 2) p[i] = fma2(p[i], m, c);                     // FFMA2
      if (MODE == 3) p[i] = add2(p[i], c);                        // FADD2
      if (MODE == 4) { p[i] = fma2(p[i], m, c); q[i] = fadd(q[i], s); }  // FFMA2 + FADD
      if (MODE == 5) { p[i] = add2(p[i], c); q[i] = ffma(q[i], s, 1e-3f); }  // FADD2 + FFMA
      if (MODE == 6) { p[i] = fma2(p[i], m, c); p[i] = add2(p[i], c); }  // FFMA2 + FADD2 (dependent)
    }
  }
  float r = 0; for (int i = 0; i < 8; ++i) { float2 v = U(p[i]); r += v.x + v.y + q[i]; }
  out[blockIdx.x * blockDim.x + threadIdx.x] = r;
}
template <int MODE> void run(float* d, const char* name, double ops_per_it) {
  cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
  int iters = 2048;
  k<MODE><<<148 * 8, 256>>>(d, 16, 1.0001f);
  cudaEventRecord(e0); k<MODE><<<148 * 8, 256>>>(d, iters, 1.0001f); cudaEventRecord(e1); cudaEventSynchronize(e1);
  float ms; cudaEventElapsedTime(&ms, e0, e1);
  double warp_instr = 148.0 * 8 * 8 * iters * 8 * ops_per_it;  // warps * iters * chains * instr/chain-iter
  printf("%-16s %.3f ms  %.3f warp-instr/clk/SM @1.9GHz\n", name, ms, warp_instr / (ms * 1e-3) / 148 / 1.9e9);
}
int main() {
  float* d; cudaMalloc(&d, 148 * 8 * 256 * 4);
  for (int rep = 0; rep < 2; ++rep) {
    run<0>(d, "FFMA", 1); run<1>(d, "FADD", 1); run<2>(d, "FFMA2", 1); run<3>(d, "FADD2", 1);
    run<4>(d, "FFMA2+FADD", 2); run<5>(d, "FADD2+FFMA", 2); run<6>(d, "FFMA2+FADD2", 2);
  }
  return 0;
}
