// FFMA2 / FADD2 throughput by operand form (register-file operand bandwidth), at 1..4 warps per SM
// sub-partition (the row kernel runs 3 compute warps per sub-partition):
//   A  fma(x64, imm, y64)            two 64-bit register operands + immediate (fused constant twiddles)
//   B  fma(x64, s32 broadcast, y64)  two 64-bit + one 32-bit register (complex multiply, second half)
//   C  fma(x64, y64, z64)            three 64-bit register operands
//   D  add(x64, y64)
//   E  mul(x64, s32 broadcast)       (complex multiply, first half)
// each with index offsets (o1, o2, o3) into a 48-entry register array; offsets of equal parity put all
// operands of an instruction into register pairs of equal parity.
#include <cstdint>
#include <cstdio>
__device__ __forceinline__ uint64_t P(float x, float y) { uint64_t r; asm("mov.b64 %0, {%1, %2};" : "=l"(r) : "f"(x), "f"(y)); return r; }
__device__ __forceinline__ float2 U(uint64_t r) { float2 v; asm("mov.b64 {%0, %1}, %2;" : "=f"(v.x), "=f"(v.y) : "l"(r)); return v; }
__device__ __forceinline__ uint64_t fma2(uint64_t a, uint64_t b, uint64_t c) { uint64_t r; asm volatile("fma.rn.f32x2 %0, %1, %2, %3;" : "=l"(r) : "l"(a), "l"(b), "l"(c)); return r; }
__device__ __forceinline__ uint64_t add2(uint64_t a, uint64_t b) { uint64_t r; asm volatile("add.rn.f32x2 %0, %1, %2;" : "=l"(r) : "l"(a), "l"(b)); return r; }
__device__ __forceinline__ uint64_t mul2(uint64_t a, uint64_t b) { uint64_t r; asm volatile("mul.rn.f32x2 %0, %1, %2;" : "=l"(r) : "l"(a), "l"(b)); return r; }
constexpr int NR = 44;
template <int MODE, int O1, int O2, int O3> __global__ void __launch_bounds__(512, 1) k(float2* out, int iters, float2 s) {
  uint64_t x[NR];
  float sc[4] = {s.x, s.y, s.x + s.y, s.x - s.y};
#pragma unroll
  for (int i = 0; i < NR; ++i) x[i] = P(threadIdx.x * 1e-3f + i, i * 1e-3f);
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int i = 0; i < NR; ++i) {
      const uint64_t a = x[(i + O1) % NR], b = x[(i + O2) % NR], c = x[(i + O3) % NR];
      if (MODE == 0) x[i] = fma2(a, P(0.70710678f, 0.70710678f), c);
      if (MODE == 1) x[i] = fma2(a, P(sc[i & 3], sc[i & 3]), c);
      if (MODE == 2) x[i] = fma2(a, b, c);
      if (MODE == 3) x[i] = add2(a, b);
      if (MODE == 4) x[i] = mul2(a, P(sc[i & 3], sc[i & 3]));
    }
  }
  float2 r = U(x[0]);
#pragma unroll
  for (int i = 1; i < NR; ++i) { float2 q = U(x[i]); r.x += q.x; r.y += q.y; }
  out[blockIdx.x * blockDim.x + threadIdx.x] = r;
}
template <int MODE, int O1, int O2, int O3> void run(const char* name, float2* d) {
  cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
  const int iters = 2000;
  printf("%-34s offsets (%2d,%2d,%2d):", name, O1, O2, O3);
  for (int threads : {128, 384, 512}) {
    float best = 1e9;
    for (int rep = 0; rep < 3; ++rep) {
      cudaEventRecord(e0); k<MODE, O1, O2, O3><<<148, threads>>>(d, iters, make_float2(0.999f, 1e-3f)); cudaEventRecord(e1); cudaEventSynchronize(e1);
      float ms; cudaEventElapsedTime(&ms, e0, e1); if (ms < best) best = ms;
    }
    const double w = (double)(threads / 32) / 4 * iters * NR, cycles = best * 1e-3 * 1.965e9;
    printf("  %dw %.3f", threads / 128, w / cycles);
  }
  printf("  warp-instr/clk/SMSP\n");
}
int main() {
  float2* d; cudaMalloc(&d, 148 * 1024 * sizeof(float2));
  run<0, 5, 11, 17>("A fma(x64, imm, y64)", d);
  run<0, 5, 10, 16>("A fma(x64, imm, y64)", d);
  run<1, 5, 11, 17>("B fma(x64, s32, y64)", d);
  run<1, 5, 10, 16>("B fma(x64, s32, y64)", d);
  run<2, 5, 11, 17>("C fma(x64, y64, z64)", d);
  run<2, 5, 10, 15>("C fma(x64, y64, z64)", d);
  run<2, 5, 10, 16>("C fma(x64, y64, z64)", d);
  run<2, 4, 9, 13>("C fma(x64, y64, z64)", d);
  run<3, 5, 11, 17>("D add(x64, y64)", d);
  run<3, 5, 10, 15>("D add(x64, y64)", d);
  run<4, 5, 11, 17>("E mul(x64, s32)", d);
  return 0;
}
