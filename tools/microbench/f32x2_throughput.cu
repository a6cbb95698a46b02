#include <cstdint>
#include <cstdio>
__device__ __forceinline__ uint64_t P(float x, float y) { uint64_t r; asm("mov.b64 %0, {%1, %2};" : "=l"(r) : "f"(x), "f"(y)); return r; }
__device__ __forceinline__ float2 U(uint64_t r) { float2 v; asm("mov.b64 {%0, %1}, %2;" : "=f"(v.x), "=f"(v.y) : "l"(r)); return v; }
__device__ __forceinline__ uint64_t mul2(uint64_t a, uint64_t b) { uint64_t r; asm("mul.rn.f32x2 %0, %1, %2;" : "=l"(r) : "l"(a), "l"(b)); return r; }
__device__ __forceinline__ uint64_t fma2(uint64_t a, uint64_t b, uint64_t c) { uint64_t r; asm("fma.rn.f32x2 %0, %1, %2, %3;" : "=l"(r) : "l"(a), "l"(b), "l"(c)); return r; }
__global__ void cm2(float2* a, const float2* w) {
  int i = threadIdx.x; float2 x = a[i], t = w[i];
  uint64_t p = mul2(P(t.x, t.y), P(x.x, x.x));
  uint64_t r = fma2(P(t.y, t.x), P(-x.y, x.y), p);
  a[i] = U(r);
}
__global__ void cm3(float2* a, const float2* w) {
  int i = threadIdx.x; float2 x = a[i], t = w[i];
  uint64_t p = mul2(P(x.x, x.x), P(t.x, t.y));
  uint64_t r = fma2(P(x.y, x.y), P(-t.y, t.x), p);
  a[i] = U(r);
}
// throughput microbenchmarks: 8 independent chains
__global__ void bench_ffma2(float2* out, int iters, float2 s) {
  uint64_t acc[8]; uint64_t m = P(s.x, s.y), c = P(s.y, s.x);
  for (int k=0;k<8;++k) acc[k] = P(threadIdx.x + k, k);
  for (int it=0; it<iters; ++it) {
    #pragma unroll
    for (int k=0;k<8;++k) acc[k] = fma2(acc[k], m, c);
  }
  float2 r = U(acc[0]); for (int k=1;k<8;++k){ float2 q=U(acc[k]); r.x+=q.x; r.y+=q.y; }
  out[blockIdx.x*blockDim.x+threadIdx.x] = r;
}
__global__ void bench_ffma(float2* out, int iters, float2 s) {
  float acc[16];
  for (int k=0;k<16;++k) acc[k] = threadIdx.x + k;
  for (int it=0; it<iters; ++it) {
    #pragma unroll
    for (int k=0;k<16;++k) acc[k] = fmaf(acc[k], s.x, s.y + k);
  }
  float r=0; for (int k=0;k<16;++k) r+=acc[k];
  out[blockIdx.x*blockDim.x+threadIdx.x] = make_float2(r, 0);
}
int main() {
  float2* d; cudaMalloc(&d, 148*1024*8*sizeof(float2));
  cudaEvent_t e0,e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
  int iters = 4096;
  for (int rep=0; rep<2; ++rep) {
    cudaEventRecord(e0); bench_ffma<<<148*8, 256>>>(d, iters, make_float2(0.999f, 1e-3f)); cudaEventRecord(e1); cudaEventSynchronize(e1);
    float ms; cudaEventElapsedTime(&ms, e0, e1);
    double lane_ops = 148.0*8*256*iters*16; printf("FFMA : %.3f ms  %.2f Tlane-instr/s  (%.1f TFLOP/s)\n", ms, lane_ops/ms/1e9, 2*lane_ops/ms/1e9);
    cudaEventRecord(e0); bench_ffma2<<<148*8, 256>>>(d, iters, make_float2(0.999f, 1e-3f)); cudaEventRecord(e1); cudaEventSynchronize(e1);
    cudaEventElapsedTime(&ms, e0, e1);
    lane_ops = 148.0*8*256*iters*8; printf("FFMA2: %.3f ms  %.2f Tlane-instr/s  (%.1f TFLOP/s)\n", ms, lane_ops/ms/1e9, 4*lane_ops/ms/1e9);
  }
  return 0;
}
