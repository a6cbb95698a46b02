// Checks the packed (FP32x2) and scalar register codelets against an fp64 DFT.
#include <cstdio>
#include <cmath>
#include <vector>
#include "../../paper_1802_10291_b200/csrc/mci_pk.cuh"
using namespace mci;
template <int R, int DIR> __global__ void kp(const float2* in, float2* out) {
  pkx::pk x[R]; for (int i = 0; i < R; ++i) x[i] = pkx::mk(in[threadIdx.x * R + i]);
  pkx::dft<R, DIR>(x); for (int i = 0; i < R; ++i) out[threadIdx.x * R + i] = pkx::f2(x[i]);
}
template <int R, int DIR> __global__ void ks(const float2* in, float2* out) {
  float2 x[R]; for (int i = 0; i < R; ++i) x[i] = in[threadIdx.x * R + i];
  cl::dft_big<R, DIR>(x); for (int i = 0; i < R; ++i) out[threadIdx.x * R + i] = x[i];
}
template <int R, int DIR> double check(bool packed) {
  const int T = 32; std::vector<float2> h(T * R), o(T * R);
  for (int i = 0; i < T * R; ++i) h[i] = make_float2(std::sin(1.3 * i + 0.2), std::cos(0.7 * i * i + 0.1));
  float2 *din, *dout; cudaMalloc(&din, T * R * 8); cudaMalloc(&dout, T * R * 8);
  cudaMemcpy(din, h.data(), T * R * 8, cudaMemcpyHostToDevice);
  if (packed) kp<R, DIR><<<1, T>>>(din, dout); else ks<R, DIR><<<1, T>>>(din, dout);
  cudaMemcpy(o.data(), dout, T * R * 8, cudaMemcpyDeviceToHost);
  double err = 0, ref = 0;
  for (int t = 0; t < T; ++t) for (int k = 0; k < R; ++k) {
    double re = 0, im = 0;
    for (int n = 0; n < R; ++n) { double a = DIR * 2 * M_PI * n * k / R; re += h[t*R+n].x * cos(a) - h[t*R+n].y * sin(a); im += h[t*R+n].x * sin(a) + h[t*R+n].y * cos(a); }
    err = fmax(err, hypot(o[t*R+k].x - re, o[t*R+k].y - im)); ref = fmax(ref, hypot(re, im));
  }
  cudaFree(din); cudaFree(dout); return err / ref;
}
int main() {
  int bad = 0;
#define C(R, D) { double ep = check<R, D>(true), es = check<R, D>(false); printf("R=%2d DIR=%+d packed %.2e scalar %.2e\n", R, D, ep, es); bad += (ep > 1e-5) + (es > 1e-5); }
  C(4, -1) C(8, -1) C(16, -1) C(32, -1) C(64, -1) C(4, 1) C(8, 1) C(16, 1) C(32, 1) C(64, 1)
  printf(bad ? "CODELET CHECK FAILED\n" : "codelets ok\n");
  return bad;
}
