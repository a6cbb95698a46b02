// FP64 (DFMA) and FP32 (FFMA) vector throughput on this GPU: the ALU peak the
// off-grid evaluator (fp64 rotation sums, mci_anylen.cu) is measured against.
// Many independent FMA chains per thread, all SMs, CUDA-event timing.
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o f64_throughput.bin f64_throughput.cu
#include <cstdio>
#include <cuda_runtime.h>

template <typename T, int CH>
__global__ void fma_kernel(T *out, int iters, T a, T b) {
    T x[CH];
#pragma unroll
    for (int c = 0; c < CH; ++c) x[c] = (T)(threadIdx.x + c);
    for (int i = 0; i < iters; ++i) {
#pragma unroll
        for (int c = 0; c < CH; ++c) x[c] = fma(x[c], a, b);
    }
    T s = 0;
#pragma unroll
    for (int c = 0; c < CH; ++c) s += x[c];
    out[blockIdx.x * blockDim.x + threadIdx.x] = s;
}

template <typename T> double run(int blocks_per_sm, int threads, int iters) {
    int nsm = 0;
    cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, 0);
    const int blocks = nsm * blocks_per_sm;
    T *out;
    cudaMalloc(&out, sizeof(T) * blocks * threads);
    constexpr int CH = 8;
    fma_kernel<T, CH><<<blocks, threads>>>(out, 10, (T)0.999, (T)0.001);
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0);
    cudaEventCreate(&e1);
    cudaEventRecord(e0);
    fma_kernel<T, CH><<<blocks, threads>>>(out, iters, (T)0.999, (T)0.001);
    cudaEventRecord(e1);
    cudaEventSynchronize(e1);
    float ms = 0;
    cudaEventElapsedTime(&ms, e0, e1);
    cudaFree(out);
    const double flops = 2.0 * CH * (double)iters * blocks * threads;
    return flops / (ms * 1e-3) / 1e12;
}

int main() {
    printf("FP64 DFMA: %.2f TFLOP/s\n", run<double>(4, 256, 20000));
    printf("FP32 FFMA: %.2f TFLOP/s\n", run<float>(4, 256, 40000));
    cudaError_t e = cudaGetLastError();
    printf("status: %s\n", cudaGetErrorString(e));
    return e != cudaSuccess;
}
