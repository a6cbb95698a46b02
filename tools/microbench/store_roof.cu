// I/O-only roofline for the config-2 shape: every row reads 3 x 1024 floats and
// writes 16384 floats (65536 rows: 0.8 GB read, 4.3 GB written), with trivial
// arithmetic.  Measures what the HBM system sustains for this write-dominated mix
// under several store schemes; the row kernel's time is judged against it.
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o store_roof.bin store_roof.cu
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>

constexpr int MN = 3072, L = 16384;

// variant 0: float2 streaming stores, 128 threads per row group, CTAs of G groups
template <int G, int VEC>
__global__ void __launch_bounds__(128 * G) io_kernel(const float *__restrict__ g, float *__restrict__ f, int64_t rows) {
    const int grp = threadIdx.x / 128, tid = threadIdx.x % 128;
    for (int64_t row = (int64_t)blockIdx.x * G + grp; row < rows; row += (int64_t)gridDim.x * G) {
        float s = 0.f;
        const float *src = g + row * MN;
#pragma unroll
        for (int j = 0; j < MN / 128; ++j) s += __ldcs(src + tid + 128 * j);
        float *dst = f + row * L;
        if (VEC == 2) {
            float2 *d2 = reinterpret_cast<float2 *>(dst);
#pragma unroll 16
            for (int j = 0; j < L / 256; ++j) __stcs(d2 + tid + 128 * j, make_float2(s + j, s - j));
        } else {
            float4 *d4 = reinterpret_cast<float4 *>(dst);
#pragma unroll 16
            for (int j = 0; j < L / 512; ++j) __stcs(d4 + tid + 128 * j, make_float4(s + j, s - j, s, -s));
        }
    }
}

template <int G, int VEC> float run(const float *g, float *f, int64_t rows, int ctas_per_sm) {
    int nsm = 148;
    cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, 0);
    const int grid = nsm * ctas_per_sm;
    cudaEvent_t a, b;
    cudaEventCreate(&a);
    cudaEventCreate(&b);
    for (int i = 0; i < 3; ++i) io_kernel<G, VEC><<<grid, 128 * G>>>(g, f, rows);
    cudaEventRecord(a);
    const int it = 20;
    for (int i = 0; i < it; ++i) io_kernel<G, VEC><<<grid, 128 * G>>>(g, f, rows);
    cudaEventRecord(b);
    cudaEventSynchronize(b);
    float ms = 0;
    cudaEventElapsedTime(&ms, a, b);
    return ms / it;
}

int main() {
    const int64_t rows = 65536;
    float *g, *f;
    cudaMalloc(&g, rows * MN * 4);
    cudaMalloc(&f, rows * L * 4);
    cudaMemset(g, 0, rows * MN * 4);
    const double bytes = (double)rows * (MN + L) * 4;
    struct { const char *name; float ms; } r[] = {
        {"G=3 float2, 1 CTA/SM (row-kernel shape)", run<3, 2>(g, f, rows, 1)},
        {"G=3 float4, 1 CTA/SM", run<3, 4>(g, f, rows, 1)},
        {"G=2 float2, 1 CTA/SM", run<2, 2>(g, f, rows, 1)},
        {"G=1 float2, 8 CTA/SM", run<1, 2>(g, f, rows, 8)},
        {"G=1 float4, 8 CTA/SM", run<1, 4>(g, f, rows, 8)},
        {"G=1 float4, 16 CTA/SM", run<1, 4>(g, f, rows, 16)},
    };
    for (auto &x : r) printf("%-42s %.3f ms  %.0f GB/s\n", x.name, x.ms, bytes / x.ms / 1e6);
    cudaError_t e = cudaGetLastError();
    printf("status: %s\n", cudaGetErrorString(e));
    return e != cudaSuccess;
}
