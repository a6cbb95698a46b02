// TMEM as a per-thread read-only table: throughput of tcgen05.ld (32x32b) versus
// LDS.128 for the same bytes, with 4, 8 and 12 warps per SM (one CTA per SM).
// Question it answers: can the row kernel's per-thread twiddle tables live in TMEM
// (lane = thread, columns = table entries) instead of shared memory / L1?
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o tmem_ld tmem_ld.cu
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>

__device__ __forceinline__ uint32_t smem_u32(const void *p) { return (uint32_t)__cvta_generic_to_shared(p); }

template <int MODE>  // 0: tcgen05.ld x16 (64 B/thread), 1: 4 x LDS.128 (64 B/thread)
__global__ void bench(float *out, int iters, long long *cyc) {
    __shared__ uint32_t tbase;
    __shared__ __align__(16) float4 tab[128 * 4 * 4 + 8];
    const int warp = threadIdx.x / 32;
    if (warp == 0) {
        asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 512;" ::"r"(smem_u32(&tbase)));
        asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
    }
    for (int i = threadIdx.x; i < 128 * 4 * 4; i += blockDim.x) tab[i] = make_float4(i, 1, 2, 3);
    asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
    __syncthreads();
    asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
    const uint32_t tb = tbase;
    const uint32_t lanebase = (uint32_t)(32 * (warp & 3)) << 16;
    // fill 128 columns of this thread's lane (warps 0-3 only)
    if (warp < 4) {
        for (int c = 0; c < 128; c += 8) {
            uint32_t v[8];
            for (int k = 0; k < 8; ++k) v[k] = __float_as_uint((float)(threadIdx.x + c + k));
            asm volatile("tcgen05.st.sync.aligned.32x32b.x8.b32 [%0], {%1,%2,%3,%4,%5,%6,%7,%8};" ::"r"(tb + lanebase + c),
                         "r"(v[0]), "r"(v[1]), "r"(v[2]), "r"(v[3]), "r"(v[4]), "r"(v[5]), "r"(v[6]), "r"(v[7]));
        }
        asm volatile("tcgen05.wait::st.sync.aligned;" ::: "memory");
    }
    asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
    __syncthreads();
    asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
    float acc = 0.f;
    long long t0 = clock64();
    for (int it = 0; it < iters; ++it) {
        const int c = (it * 16) & 127;
        if (MODE == 0) {
            uint32_t v[16];
            asm volatile(
                "tcgen05.ld.sync.aligned.32x32b.x16.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15}, [%16];"
                : "=r"(v[0]), "=r"(v[1]), "=r"(v[2]), "=r"(v[3]), "=r"(v[4]), "=r"(v[5]), "=r"(v[6]), "=r"(v[7]),
                  "=r"(v[8]), "=r"(v[9]), "=r"(v[10]), "=r"(v[11]), "=r"(v[12]), "=r"(v[13]), "=r"(v[14]), "=r"(v[15])
                : "r"(tb + lanebase + c));
            asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
#pragma unroll
            for (int k = 0; k < 16; ++k) acc += __uint_as_float(v[k]);
        } else {
            const float4 *p = tab + (threadIdx.x & 127) * 4 + ((it & 3) * 512);
            float4 a = p[0], b = p[1], d = p[2], e = p[3];
            acc += a.x + a.y + a.z + a.w + b.x + b.y + b.z + b.w + d.x + d.y + d.z + d.w + e.x + e.y + e.z + e.w;
        }
    }
    long long t1 = clock64();
    asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
    __syncthreads();
    if (warp == 0) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 512;" ::"r"(tb));
    out[blockIdx.x * blockDim.x + threadIdx.x] = acc;
    if (threadIdx.x == 0) cyc[blockIdx.x] = t1 - t0;
}

int main() {
    float *out;
    long long *cyc;
    cudaMalloc(&out, 148 * 1024 * 4);
    cudaMalloc(&cyc, 148 * 8);
    const int iters = 4096;
    for (int mode = 0; mode < 2; ++mode)
        for (int warps = 4; warps <= 16; warps += 4) {
            cudaEvent_t a, b;
            cudaEventCreate(&a);
            cudaEventCreate(&b);
            for (int rep = 0; rep < 2; ++rep) {
                cudaEventRecord(a);
                if (mode == 0) bench<0><<<148, warps * 32>>>(out, iters, cyc);
                else bench<1><<<148, warps * 32>>>(out, iters, cyc);
                cudaEventRecord(b);
                cudaEventSynchronize(b);
            }
            float ms;
            cudaEventElapsedTime(&ms, a, b);
            long long c;
            cudaMemcpy(&c, cyc, 8, cudaMemcpyDeviceToHost);
            const double bytes_per_sm = (double)warps * 32 * 64 * iters;
            printf("%s warps/SM=%2d: %.3f ms, %lld cyc, %.1f B/clk/SM  (%s)\n", mode ? "LDS.128 " : "tcgen05.ld", warps,
                   ms, c, bytes_per_sm / c, cudaGetErrorString(cudaGetLastError()));
        }
    return 0;
}
