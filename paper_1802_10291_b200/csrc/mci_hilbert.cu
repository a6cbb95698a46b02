// Analytic-output (f and Hf) MCI row kernel for BASELINE.json configs[2]:
// M = 2 channels (f, f'), N = 4096 samples, L = 65536 outputs, fp32.
//
// Mathematics as in mci_fused.cu: forward DFT (Lemma 1),
// per-class solve (Eq. matrixeqn1), Hermitian part, and the
// Hilbert twin through the one-sided analytic spectrum Z(0) = X(0),
// Z(k) = 2 X(k) (Example 4; multiplier -i sgn k,
// PAPER.md:107-116): one complex inverse DFT gives z = f + i Hf.
// Layout: L = R S with S = 4096 = K and R = 16: output phase p1 of p = 16 p2 + p1
// is a 4096-point inverse DFT of Z(k) e^{2 pi i k p1 / L} (k' = k mod S; k' = 0
// also receives k = K).  One CTA (256 threads, 8 warps) per SM owns a row:
//   * forward: one complex 4096-point FFT of (g0 + i g1) on warps 0-1 (radix 64 x 64),
//     channels scaled by exact powers of two;
//   * solve: 2049 classes -> Z[0..K] in shared memory;
//   * two CTAs per row, 2 rounds of 4 FFTs each: lanes 4*tl + c run phase p1 on butterfly
//     t = 8 warp + tl; the pre-twiddle is fused into the first pass's loads;
//     two register radix-64 passes (packed FP32x2), padded buffers;
//   * each quad of lanes writes 16 contiguous bytes of f and of Hf; the two CTAs
//     of a row write the two halves of every 32-byte sector at the same time, so
//     partial sectors merge in L2 instead of being read back from HBM.
#include <cstdint>

#include "mci_internal.h"
#include "mci_pk.cuh"

namespace mci {

namespace hilk {
constexpr int M = 2, N = 4096, S = 4096, K = 4096, L = 65536, R = 16, NT = 256;
constexpr int BUF = S + S / 64 + 4;  // padded FFT buffer (pad6); +4 spreads the 4 FFTs of a half-warp over banks
__device__ __forceinline__ int pad6(int a) { return a + (a >> 6); }
__device__ __forceinline__ float pow2f(int e) { return __int_as_float((127 + e) << 23); }
__device__ __forceinline__ void bar() { __syncthreads(); }
}  // namespace hilk

struct HilbertTables {
    const float2 *Qt;   // [N/2+1][2][2]   H^{-1}/N per class
    const float2 *whi;  // [256]  e^{+2 pi i 256 h / L}
    const float2 *wlo;  // [256]  e^{+2 pi i l / L}
    const float2 *itw;  // [64][64] e^{+2 pi i j t / 4096}  (inverse pass 2; conj for the forward)
};

__global__ void __launch_bounds__(hilk::NT, 1)
    mci_hilbert_kernel(const float *__restrict__ g, float *__restrict__ f, float *__restrict__ hf, int64_t rows,
                       HilbertTables tb) {
    using namespace hilk;
    using namespace pkx;
    extern __shared__ __align__(16) unsigned char smem[];
    float2 *Z = reinterpret_cast<float2 *>(smem);  // K+1 (+pad)
    float2 *bufs = Z + (K + 2);                     // 4 x BUF
    float2 *whi = bufs + 4 * BUF;                   // 256
    float2 *wlo = whi + 256;                        // 256
    float2 *itw = wlo + 256;                        // 4096
    __shared__ float ssc[4];
    for (int i = threadIdx.x; i < 256; i += NT) {
        whi[i] = tb.whi[i];
        wlo[i] = tb.wlo[i];
    }
    for (int i = threadIdx.x; i < 4096; i += NT) itw[i] = tb.itw[i];
    __syncthreads();
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31, tid = threadIdx.x;
    const int c = lane & 3;                 // FFT (phase) within the round
    const int t = 8 * warp + (lane >> 2);   // butterfly index 0..63
    float2 *buf = bufs + c * BUF;

    // Two CTAs (adjacent blockIdx, co-scheduled) share a row: half hh runs phases
    // p1 = 4 hh + c (round 0) and 8 + 4 hh + c (round 1), so every 32-byte sector of
    // f / Hf (8 consecutive phases) is completed by two concurrent rounds.
    const int hh = blockIdx.x & 1;
    for (int64_t row = blockIdx.x >> 1; row < rows; row += gridDim.x >> 1) {
        const float *g0 = g + row * (int64_t)(M * N), *g1 = g0 + N;
        bar();  // previous row done with all buffers
        // ---- forward (warps 0-1): 4096-point FFT of (g0 + i g1), radix 64 x 64, in buffer 0
        if (warp < 2) {
            const int i = tid;  // butterfly 0..63
            pk x[64];
            float m0 = 0.f, m1 = 0.f;
#pragma unroll
            for (int j = 0; j < 64; ++j) {
                const float a = __ldg(g0 + i + 64 * j), b = __ldg(g1 + i + 64 * j);
                m0 = fmaxf(m0, fabsf(a));
                m1 = fmaxf(m1, fabsf(b));
                x[j] = mk(a, b);
            }
#pragma unroll
            for (int o = 16; o; o >>= 1) {
                m0 = fmaxf(m0, __shfl_xor_sync(0xffffffffu, m0, o));
                m1 = fmaxf(m1, __shfl_xor_sync(0xffffffffu, m1, o));
            }
            if (lane == 0) {
                ssc[2 * warp] = m0;
                ssc[2 * warp + 1] = m1;
            }
            asm volatile("bar.sync 1, 64;" ::: "memory");
            m0 = fmaxf(ssc[0], ssc[2]);
            m1 = fmaxf(ssc[1], ssc[3]);
            const int E0 = (__float_as_int(m0) >> 23) & 0xff, E1 = (__float_as_int(m1) >> 23) & 0xff;
            const int e0 = E0 == 0 ? 0 : max(-100, min(100, E0 - 126));
            const int e1 = E1 == 0 ? 0 : max(-100, min(100, E1 - 126));
            const pk sc = mk(pow2f(-e0), pow2f(-e1));
#pragma unroll
            for (int j = 0; j < 64; ++j) x[j] = mul(x[j], sc);
            dft<64, -1>(x);
#pragma unroll
            for (int j = 0; j < 64; ++j) bufs[pad6(64 * i + j)] = f2(x[j]);
            asm volatile("bar.sync 1, 64;" ::: "memory");
#pragma unroll
            for (int j = 0; j < 64; ++j) x[j] = mk(bufs[pad6(i + 64 * j)]);
#pragma unroll
            for (int j = 1; j < 64; ++j) x[j] = pkx::cmul(x[j], pkx::conj(mk(itw[j * 64 + i])));
            dft<64, -1>(x);
#pragma unroll
            for (int j = 0; j < 64; ++j) bufs[pad6(i + 64 * j)] = f2(x[j]);
            if (tid == 0) {
                ssc[0] = 0.5f * pow2f(e0);
                ssc[1] = 0.5f * pow2f(e1);
            }
        }
        bar();
        // ---- solve: j_q = q - N (elements q - N, q); Z(0) = X(0), Z(k) = 2 X(k)
        {
            const float h0 = ssc[0], h1 = ssc[1];
            for (int q = tid; q <= N / 2; q += NT) {
                const pk zq = mk(bufs[pad6(q)]), zm = mk(bufs[pad6((N - q) & (N - 1))]);
                const pk G0 = mul(add(zq, pkx::conj(zm)), bc(h0));
                const pk G1 = mul(rot<-1>(sub(zq, pkx::conj(zm))), bc(h1));
                const float2 *Qq = tb.Qt + q * 4;
                const pk v0 = add(pkx::cmul(G0, mk(__ldg(Qq + 0))), pkx::cmul(G1, mk(__ldg(Qq + 2))));
                const pk v1 = add(pkx::cmul(G0, mk(__ldg(Qq + 1))), pkx::cmul(G1, mk(__ldg(Qq + 3))));
                if (q == 0) {  // elements -N (= -K) and 0
                    Z[0] = make_float2(f2(v1).x, 0.f);
                    Z[K] = f2(pkx::conj(v0));  // 2 * conj(a(-K)) / 2
                } else if (2 * q == N) {  // elements -N/2, N/2
                    Z[N / 2] = f2(add(v1, pkx::conj(v0)));  // 2 * (a + conj a-)/2
                } else {
                    Z[N - q] = f2(mul(pkx::conj(v0), bc(2.f)));
                    Z[q] = f2(mul(v1, bc(2.f)));
                }
            }
        }
        bar();
        // ---- 2 rounds of 4 phases: p1 = 8 r + 4 hh + c
        for (int r = 0; r < 2; ++r) {
            const int p1 = 8 * r + 4 * hh + c;
            pk x[64];
            // pass 1 (Ls = 1): Zin(k') = Z(k') w^{k' p1} (+ Z(K) w^{K p1} at k' = 0), w = e^{2 pi i/L}
#pragma unroll
            for (int j = 0; j < 64; ++j) {
                const int kp = t + 64 * j;
                const int m = (kp * p1) & (L - 1);
                const pk w = pkx::cmul(mk(whi[m >> 8]), mk(wlo[m & 255]));
                x[j] = pkx::cmul(mk(Z[kp]), w);
            }
            if (t == 0) {
                const int m = (K * p1) & (L - 1);
                const pk w = pkx::cmul(mk(whi[m >> 8]), mk(wlo[m & 255]));
                x[0] = add(x[0], pkx::cmul(mk(Z[K]), w));
            }
            dft<64, 1>(x);
            bar();  // previous round's pass-2 loads are done before buffers are rewritten
#pragma unroll
            for (int j = 0; j < 64; ++j) buf[pad6(64 * t + j)] = f2(x[j]);
            bar();
            // pass 2 (Ls = 64)
#pragma unroll
            for (int j = 0; j < 64; ++j) x[j] = mk(buf[pad6(t + 64 * j)]);
#pragma unroll
            for (int j = 1; j < 64; ++j) x[j] = pkx::cmul(x[j], mk(itw[j * 64 + t]));
            dft<64, 1>(x);
            // outputs p = 16 p2 + p1, p2 = t + 64 j: z = f + i Hf
            float *fr = f + row * (int64_t)L + p1, *hr = hf + row * (int64_t)L + p1;
#pragma unroll
            for (int j = 0; j < 64; ++j) {
                const float2 z = f2(x[j]);
                const int64_t o = (int64_t)R * (t + 64 * j);
                fr[o] = z.x;
                hr[o] = z.y;
            }
        }
    }
}

bool hilbert_supported(const Axis1D &ax) {
    return ax.dtype == MCI_F32 && ax.analytic && ax.M == 2 && ax.N == 4096 && ax.L == 65536 && ax.S == 4096;
}

cudaError_t launch_hilbert(const Axis1D &ax, int64_t rows, const void *g, void *f, void *hf, cudaStream_t st,
                           int *n_launches) {
    if (rows <= 0) return cudaSuccess;
    using namespace hilk;
    HilbertTables tb;
    tb.Qt = (const float2 *)ax.Qt;
    const float2 *base = (const float2 *)ax.rowtab;  // [whi 256][wlo 256][itw 4096]
    tb.whi = base;
    tb.wlo = base + 256;
    tb.itw = base + 512;
    const size_t smem = (size_t)(K + 2 + 4 * BUF + 512 + 4096) * 8;
    cudaError_t e = cudaFuncSetAttribute(mci_hilbert_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    if (e != cudaSuccess) return e;
    int dev = 0, nsm = 148;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, dev);
    int64_t grid = nsm & ~1;  // CTA pairs, one row per pair
    if (grid > 2 * rows) grid = 2 * rows;
    if (n_launches) *n_launches += 1;
    mci_hilbert_kernel<<<(unsigned)grid, NT, smem, st>>>((const float *)g, (float *)f, (float *)hf, rows, tb);
    return cudaGetLastError();
}

}  // namespace mci
