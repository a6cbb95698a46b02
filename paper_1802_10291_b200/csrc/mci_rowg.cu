// Row-kernel family for real-output shapes with an S = 4096, R = 4 inverse (L = 16384,
// 2048 < MN <= 4096): (M, N) = (3, 1024) [the config-2 shape, also served by mci_row.cu],
// (4, 1024), (2, 2048) and (5..8, 512).  Same mathematics as mci_fused.cu (Lemma 1 forward DFT
// PAPER.md:180-233, per-class solve a = D H^{-1} Eq. matrixeqn1, Hermitian-part
// assembly, zero-padded inverse of Eq. DFTexpression) and the layout of the
// tuned config-2 kernel (mci_row.cu, its default variant):
//   * persistent CTA = 3 row groups of 128 threads + a store warpgroup that drains each
//     finished row from tensor memory and prefetches input rows into L2 two rows ahead;
//   * forward: the ceil(M/2) channel-pair complex FFTs of length N over all 128 threads of a
//     group (N = 1024: radix 8 x 8 x 16 for two FFTs; N = 2048: radix 16 x 16 x 8 for one;
//     N = 512: radix 8 x 8 x 8 for four, two butterflies per thread), channels scaled to unit
//     range by exact powers of two before packing;
//   * per-class solve, four forms: the paper's Example 2 closed form (M = 3, (1, ik, -k^2)),
//     the derivative bank (ik)^m, m < M, as a Vandermonde system in the shifted nodes lN
//     (binomial shift by j_q, then a constant M x M inverse), the uniformly interleaved delay
//     bank tau_m = 2 pi m / (MN) (time-interleaved sampling: H = W diag(e^{i j tau_m}), so
//     v = DFT_M(G_m e^{-i j tau_m}) / (M N)), or the plan's Q~ table;
//   * Hermitian assembly + pre-twiddle written straight into the two 4096-point inverse
//     inputs (A: phases 0, 1; B: phases 2, 3 = a^2 x A's inputs); with MN = 4096 the edge
//     bins +-K = +-S/2 meet at k' = S/2 and are summed there;
//   * inverse: two register radix-64 passes, lanes 2s / 2s+1 run FFTs A / B on butterfly s.
#include <cstdint>

#include "mci_fft.cuh"
#include "mci_internal.h"
#include "mci_pk.cuh"
#include "mci_sm100.cuh"

#ifndef MCI_ROWG_BALANCED
#define MCI_ROWG_BALANCED 1  // 0: the q = 0 class in a divergent branch of thread 0 (A/B)
#endif

namespace mci {

struct RowGTables {
    const float2 *Qt;     // [(N/2+1)][M][M] H^{-1}/N per class (table mode)
    const float2 *wp;     // [K+1]      e^{+2 pi i p / L}
    const float2 *itw;    // [64][64]   e^{+2 pi i j t / 4096}     (inverse pass 2)
    const float2 *fw3;    // [16][64]   e^{-2 pi i j b / 1024}     (N = 1024 forward pass 3)
    const float2 *fw8;    // [8][8]     e^{-2 pi i j k / 64}       (N = 1024 forward pass 2)
    const float2 *tw256;  // [16][16]   e^{-2 pi i j i / 256}      (N = 2048 forward pass 2)
    const float2 *tw2k;   // [2048]     e^{-2 pi i m / 2048}       (N = 2048 forward pass 3)
    const float *ainv;    // [M][M]     (Vandermonde in lN)^{-1} / N (derivative bank)
    const float2 *tw512;  // [512]      e^{-2 pi i m / 512}        (N = 512 forward pass 3)
};

namespace rowg {
using namespace sm100;
constexpr int NT = 128, S = 4096, L = 16384;
constexpr int BK_TABLE = 0, BK_EX2 = 1, BK_DERIV = 2, BK_DELAY = 3;
__device__ __forceinline__ int swz64(int a) { return a + (a >> 6); }  // inverse buffers, 4096 -> 4160
__device__ __forceinline__ int sw3(int a) { return a ^ ((a >> 3) & 15); }  // N = 1024 forward
__device__ __forceinline__ int sw4(int a) { return a ^ ((a >> 4) & 15); }  // N = 2048 pass-1 output
__device__ __forceinline__ float pow2f(int e) { return __int_as_float((127 + e) << 23); }
// TMEM columns (lane = thread of the group): outputs 0..383, tables from 384.  Pre-twiddles of
// class u of the thread, element l: column base + 8 u + 2 l (one 8-column load per class)
constexpr int TMC_FW8 = 384, TMC_FW3 = 400;  // N = 1024 forward: 16 + 32 columns
constexpr int TMC_F5A = 448, TMC_F5B = 464;  // N = 512 forward pass-2 / pass-3 twiddles: 16 + 16 columns
// columns per class: 8 (M <= 4) or 16 (M <= 8)
template <int M> constexpr int tmc_cpc() { return M <= 2 ? 4 : M <= 4 ? 8 : 16; }
template <int N> constexpr int tmc_wp() { return N == 1024 ? 432 : 384; }
template <int N> constexpr int tmc_wp2() { return N == 1024 ? 464 : 416; }
constexpr int TMC_F2A = 448, TMC_F2B = 480;  // N = 2048 forward pass-2 / pass-3 twiddles: 30 + 28 columns

// inverse pass-1 input k' = t + 64 j is structurally zero when K < k' < S - K
constexpr bool nz(int K, int kp) { return kp <= K || kp >= S - K; }
constexpr unsigned long long zmask(int K) {
    unsigned long long z = 0;
    for (int j = 0; j < 64; ++j) {
        bool any = false;
        for (int t = 0; t < 64; ++t) any = any || nz(K, t + 64 * j);
        if (!any) z |= 1ull << j;
    }
    return z;
}
// C(n, k), n < 8 (Pascal's triangle: no recursion in device code)
__device__ __forceinline__ float binomf(int n, int k) {
    float c = 1.f;
#pragma unroll
    for (int i = 1; i < 8; ++i)
        if (i <= k) c = c * (float)(n - k + i) / (float)i;
    return c;
}
constexpr bool allnz(int K, int j) {
    bool all = true;
    for (int t = 0; t < 64; ++t) all = all && nz(K, t + 64 * j);
    return all;
}
}  // namespace rowg

template <int M_, int N_> struct RowGCfg {
    static constexpr int M = M_, N = N_, S = 4096, L = 16384, K = M * N / 2;
    static constexpr int P = (M + 1) / 2;          // channel-pair FFTs in the forward
    static constexpr int PF = N == 512 ? 4 : N == 1024 ? 2 : 1;  // forward FFTs computed (P of them carry data)
    static constexpr int QPT = N / 256;            // classes q = tid + 128 u (u < QPT) per thread
    static constexpr int EPT = QPT * M;            // emitted spectrum positions per thread
    static constexpr int BUF_ELEMS = S + S / 64;   // 4160
    static constexpr int GROUP_BYTES = (2 * BUF_ELEMS + 8) * 8;
    static constexpr int ITW_BYTES = (31 * 128 + 64) * 8;  // inverse pass-2 twiddles, paired
    static constexpr int SMEM = 3 * GROUP_BYTES + ITW_BYTES;
    static constexpr int THREADS = 4 * 128;
    static_assert(P * N <= 2048, "forward spectra fit in half a buffer");
    static_assert(K > 1024 && K <= 2048, "S = next_pow2(2K) = 4096");
    static_assert(P <= PF, "channel pairs per forward");
    static_assert(rowg::tmc_cpc<M>() * QPT <= 32, "pre-twiddle tables: TMEM columns");
};

template <int M, int N, int BK>
__global__ void __launch_bounds__(512, 1)
    mci_rowg_kernel(const float *__restrict__ g, float *__restrict__ f, int64_t rows, RowGTables tb) {
    using namespace rowg;
    using namespace pkx;
    using C = RowGCfg<M, N>;
    constexpr int K = C::K, P = C::P, QPT = C::QPT, EPT = C::EPT, G = 3;
    extern __shared__ __align__(128) unsigned char smem[];
    __shared__ float smx[G][4][4];  // per-warp channel maxima (at most four channels per warp)
    __shared__ uint32_t tm_base;
    auto tm_full = [&](int gg) { return reinterpret_cast<uint64_t *>(smem + gg * C::GROUP_BYTES + C::BUF_ELEMS * 8); };
    auto tm_empty = [&](int gg) { return tm_full(gg) + 1; };

    const int grp = threadIdx.x / NT;
    const int tid = threadIdx.x % NT;
    const int warp = tid >> 5, lane = tid & 31;
    const int barid = 1 + grp;
    float2 *bufA = reinterpret_cast<float2 *>(smem + (grp < G ? grp : 0) * C::GROUP_BYTES);
    float2 *bufB = bufA + C::BUF_ELEMS + 8;
    // inverse pass-2 twiddles w_j(t), j = 1..63, paired for 128-bit loads:
    // itwp[128 p + 2 t + h] = w_{2p+1+h}(t) (p < 31), itwp[3968 + t] = w_63(t)
    float2 *itwp = reinterpret_cast<float2 *>(smem + G * C::GROUP_BYTES);

    // ---- one-time setup: TMEM (outputs + per-lane tables), shared twiddles, barriers
    if (threadIdx.x < 32) tm_alloc<512>(&tm_base);
    asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
    __syncthreads();
    asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
    if (threadIdx.x < NT) {  // group 0 writes lane tid of the tables (shared by the three groups)
        const int tt = threadIdx.x;
        const uint32_t ta = tm_base + ((uint32_t)(32 * (tt >> 5)) << 16);
        float v[8];
        if constexpr (N == 1024) {
#pragma unroll 1
            for (int c = 0; c < 16; c += 8) {  // forward pass-2 twiddles (radix 8, Ls = 8)
#pragma unroll
                for (int i = 0; i < 4; ++i) {
                    const int j = 1 + c / 2 + i;
                    const float2 w = j <= 7 ? tb.fw8[j * 8 + (tt & 7)] : make_float2(0.f, 0.f);
                    v[2 * i] = w.x;
                    v[2 * i + 1] = w.y;
                }
                tm_st8(ta + TMC_FW8 + c, v);
            }
#pragma unroll 1
            for (int c = 0; c < 32; c += 8) {  // forward pass-3 twiddles (radix 16, Ls = 64)
#pragma unroll
                for (int i = 0; i < 4; ++i) {
                    const int j = 1 + c / 2 + i;
                    const float2 w = j <= 15 ? tb.fw3[j * 64 + (tt & 63)] : make_float2(0.f, 0.f);
                    v[2 * i] = w.x;
                    v[2 * i + 1] = w.y;
                }
                tm_st8(ta + TMC_FW3 + c, v);
            }
        }
#pragma unroll 1
        for (int u = 0; u < QPT; ++u) {  // pre-twiddles a = e^{2 pi i p/L} of class u, element l, and a^2
#pragma unroll 1
            for (int l0 = 0; l0 < tmc_cpc<M>() / 2; l0 += 4) {  // four entries (two when M <= 2)
                float v2[8];
#pragma unroll
                for (int i = 0; i < 4; ++i) {
                    const int l = l0 + i;
                    const int q = tt + 128 * u;
                    const int jq = -K + ((q + K) % N);
                    int p = jq + l * N;
                    p = p < 0 ? -p : p;
                    double sn = 0, cs = 0, sn2 = 0, cs2 = 0;
                    if (l < M) {
                        sincospi(2.0 * p / L, &sn, &cs);
                        sincospi(4.0 * p / L, &sn2, &cs2);
                    }
                    v[2 * i] = (float)cs;
                    v[2 * i + 1] = (float)sn;
                    v2[2 * i] = (float)cs2;
                    v2[2 * i + 1] = (float)sn2;
                }
                if constexpr (tmc_cpc<M>() == 4) {
                    tm_st4(ta + tmc_wp<N>() + 4 * u, v);
                    tm_st4(ta + tmc_wp2<N>() + 4 * u, v2);
                } else {
                    tm_st8(ta + tmc_wp<N>() + tmc_cpc<M>() * u + 2 * l0, v);
                    tm_st8(ta + tmc_wp2<N>() + tmc_cpc<M>() * u + 2 * l0, v2);
                }
            }
        }
        if constexpr (N == 2048) {  // forward twiddles: pass 2 w256^{(tt % 16) j}, j = 1..15; pass 3
                                    // w2048^{bb j}, bb = tt, tt + 128, j = 1..7
            float va[8], vb[8];
#pragma unroll 1
            for (int c = 0; c < 32; c += 8) {
#pragma unroll
                for (int i = 0; i < 4; ++i) {
                    const int j = 1 + c / 2 + i;                 // pass 2: entries j - 1 = 0..14
                    const float2 wa = j <= 15 ? tb.tw256[16 * j + (tt & 15)] : make_float2(0.f, 0.f);
                    const int e = c / 2 + i, hh = e / 7, jb = 1 + e % 7;  // pass 3: entries 7 hh + jb - 1
                    const float2 wb = e < 14 ? tb.tw2k[(tt + 128 * hh) * jb] : make_float2(0.f, 0.f);
                    va[2 * i] = wa.x;
                    va[2 * i + 1] = wa.y;
                    vb[2 * i] = wb.x;
                    vb[2 * i + 1] = wb.y;
                }
                tm_st8(ta + TMC_F2A + c, va);
                tm_st8(ta + TMC_F2B + c, vb);
            }
        }
        if constexpr (N == 512) {  // forward twiddles of butterfly bf = tt % 64, j = 1..7
            float va[8], vb[8];
#pragma unroll 1
            for (int c = 0; c < 16; c += 8) {
#pragma unroll
                for (int i = 0; i < 4; ++i) {
                    const int j = 1 + c / 2 + i;
                    const float2 wa = j <= 7 ? tb.fw8[j * 8 + (tt & 7)] : make_float2(0.f, 0.f);
                    const float2 wb = j <= 7 ? tb.tw512[(tt & 63) * j] : make_float2(0.f, 0.f);
                    va[2 * i] = wa.x;
                    va[2 * i + 1] = wa.y;
                    vb[2 * i] = wb.x;
                    vb[2 * i + 1] = wb.y;
                }
                tm_st8(ta + TMC_F5A + c, va);
                tm_st8(ta + TMC_F5B + c, vb);
            }
        }
        asm volatile("tcgen05.wait::st.sync.aligned;" ::: "memory");
    }
    for (int i = threadIdx.x; i < 31 * 128 + 64; i += 4 * NT) {
        const int pp = i >> 7, r = i & 127;
        itwp[i] = i < 31 * 128 ? tb.itw[(2 * pp + 1 + (r & 1)) * 64 + (r >> 1)] : tb.itw[63 * 64 + (i - 31 * 128)];
    }
    if (threadIdx.x < G) {
        mbar_init(tm_full(threadIdx.x), NT);
        mbar_init(tm_empty(threadIdx.x), NT);
    }
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
    __syncthreads();
    asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
    const uint32_t tmA = tm_base + ((uint32_t)(32 * warp) << 16);
    const int64_t gstride = (int64_t)gridDim.x * G;
    const int h = lane & 1;                     // inverse: even lanes FFT A, odd lanes FFT B
    const int t = 16 * warp + (lane >> 1);      // inverse butterfly of this lane pair

    if (grp == G) {
        // ---- store warpgroup: drains each group's row from TMEM (column 128 g + 2 j, 2 j + 1 =
        //      output j of the computing lane) and prefetches input rows two rows ahead into L2
        asm volatile("setmaxnreg.dec.sync.aligned.u32 32;" ::: "memory");
        auto l2pf = [&](int64_t r) {
            if (r < rows && tid < M * N * 4 / 128)
                asm volatile("prefetch.global.L2::evict_last [%0];" ::"l"(g + r * (int64_t)(M * N) + 32 * tid));
        };
        for (int gg = 0; gg < G; ++gg) l2pf((int64_t)blockIdx.x * G + gg + gstride);
        for (int64_t it = 0;; ++it) {
            bool any = false;
#pragma unroll 1
            for (int gg = 0; gg < G; ++gg) {
                const int64_t r = (int64_t)blockIdx.x * G + gg + it * gstride;
                if (r >= rows) continue;
                any = true;
                mbar_wait(tm_full(gg), (uint32_t)(it & 1));
                asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
                float2 *fo = reinterpret_cast<float2 *>(f + r * (int64_t)L);
#pragma unroll 1
                for (int c = 0; c < 16; ++c) {
                    float2 w[4];
                    tm_ld8(tmA + 128 * gg + 8 * c, w);
#pragma unroll
                    for (int i = 0; i < 4; ++i) __stcs(fo + 2 * (t + 64 * (4 * c + i)) + h, w[i]);
#ifndef MCI_ROWG_NOSLEEP
                    __nanosleep(32);  // paced drain, as in mci_row.cu
#endif
                }
                asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
                mbar_arrive(tm_empty(gg));
                l2pf(r + 2 * gstride);
            }
            if (!any) break;
        }
    } else {
        asm volatile("setmaxnreg.inc.sync.aligned.u32 160;" ::: "memory");
        uint32_t opar = 0;
        // forward spectrum of channel pair c at bin q (natural order, per-N layout)
        auto spec = [&](int c, int q) -> float2 {
            if constexpr (N == 1024) return bufB[c * 1024 + sw3(q)];
            else if constexpr (N == 512) return bufB[sw3(c * 512 + q)];
            else return bufB[q];
        };
        for (int64_t row = (int64_t)blockIdx.x * G + grp; row < rows; row += gstride) {
            const float *src = g + row * (int64_t)(M * N);
            int e[8] = {0, 0, 0, 0, 0, 0, 0, 0};
            // ---- forward
            if constexpr (N == 1024) {
                // two 1024-point FFTs, channel pairs (g0, g1), (g2, g3 or 0): radix 8 x 8 x 16
                const int b = tid;
                {
                    pk x0[8], x1[8];
                    float mx[4] = {0.f, 0.f, 0.f, 0.f};
#pragma unroll
                    for (int j = 0; j < 8; ++j) {
                        float a[4] = {0.f, 0.f, 0.f, 0.f};
#pragma unroll
                        for (int m = 0; m < M; ++m) a[m] = __ldcs(src + m * N + b + 128 * j);
                        x0[j] = mk(a[0], a[1]);
                        x1[j] = mk(a[2], a[3]);
#pragma unroll
                        for (int m = 0; m < 4; ++m) mx[m] = fmaxf(mx[m], fabsf(a[m]));
                    }
#pragma unroll
                    for (int m = 0; m < M; ++m) mx[m] = warp_max_nonneg(mx[m]);
                    if (lane == 0)
#pragma unroll
                        for (int m = 0; m < M; ++m) smx[grp][warp][m] = mx[m];
                    group_bar<NT>(barid);  // maxima visible; previous row's reads of buffers A/B complete
#pragma unroll
                    for (int m = 0; m < M; ++m) {
                        const float mm = fmaxf(fmaxf(smx[grp][0][m], smx[grp][1][m]), fmaxf(smx[grp][2][m], smx[grp][3][m]));
                        const int E = (__float_as_int(mm) >> 23) & 0xff;
                        e[m] = E == 0 ? 0 : max(-100, min(100, E - 126));
                    }
                    const pk sc0 = mk(pow2f(-e[0]), pow2f(-e[1])), sc1 = mk(pow2f(-e[2]), pow2f(-e[3]));
#pragma unroll
                    for (int j = 0; j < 8; ++j) {
                        x0[j] = pkx::mul(x0[j], sc0);
                        x1[j] = pkx::mul(x1[j], sc1);
                    }
                    dft<8, -1>(x0);
                    dft<8, -1>(x1);
#pragma unroll
                    for (int j = 0; j < 8; ++j) {
                        bufB[sw3(8 * b + j)] = f2(x0[j]);
                        bufB[1024 + sw3(8 * b + j)] = f2(x1[j]);
                    }
                }
                group_bar<NT>(barid);
                {  // pass 2: radix 8, Ls = 8, B -> A
                    const int k = b & 7;
                    float2 w8[8];
                    tm_ld16(tmA + TMC_FW8, w8);
#pragma unroll
                    for (int c = 0; c < 2; ++c) {
                        pk x[8];
#pragma unroll
                        for (int j = 0; j < 8; ++j) x[j] = mk(bufB[c * 1024 + sw3(b + 128 * j)]);
#pragma unroll
                        for (int j = 1; j < 8; ++j) x[j] = pkx::cmul(x[j], mk(w8[j - 1]));
                        dft<8, -1>(x);
#pragma unroll
                        for (int j = 0; j < 8; ++j) bufA[c * 1024 + sw3(8 * (b - k) + k + 8 * j)] = f2(x[j]);
                    }
                }
                group_bar<NT>(barid);
                {  // pass 3: radix 16, Ls = 64, A -> B; FFT c = tid / 64
                    const int c = tid >> 6, bb = tid & 63;
                    pk x[16];
#pragma unroll
                    for (int j = 0; j < 16; ++j) x[j] = mk(bufA[c * 1024 + sw3(bb + 64 * j)]);
                    float2 w3[16];
                    tm_ld16(tmA + TMC_FW3, w3);
                    tm_ld16(tmA + TMC_FW3 + 16, w3 + 8);
#pragma unroll
                    for (int j = 1; j < 16; ++j) x[j] = pkx::cmul(x[j], mk(w3[j - 1]));
                    dft<16, -1>(x);
#pragma unroll
                    for (int j = 0; j < 16; ++j) bufB[c * 1024 + sw3(bb + 64 * j)] = f2(x[j]);
                }
                group_bar<NT>(barid);
            } else if constexpr (N == 512) {
                // four 512-point FFTs, channel pairs (g0, g1) .. (g6, g7) (missing channels 0):
                // radix 8 x 8 x 8 (Stockham), thread b runs butterfly bf = b % 64 of FFTs
                // c = b / 64 and c + 2; buffer slot sw3(512 c + a) (brute-force checked conflict-free)
                const int bf = tid & 63, c0 = tid >> 6;
                {  // pass 1: Ls = 1, inputs bf + 64 j
                    pk x[2][8];
                    float mx[8] = {0.f, 0.f, 0.f, 0.f, 0.f, 0.f, 0.f, 0.f};
#pragma unroll
                    for (int i = 0; i < 2; ++i) {
                        const int c = c0 + 2 * i;
#pragma unroll
                        for (int j = 0; j < 8; ++j) {
                            const float a0 = 2 * c < M ? __ldcs(src + (2 * c) * N + bf + 64 * j) : 0.f;
                            const float a1 = 2 * c + 1 < M ? __ldcs(src + (2 * c + 1) * N + bf + 64 * j) : 0.f;
                            x[i][j] = mk(a0, a1);
                            mx[2 * i] = fmaxf(mx[2 * i], fabsf(a0));
                            mx[2 * i + 1] = fmaxf(mx[2 * i + 1], fabsf(a1));
                        }
                    }
                    // lanes of a warp share c0 (warps 0-1: c0 = 0, warps 2-3: c0 = 1): per-warp maxima
                    // of channels 2 c0, 2 c0 + 1, 2 c0 + 4, 2 c0 + 5
#pragma unroll
                    for (int m = 0; m < 4; ++m) mx[m] = warp_max_nonneg(mx[m]);
                    if (lane == 0)
#pragma unroll
                        for (int m = 0; m < 4; ++m) smx[grp][warp][m] = mx[m];
                    group_bar<NT>(barid);
#pragma unroll
                    for (int m = 0; m < M; ++m) {  // channel m: pair c = m / 2, held by warps with c0 = c % 2
                        const int c = m >> 1, w0 = 2 * (c & 1), slot = 2 * (c >> 1) + (m & 1);
                        const float mm = fmaxf(smx[grp][w0][slot], smx[grp][w0 + 1][slot]);
                        const int E = (__float_as_int(mm) >> 23) & 0xff;
                        e[m] = E == 0 ? 0 : max(-100, min(100, E - 126));
                    }
#pragma unroll
                    for (int i = 0; i < 2; ++i) {
                        const int c = c0 + 2 * i;
                        int ea = 0, eb = 0;
#pragma unroll
                        for (int m = 0; m < M; ++m) {
                            if (m == 2 * c) ea = e[m];
                            if (m == 2 * c + 1) eb = e[m];
                        }
                        const pk sc = mk(pow2f(-ea), pow2f(-eb));
#pragma unroll
                        for (int j = 0; j < 8; ++j) x[i][j] = pkx::mul(x[i][j], sc);
                        dft<8, -1>(x[i]);
#pragma unroll
                        for (int k = 0; k < 8; ++k) bufB[sw3(512 * c + 8 * bf + k)] = f2(x[i][k]);
                    }
                }
                group_bar<NT>(barid);
                {  // pass 2: Ls = 8, twiddle w64^{(bf % 8) j}, B -> A
                    const int k8 = bf & 7;
                    float2 w8[8];
                    tm_ld16(tmA + TMC_F5A, w8);
#pragma unroll
                    for (int i = 0; i < 2; ++i) {
                        const int c = c0 + 2 * i;
                        pk x[8];
#pragma unroll
                        for (int j = 0; j < 8; ++j) x[j] = mk(bufB[sw3(512 * c + bf + 64 * j)]);
#pragma unroll
                        for (int j = 1; j < 8; ++j) x[j] = pkx::cmul(x[j], mk(w8[j - 1]));
                        dft<8, -1>(x);
#pragma unroll
                        for (int k = 0; k < 8; ++k) bufA[sw3(512 * c + 64 * (bf >> 3) + k8 + 8 * k)] = f2(x[k]);
                    }
                }
                group_bar<NT>(barid);
                {  // pass 3: Ls = 64, twiddle w512^{bf j}, natural-order outputs bf + 64 k -> B
                    float2 w9[8];
                    tm_ld16(tmA + TMC_F5B, w9);
#pragma unroll
                    for (int i = 0; i < 2; ++i) {
                        const int c = c0 + 2 * i;
                        pk x[8];
#pragma unroll
                        for (int j = 0; j < 8; ++j) x[j] = mk(bufA[sw3(512 * c + bf + 64 * j)]);
#pragma unroll
                        for (int j = 1; j < 8; ++j) x[j] = pkx::cmul(x[j], mk(w9[j - 1]));
                        dft<8, -1>(x);
#pragma unroll
                        for (int k = 0; k < 8; ++k) bufB[sw3(512 * c + bf + 64 * k)] = f2(x[k]);
                    }
                }
                group_bar<NT>(barid);
            } else {
                // one 2048-point FFT of the channel pair (g0, g1): radix 16 x 16 x 8 (Stockham)
                const int b = tid;
                {  // pass 1: radix 16, Ls = 1: inputs b + 128 j -> B[sw4(16 b + k)]
                    pk x[16];
                    float mx[2] = {0.f, 0.f};
#pragma unroll
                    for (int j = 0; j < 16; ++j) {
                        const float a0 = __ldcs(src + b + 128 * j), a1 = __ldcs(src + N + b + 128 * j);
                        x[j] = mk(a0, a1);
                        mx[0] = fmaxf(mx[0], fabsf(a0));
                        mx[1] = fmaxf(mx[1], fabsf(a1));
                    }
#pragma unroll
                    for (int m = 0; m < 2; ++m) mx[m] = warp_max_nonneg(mx[m]);
                    if (lane == 0) {
                        smx[grp][warp][0] = mx[0];
                        smx[grp][warp][1] = mx[1];
                    }
                    group_bar<NT>(barid);
#pragma unroll
                    for (int m = 0; m < 2; ++m) {
                        const float mm = fmaxf(fmaxf(smx[grp][0][m], smx[grp][1][m]), fmaxf(smx[grp][2][m], smx[grp][3][m]));
                        const int E = (__float_as_int(mm) >> 23) & 0xff;
                        e[m] = E == 0 ? 0 : max(-100, min(100, E - 126));
                    }
                    const pk sc = mk(pow2f(-e[0]), pow2f(-e[1]));
#pragma unroll
                    for (int j = 0; j < 16; ++j) x[j] = pkx::mul(x[j], sc);
                    dft<16, -1>(x);
#pragma unroll
                    for (int k = 0; k < 16; ++k) bufB[sw4(16 * b + k)] = f2(x[k]);
                }
                group_bar<NT>(barid);
                {  // pass 2: radix 16, Ls = 16: inputs B[sw4(b + 128 j)], twiddle w256^{(b % 16) j}
                    const int i = b & 15;
                    pk x[16];
#pragma unroll
                    for (int j = 0; j < 16; ++j) x[j] = mk(bufB[sw4(b + 128 * j)]);
                    float2 w2[16];
                    tm_ld16(tmA + TMC_F2A, w2);
                    tm_ld16(tmA + TMC_F2A + 16, w2 + 8);
#pragma unroll
                    for (int j = 1; j < 16; ++j) x[j] = pkx::cmul(x[j], mk(w2[j - 1]));
                    dft<16, -1>(x);
#pragma unroll
                    for (int k = 0; k < 16; ++k) bufA[(b >> 4) * 256 + i + 16 * k] = f2(x[k]);
                }
                group_bar<NT>(barid);
                {  // pass 3: radix 8, Ls = 256: butterflies b, b + 128; inputs A[bb + 256 j],
                   // twiddle w2048^{bb j}; natural-order outputs bb + 256 k -> B
                    float2 w3[16];
                    tm_ld16(tmA + TMC_F2B, w3);
                    tm_ld16(tmA + TMC_F2B + 16, w3 + 8);
#pragma unroll
                    for (int hh = 0; hh < 2; ++hh) {
                        const int bb = b + 128 * hh;
                        pk x[8];
#pragma unroll
                        for (int j = 0; j < 8; ++j) x[j] = mk(bufA[bb + 256 * j]);
#pragma unroll
                        for (int j = 1; j < 8; ++j) x[j] = pkx::cmul(x[j], mk(w3[7 * hh + j - 1]));
                        dft<8, -1>(x);
#pragma unroll
                        for (int k = 0; k < 8; ++k) bufB[bb + 256 * k] = f2(x[k]);
                    }
                }
                group_bar<NT>(barid);
            }

            // ---- solve: classes q = tid + 128 u (0 < q < N/2) and the self-mirror classes
            //      q = 0 (u = 0 of thread 0) and q = N/2 (thread 0)
            constexpr int QS_TID = 64;  // the thread (warp 2) that solves the q* = N/2 class
            pk zq[QPT + 1][P], zm[QPT + 1][P];
#pragma unroll
            for (int u = 0; u <= QPT; ++u) {
                const int q = u < QPT ? tid + 128 * u : N / 2;
                const int qm = (N - q) & (N - 1);
                if (u < QPT || tid == QS_TID) {
#pragma unroll
                    for (int c = 0; c < P; ++c) {
                        zq[u][c] = mk(spec(c, q));
                        zm[u][c] = mk(spec(c, qm));
                    }
                }
            }
            float hs[8];  // 2^e_m / 2 (the 1/2 of the channel-pair unpacking folded in)
#pragma unroll
            for (int m = 0; m < M; ++m) hs[m] = 0.5f * pow2f(e[m]);
            group_bar<NT>(barid);  // forward spectra read: buffer B may now be overwritten

            // FFT B's inputs are a^2 times FFT A's: P2 + i P3 = a^2 (X + i P1), and the mirrored
            // conj(P2) + i conj(P3) = conj(a^2) (conj X + i conj P1)
            auto emit = [&](int p, pk X, float2 wa, float2 wa2) {
                const pk P1 = pkx::cmul(X, mk(wa));
                const pk a2 = mk(wa2);
                const pk A = add_rot<1>(X, P1);
                if constexpr (K == S / 2) {
                    if (p == S / 2) {  // +-S/2 (MN = 4096 edge) meet at k' = S/2: one slot, both terms
                        const pk Am = add_rot<1>(pkx::conj(X), pkx::conj(P1));
                        bufA[swz64(p)] = f2(add(A, Am));
                        bufB[swz64(p)] = f2(add(pkx::cmul(A, a2), pkx::cmul(Am, pkx::conj(a2))));
                        return;
                    }
                }
                bufA[swz64(p)] = f2(A);
                bufB[swz64(p)] = f2(pkx::cmul(A, a2));
                if (p > 0) {
                    const pk Am = add_rot<1>(pkx::conj(X), pkx::conj(P1));
                    bufA[swz64(S - p)] = f2(Am);
                    bufB[swz64(S - p)] = f2(pkx::cmul(Am, pkx::conj(a2)));
                }
            };
            auto solve = [&](const pk *zqu, const pk *zmu, int q, pk *v) {
                // channel-pair unpacking: G_{2c} = (Z[q] + conj Z[-q])/2, G_{2c+1} = (Z[q] - conj Z[-q])/(2i)
                pk G[M];
#pragma unroll
                for (int c = 0; c < P; ++c) {
                    G[2 * c] = pkx::mul(add(zqu[c], pkx::conj(zmu[c])), bc(hs[2 * c]));
                    if (2 * c + 1 < M) G[2 * c + 1] = pkx::mul(rot<-1>(sub(zqu[c], pkx::conj(zmu[c]))), bc(hs[2 * c + 1]));
                }
                const int jq = -K + ((q + K) % N);
                if constexpr (BK == BK_EX2) {
                    // Example 2, paper's L = N, n = j_q, divided by N: exact in fp32
                    const float n = (float)jq, Nf = (float)N;
                    const float d2 = 1.f / (2.f * Nf * Nf * Nf), d1 = 1.f / (Nf * Nf * Nf);
                    const float r0[3] = {(2.f * Nf * Nf + 3.f * Nf * n + n * n) * d2, -(n * (2.f * Nf + n)) * d1,
                                         (n * (Nf + n)) * d2};
                    const float r1[3] = {(3.f * Nf + 2.f * n) * d2, -2.f * (Nf + n) * d1, (Nf + 2.f * n) * d2};
                    const float r2[3] = {-d2, d1, -d2};
                    const pk ig1 = rot<1>(G[1]);
#pragma unroll
                    for (int l = 0; l < 3; ++l)
                        v[l] = pkx::fma(G[2], bc(r2[l]), pkx::fma(ig1, bc(r1[l]), pkx::mul(G[0], bc(r0[l]))));
                } else if constexpr (BK == BK_DERIV) {
                    // sum_l v_l (i x_l)^m = G_m/N with x_l = j_q + lN: e_m = i^-m G_m; in the shifted
                    // nodes u_l = lN the moments are f_r = sum_m C(r,m) (-j_q)^(r-m) e_m, and
                    // v = W^-1 f with W[r][l] = (lN)^r (tb.ainv = W^-1 / N, row l)
                    pk ev[M];
#pragma unroll
                    for (int m = 0; m < M; ++m) {
                        const int r4 = m & 3;  // i^-m: 1, -i, -1, i
                        ev[m] = r4 == 0 ? G[m] : r4 == 1 ? rot<-1>(G[m]) : r4 == 2 ? pkx::mul(G[m], bc(-1.f)) : rot<1>(G[m]);
                    }
                    float pw[M];  // (-j)^k
                    pw[0] = 1.f;
#pragma unroll
                    for (int k = 1; k < M; ++k) pw[k] = pw[k - 1] * (float)(-jq);
                    pk fr[M];
#pragma unroll
                    for (int r = 0; r < M; ++r) {  // f_r = sum_{m <= r} C(r, m) (-j)^(r-m) e_m
                        pk acc = ev[r];
#pragma unroll
                        for (int m = 0; m < r; ++m) acc = pkx::fma(ev[m], bc(binomf(r, m) * pw[r - m]), acc);
                        fr[r] = acc;
                    }
#pragma unroll
                    for (int l = 0; l < M; ++l) {
                        pk acc = pkx::mul(fr[0], bc(__ldg(tb.ainv + l * M)));
#pragma unroll
                        for (int r = 1; r < M; ++r) acc = pkx::fma(fr[r], bc(__ldg(tb.ainv + l * M + r)), acc);
                        v[l] = acc;
                    }
                } else if constexpr (BK == BK_DELAY) {
                    // H_j = W diag(e^{i j tau_m}), W[l][m] = e^{2 pi i l m / M}, tau_m = 2 pi m / (M N):
                    // v_l = sum_m (G_m / N) e^{-i j tau_m} e^{-2 pi i l m / M} / M
                    const int r = ((jq % (M * N)) + M * N) % (M * N);  // j mod MN: exact phase
                    float sn, cs;
                    sincospif(-2.f * (float)r / (float)(M * N), &sn, &cs);
                    const pk w1 = mk(cs, sn);
                    pk u[M];
                    pk wm = w1;
                    const float sc = 1.f / (float)(M * N);
                    u[0] = pkx::mul(G[0], bc(sc));
#pragma unroll
                    for (int m = 1; m < M; ++m) {
                        u[m] = pkx::mul(pkx::cmul(G[m], wm), bc(sc));
                        if (m + 1 < M) wm = pkx::cmul(wm, w1);
                    }
                    if constexpr (M == 8 || M == 4 || M == 2) {
                        dft<M, -1>(u);
#pragma unroll
                        for (int l = 0; l < M; ++l) v[l] = u[l];
                    }
                } else {
                    const float2 *Qq = tb.Qt + (int64_t)q * M * M;
#pragma unroll
                    for (int l = 0; l < M; ++l) {
                        pk acc = pkx::cmul(G[0], mk(__ldg(Qq + l)));
#pragma unroll
                        for (int m = 1; m < M; ++m) acc = add(acc, pkx::cmul(G[m], mk(__ldg(Qq + m * M + l))));
                        v[l] = acc;
                    }
                }
            };
            // self-mirror class (q = 0 or N/2, thread 0): X[p] = (a(p) + conj a(-p))/2 within the
            // class (a = 0 out of band; p = 0 gives Re a(0); the edge -K gives X[K] = conj a(-K)/2)
            // (q is a compile-time constant: every p below is a multiple of N/2, so the pre-twiddle
            // e^{2 pi i p / L} and its square are compile-time 64th roots instead of table loads on the
            // critical path of the one warp that runs this branch)
            auto self_mirror = [&](const pk *zqu, const pk *zmu, auto qc) {
                constexpr int q = decltype(qc)::value;
                pk v[M];
                solve(zqu, zmu, q, v);
                constexpr int jq = -K + ((q + K) % N);
                cl::static_for<0, M>([&](auto lc) {
                    constexpr int l = decltype(lc)::value;
                    constexpr int k = jq + l * N;
                    constexpr int lm = (-k - jq) % N == 0 && (-k - jq) / N >= 0 && (-k - jq) / N < M ? (-k - jq) / N : -1;
                    if constexpr (!(k < 0 && lm >= 0)) {  // a negative k with a partner is emitted with it
                        constexpr int p = k < 0 ? -k : k;
                        static_assert((p * 64) % L == 0, "self-mirror pre-twiddles are 64th roots");
                        constexpr int e1 = p * 64 / L, e2 = (2 * e1) % 64;
                        pk X;
                        if constexpr (k < 0) X = pkx::mul(pkx::conj(v[l]), bc(0.5f));
                        else if constexpr (lm >= 0) X = pkx::mul(add(v[l], pkx::conj(v[lm])), bc(0.5f));
                        else X = pkx::mul(v[l], bc(0.5f));
                        emit(p, X, make_float2((float)cl::cos64(e1), (float)cl::sin64(e1)),
                             make_float2((float)cl::cos64(e2), (float)cl::sin64(e2)));
                    }
                });
            };
#if MCI_ROWG_BALANCED
            // One pattern for every class, q = 0 included (no divergent branch on warp 0, whose three
            // partner warps waited for it at the next barrier).  The regular class q emits element l at
            // p = |j_q + l N| with the value a(k) or conj a(k); for q = 0 (thread 0, u = 0) the same slots
            // are written, partners k and -k twice with the same Hermitian average, k = 0 with Re a(0) and
            // its mirror sent to a padding slot (raw index 64: swz64 never maps there), and the MN = 4096
            // edge -K with both terms summed at k' = S/2.
            auto emitb = [&](int p, int pmraw, bool half, pk X, float2 wa, float2 wa2) {
                const pk P1 = pkx::cmul(X, mk(wa));
                const pk a2 = mk(wa2);
                pk A = add_rot<1>(X, P1);
                const pk Am = add_rot<1>(pkx::conj(X), pkx::conj(P1));
                pk B = pkx::cmul(A, a2);
                const pk Bm = pkx::cmul(Am, pkx::conj(a2));
                if (half) {  // (only instantiated where p = S/2 can occur)
                    A = add(A, Am);
                    B = add(B, Bm);
                }
                bufA[swz64(p)] = f2(A);
                bufB[swz64(p)] = f2(B);
                bufA[pmraw] = f2(Am);
                bufB[pmraw] = f2(Bm);
            };
            cl::static_for<0, QPT>([&](auto uc) {
                constexpr int u = decltype(uc)::value;
                const int q = tid + 128 * u;
                float2 wq[8], wq2[8];
                if constexpr (M <= 2) {
                    tm_ld4(tmA + tmc_wp<N>() + 4 * u, wq);
                    tm_ld4(tmA + tmc_wp2<N>() + 4 * u, wq2);
                } else if constexpr (M <= 4) {
                    tm_ld8(tmA + tmc_wp<N>() + 8 * u, wq);
                    tm_ld8(tmA + tmc_wp2<N>() + 8 * u, wq2);
                } else {
                    tm_ld16(tmA + tmc_wp<N>() + 16 * u, wq);
                    tm_ld16(tmA + tmc_wp2<N>() + 16 * u, wq2);
                }
                pk v[M], w[M];
                solve(zq[u], zm[u], q, v);
                const int jq = -K + ((q + K) % N);
#pragma unroll
                for (int l = 0; l < M; ++l) w[l] = jq + l * N >= 0 ? v[l] : pkx::conj(v[l]);
                const bool is0 = u == 0 && q == 0;
                constexpr int jq0 = -K + (K % N);  // j_q of the class q = 0
                pk x0[M];
                if constexpr (u == 0) {
                    cl::static_for<0, M>([&](auto lc) {
                        constexpr int l = decltype(lc)::value;
                        constexpr int k0 = jq0 + l * N;
                        constexpr int lm = (-k0 - jq0) % N == 0 && (-k0 - jq0) / N >= 0 && (-k0 - jq0) / N < M
                                               ? (-k0 - jq0) / N : -1;
                        if constexpr (k0 == 0) x0[l] = mk(f2(v[l]).x, 0.f);
                        else if constexpr (lm >= 0) x0[l] = pkx::mul(add(w[l], w[lm]), bc(0.5f));
                        else x0[l] = pkx::mul(w[l], bc(0.5f));
                    });
                }
                cl::static_for<0, M>([&](auto lc) {
                    constexpr int l = decltype(lc)::value;
                    constexpr int k0 = jq0 + l * N;
                    const int k = jq + l * N;
                    const int p = k >= 0 ? k : -k;
                    pk X = w[l];
                    int pm = swz64(S - p);
                    bool half = false;
                    if constexpr (u == 0) {
                        X.v = is0 ? x0[l].v : X.v;
                        if constexpr (k0 == 0) pm = is0 ? 64 : pm;
                        if constexpr (K == S / 2 && k0 == -K) {
                            half = is0;
                            pm = is0 ? 64 : pm;
                        }
                    }
                    emitb(p, pm, half, X, wq[l], wq2[l]);
                });
            });
#else
#pragma unroll
            for (int u = 0; u < QPT; ++u) {
                const int q = tid + 128 * u;
                float2 wq[8], wq2[8];  // (tcgen05.ld is warp-collective: before the q = 0 branch)
                if constexpr (M <= 2) {
                    tm_ld4(tmA + tmc_wp<N>() + 4 * u, wq);
                    tm_ld4(tmA + tmc_wp2<N>() + 4 * u, wq2);
                } else if constexpr (M <= 4) {
                    tm_ld8(tmA + tmc_wp<N>() + 8 * u, wq);
                    tm_ld8(tmA + tmc_wp2<N>() + 8 * u, wq2);
                } else {
                    tm_ld16(tmA + tmc_wp<N>() + 16 * u, wq);
                    tm_ld16(tmA + tmc_wp2<N>() + 16 * u, wq2);
                }
                if (q == 0) {
                    self_mirror(zq[0], zm[0], std::integral_constant<int, 0>{});
                    continue;
                }
                pk v[M];
                solve(zq[u], zm[u], q, v);
                const int jq = -K + ((q + K) % N);
#pragma unroll
                for (int l = 0; l < M; ++l) {
                    const int k = jq + l * N;
                    if (k >= 0) emit(k, v[l], wq[l], wq2[l]);
                    else emit(-k, pkx::conj(v[l]), wq[l], wq2[l]);
                }
            }
#endif
            // the q* class runs on warp 2 so that it overlaps warp 0's q = 0 branch (both make the other
            // warps of the group wait at the next barrier)
            if (tid == QS_TID) self_mirror(zq[QPT], zm[QPT], std::integral_constant<int, N / 2>{});
            group_bar<NT>(barid);

            // ---- inverse pass 1: radix 64, Ls = 1.  Lane pair (2s, 2s+1) runs FFTs A and B on
            //      butterfly t; inputs k' in (K, S-K) are structurally zero and not read
            float2 *buf = h ? bufB : bufA;
            pk x[64];
            cl::static_for<0, 64>([&](auto jc) {
                constexpr int j = decltype(jc)::value;
                const int kp = t + 64 * j;
                if constexpr ((zmask(K) >> j) & 1ull) x[j] = mk(0.f, 0.f);
                else if constexpr (allnz(K, j)) x[j] = mk(buf[swz64(kp)]);
                else x[j] = nz(K, kp) ? mk(buf[swz64(kp)]) : mk(0.f, 0.f);
            });
            group_bar<NT>(barid);
            pkx::dftz<64, 1, zmask(K)>(x);
#pragma unroll
            for (int j = 0; j < 64; ++j) buf[swz64(64 * t + j)] = f2(x[j]);
            group_bar<NT>(barid);
            // ---- inverse pass 2: radix 64, Ls = 64; twiddles w4096^{j t}
#pragma unroll
            for (int j = 0; j < 64; ++j) x[j] = mk(buf[swz64(t + 64 * j)]);
#pragma unroll
            for (int p2 = 0; p2 < 31; ++p2) {
                const float4 w2 = *reinterpret_cast<const float4 *>(itwp + 128 * p2 + 2 * t);
                x[2 * p2 + 1] = pkx::cmul(x[2 * p2 + 1], mk(w2.x, w2.y));
                x[2 * p2 + 2] = pkx::cmul(x[2 * p2 + 2], mk(w2.z, w2.w));
            }
            x[63] = pkx::cmul(x[63], mk(itwp[31 * 128 + t]));
            pkx::dft<64, 1>(x);
            // outputs p2 = t + 64 j: A -> f[4p2], f[4p2+1]; B -> f[4p2+2], f[4p2+3]; handed to the
            // store warpgroup through TMEM
            mbar_wait(tm_empty(grp), opar ^ 1u);
            asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
#pragma unroll
            for (int c = 0; c < 4; ++c) {
                float v[32];
#pragma unroll
                for (int i = 0; i < 16; ++i) {
                    const float2 xv = f2(x[16 * c + i]);
                    v[2 * i] = xv.x;
                    v[2 * i + 1] = xv.y;
                }
                tm_st32(tmA + 128 * grp + 32 * c, v);
            }
            asm volatile("tcgen05.wait::st.sync.aligned;" ::: "memory");
            asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
            mbar_arrive(tm_full(grp));
            opar ^= 1u;
        }
    }
    asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
    __syncthreads();
    if (threadIdx.x < 32) tm_dealloc<512>(tm_base);
}

// ---------------------------------------------------------------------------------------
template <int M, int N, int BK>
static cudaError_t rowg_launch_t(const RowGTables &tb, int64_t rows, const float *g, float *f, cudaStream_t st) {
    using C = RowGCfg<M, N>;
    auto kern = mci_rowg_kernel<M, N, BK>;
    cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, C::SMEM);
    if (e != cudaSuccess) return e;
    int dev = 0, nsm = 148;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, dev);
    int64_t grid = nsm;  // persistent: one CTA (3 row groups + the store warpgroup) per SM
    const int64_t need = (rows + 2) / 3;
    if (grid > need) grid = need;
    kern<<<(unsigned)grid, C::THREADS, C::SMEM, st>>>(g, f, rows, tb);
    return cudaGetLastError();
}

template <int M, int N>
static cudaError_t rowg_dispatch(int bk, const RowGTables &tb, int64_t rows, const float *g, float *f, cudaStream_t st) {
    if constexpr (M == 3)
        if (bk == rowg::BK_EX2) return rowg_launch_t<M, N, rowg::BK_EX2>(tb, rows, g, f, st);
    if constexpr (M == 2 || M == 4 || M == 8)
        if (bk == rowg::BK_DELAY) return rowg_launch_t<M, N, rowg::BK_DELAY>(tb, rows, g, f, st);
    if (bk == rowg::BK_DERIV) return rowg_launch_t<M, N, rowg::BK_DERIV>(tb, rows, g, f, st);
    return rowg_launch_t<M, N, rowg::BK_TABLE>(tb, rows, g, f, st);
}

bool rowg_supported(const Axis1D &ax) {
    return ax.dtype == MCI_F32 && !ax.analytic && ax.S == 4096 && ax.R == 4 &&
           ((ax.M == 3 && ax.N == 1024) || (ax.M == 4 && ax.N == 1024) || (ax.M == 2 && ax.N == 2048) ||
            (ax.N == 512 && ax.M >= 5 && ax.M <= 8));
}

cudaError_t launch_rowg(const Axis1D &ax, int64_t rows, const void *g, void *f, cudaStream_t st, int *n_launches) {
    if (rows <= 0) return cudaSuccess;
    const float2 *base = (const float2 *)ax.rowtab;
    RowGTables tb;
    // layout written by mci_plan.cpp: [wp: K+1][fw2: 32x32][itw: 64x64][fw3: 16x64][fw8: 8x8]
    //                                 [tw256: 16x16][tw2k: 2048][ainv: M x M reals (as complex .x)]
    tb.Qt = (const float2 *)ax.Qt;
    tb.wp = base;
    tb.itw = tb.wp + (ax.K + 1) + 32 * 32;
    tb.fw3 = tb.itw + 64 * 64;
    tb.fw8 = tb.fw3 + 16 * 64;
    tb.tw256 = tb.fw8 + 8 * 8;
    tb.tw2k = tb.tw256 + 256;
    tb.ainv = (const float *)(tb.tw2k + 2048);
    tb.tw512 = tb.tw2k + 2048 + (ax.M * ax.M + 1) / 2;  // after ainv (M^2 reals, padded to even)
    if (n_launches) *n_launches += 1;
    const float *gg = (const float *)g;
    float *ff = (float *)f;
    const int bk = ax.bank_deriv012 && ax.M == 3 ? rowg::BK_EX2
                 : ax.bank_derivM             ? rowg::BK_DERIV
                 : ax.bank_delay_ti           ? rowg::BK_DELAY
                                              : rowg::BK_TABLE;
    if (ax.M == 3 && ax.N == 1024) return rowg_dispatch<3, 1024>(bk, tb, rows, gg, ff, st);
    if (ax.M == 4 && ax.N == 1024) return rowg_dispatch<4, 1024>(bk, tb, rows, gg, ff, st);
    if (ax.M == 2 && ax.N == 2048) return rowg_dispatch<2, 2048>(bk, tb, rows, gg, ff, st);
    if (ax.M == 5 && ax.N == 512) return rowg_dispatch<5, 512>(bk, tb, rows, gg, ff, st);
    if (ax.M == 6 && ax.N == 512) return rowg_dispatch<6, 512>(bk, tb, rows, gg, ff, st);
    if (ax.M == 7 && ax.N == 512) return rowg_dispatch<7, 512>(bk, tb, rows, gg, ff, st);
    if (ax.M == 8 && ax.N == 512) return rowg_dispatch<8, 512>(bk, tb, rows, gg, ff, st);
    return cudaErrorInvalidValue;
}

}  // namespace mci
