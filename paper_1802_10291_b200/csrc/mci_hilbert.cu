// Analytic-output (f and Hf) MCI row kernel for BASELINE.json configs[2]:
// M = 2 channels (f, f'), N = 4096 samples, L = 65536 outputs, fp32.
//
// Mathematics as in mci_fused.cu: forward DFT (Lemma 1),
// per-class solve (Eq. matrixeqn1), Hermitian part, and the
// Hilbert twin through the one-sided analytic spectrum Z(0) = X(0),
// Z(k) = 2 X(k) (Example 4; multiplier -i sgn k,
// PAPER.md:107-116): one complex inverse DFT gives z = f + i Hf.
//
// Inverse layout: L = R S with S = 2048, R = 32.  Output phase p1 of p = 32 p2 + p1
// is the 2048-point inverse DFT over k' = k mod S of
//     Zin(k') = sum_{k = k' (mod S), 0 <= k <= K} Z(k) e^{2 pi i k p1 / L}
//             = w^{k' p1} (Z(k') + u Z(k' + S) [+ u^2 Z(2S) at k' = 0]),  u = e^{2 pi i p1 / 32}.
// One CTA (256 threads, 8 warps) owns a row (persistent over rows):
//   * forward: one complex 4096-point FFT of (g0 + i g1), channels scaled by exact
//     powers of two, as three radix-16 passes over all 256 threads;
//   * solve: 2049 classes -> Z[0..K] in shared memory; for the (1, ik) bank the
//     closed-form inverse a(j) = ((j+N) G0 + i G1)/N^2, a(j+N) = (-j G0 - i G1)/N^2
//     (exact in fp32), else the plan's Q table;
//   * 4 rounds of 8 consecutive phases p1 = 8 r + c: lanes c = lane & 7 run phase c on
//     butterfly tid >> 3, so every warp store writes 4 whole 32-byte sectors of f (and of Hf);
//     pass 1 radix 64 with the pre-twiddle fused into its loads, pass 2 radix 32 x 2.
#include <cuda.h>
#include <cudaTypedefs.h>

#include <cstdint>
#include <cstdlib>
#include <cstring>

#include "mci_internal.h"
#include "mci_pk.cuh"

#ifndef MCI_HIL_FOLD
#define MCI_HIL_FOLD 1  // 0: the seven-instruction fold (A/B)
#endif

namespace mci {

namespace hilk {
constexpr int M = 2, N = 4096, K = 4096, L = 65536, S = 2048, R = 32, NT = 256;
constexpr int BUF = 2082;               // padded 2048-point buffer (pad6 -> 2079 used); = 2 (mod 16)
constexpr int NBUF = 8;                 // one per phase of a round
constexpr int ZLEN = K + 2;             // Z[0..K] (+1 pad)
constexpr int ITW_LD = 65;              // row stride of the [32][65] twiddle table
__device__ __forceinline__ int pad6(int a) { return a + (a >> 6); }
__device__ __forceinline__ int pad4(int a) { return a + (a >> 4); }  // forward 4096-point buffer
__device__ __forceinline__ float pow2f(int e) { return __int_as_float((127 + e) << 23); }
// compute-thread barrier (named, so a store warpgroup can run beside the 8 compute warps)
__device__ __forceinline__ void bar() { asm volatile("bar.sync 1, %0;" ::"n"(NT) : "memory"); }
__device__ __forceinline__ uint32_t su32(const void *p) { return (uint32_t)__cvta_generic_to_shared(p); }
// next row's input arrives by TMA bulk copy (cp.async.bulk + mbarrier) while this row is transformed
__device__ __forceinline__ void stage_row(float *dst, const float *src, uint64_t *mb) {
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(su32(mb)), "r"(M * N * 4) : "memory");
    asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
                     su32(dst)),
                 "l"(src), "r"(M * N * 4), "r"(su32(mb))
                 : "memory");
}
__device__ __forceinline__ void mb_arrive(uint64_t *mb) {
    asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(su32(mb)) : "memory");
}
__device__ __forceinline__ void tm_st32(uint32_t ta, const float *v) {
    asm volatile(
        "tcgen05.st.sync.aligned.32x32b.x32.b32 [%0], {%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,%16,"
        "%17,%18,%19,%20,%21,%22,%23,%24,%25,%26,%27,%28,%29,%30,%31,%32};" ::"r"(ta),
        "f"(v[0]), "f"(v[1]), "f"(v[2]), "f"(v[3]), "f"(v[4]), "f"(v[5]), "f"(v[6]), "f"(v[7]), "f"(v[8]),
        "f"(v[9]), "f"(v[10]), "f"(v[11]), "f"(v[12]), "f"(v[13]), "f"(v[14]), "f"(v[15]), "f"(v[16]),
        "f"(v[17]), "f"(v[18]), "f"(v[19]), "f"(v[20]), "f"(v[21]), "f"(v[22]), "f"(v[23]), "f"(v[24]),
        "f"(v[25]), "f"(v[26]), "f"(v[27]), "f"(v[28]), "f"(v[29]), "f"(v[30]), "f"(v[31])
        : "memory");
}
__device__ __forceinline__ void tm_ld8(uint32_t ta, float *v) {
    asm volatile("tcgen05.ld.sync.aligned.32x32b.x8.b32 {%0,%1,%2,%3,%4,%5,%6,%7}, [%8];"
                 : "=f"(v[0]), "=f"(v[1]), "=f"(v[2]), "=f"(v[3]), "=f"(v[4]), "=f"(v[5]), "=f"(v[6]), "=f"(v[7])
                 : "r"(ta));
    asm volatile("tcgen05.wait::ld.sync.aligned;"
                 : "+f"(v[0]), "+f"(v[1]), "+f"(v[2]), "+f"(v[3]), "+f"(v[4]), "+f"(v[5]), "+f"(v[6]), "+f"(v[7])::"memory");
}
__device__ __forceinline__ void stage_wait(uint64_t *mb, uint32_t parity) {
    uint32_t done = 0;
    while (!done)
        asm volatile("{ .reg .pred p; mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2; selp.u32 %0, 1, 0, p; }"
                     : "=r"(done)
                     : "r"(su32(mb)), "r"(parity)
                     : "memory");
}
}  // namespace hilk

struct HilbertTables {
    const float2 *Qt;   // [N/2+1][2][2]   H^{-1}/N per class (table mode)
    const float2 *whi;  // [256]  e^{+2 pi i 256 h / L}
    const float2 *wlo;  // [256]  e^{+2 pi i l / L}
    const float2 *itw;  // [32][65] e^{+2 pi i j t / 2048}
    int deriv;          // 1: bank is (1, ik) -> closed-form inverse
};

// MODE 1 (STW): a fourth... (ninth to twelfth) warp set -- a store warpgroup -- takes each round's 64
// outputs per thread out of tensor memory (lane = compute thread, 128 columns per compute
// warpgroup, double-buffered by round) and writes them with the compute threads' sector-aligned
// pattern, so the output stores never stall the transform.
// MODE 2 (TS): after pass 2 the compute threads write the round's outputs into a staging tile
// [p2][8 phases] (f and Hf planes, 128 KB) laid over the phase buffers, and one thread stores it
// with TMA tensor stores (cp.async.bulk.tensor, boxes of 256 p2 x 8 phases = 32-byte runs at a
// 128-byte pitch): the 4,096 sector-scattered 32-bit global stores per row leave the LSU pipe.
// MODE 0: the compute threads store directly.
template <int MODE>
__global__ void __launch_bounds__(hilk::NT + (MODE == 1 ? 128 : 0), 1)
    mci_hilbert_kernel(const float *__restrict__ g, float *__restrict__ f, float *__restrict__ hf, int64_t rows,
                       HilbertTables tb, const __grid_constant__ CUtensorMap tmf,
                       const __grid_constant__ CUtensorMap tmh) {
    using namespace hilk;
    using namespace pkx;
    constexpr bool STW = MODE == 1, TS = MODE == 2;
    extern __shared__ __align__(16) unsigned char smem[];
    float2 *Z = reinterpret_cast<float2 *>(smem);  // [ZLEN]
    float2 *bufs = Z + ZLEN;                        // NBUF x BUF; the forward aliases bufs[0 .. 4352)
    float2 *whi = bufs + NBUF * BUF;                // 256
    float2 *wlo = whi + 256;                        // 256
    float2 *itw = wlo + 256;                        // 32 x 65
    float2 *F = bufs;                               // forward spectrum, pad4 layout (4352 slots)
    float *stage = reinterpret_cast<float *>(itw + 32 * ITW_LD);  // [2][4096] input row
    // w16[t] = wlo[16 t] = e^{2 pi i 16 t / L}: the forward pass-3 twiddle's low factor, whose
    // wlo index is a multiple of 16 (one bank pair: 16-way conflicts) -- here 16 consecutive slots
    float2 *w16 = reinterpret_cast<float2 *>(stage + M * N);
    // likewise contiguous copies of two strided whi reads: u32[p1] = whi[8 p1] (pass-1 fold
    // factor; 8 phases per warp at stride 8: 4-way) and t16[16 j + k] = whi[(j k) mod 256]
    // (forward pass-2 twiddles; stride j across lanes: up to 8-way)
    float2 *u32 = w16 + 16;
    float2 *t16 = u32 + 32;
    // TS: staging planes [2048 p2][8 phases] of f and Hf, 128-byte aligned, over the phase buffers
    float *Sf = reinterpret_cast<float *>(((uintptr_t)bufs + 127) & ~(uintptr_t)127);
    float *Sh = Sf + 2048 * 8;
    __shared__ __align__(8) uint64_t mbar;
    __shared__ float smx[8][2];
    __shared__ float ssc[2];
    __shared__ uint32_t tm_base;
    __shared__ __align__(8) uint64_t tfull[2], tempty[2];  // STW: per TMEM buffer (round parity)
    if (STW) {
        if (threadIdx.x < 32) {
            asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 512;" ::"r"(su32(&tm_base))
                         : "memory");
            asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;" ::: "memory");
        }
        if (threadIdx.x == 32) {
            for (int i = 0; i < 2; ++i) {
                asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(su32(&tfull[i])), "n"(NT) : "memory");
                asm volatile("mbarrier.init.shared::cta.b64 [%0], 128;" ::"r"(su32(&tempty[i])) : "memory");
            }
        }
    }
    for (int i = threadIdx.x; i < 256; i += NT) {
        whi[i] = tb.whi[i];
        wlo[i] = tb.wlo[i];
        if (i < 16) w16[i] = tb.wlo[16 * i];
        if (i < 32) u32[i] = tb.whi[8 * i];
        t16[i] = tb.whi[((i >> 4) * (i & 15)) & 255];
    }
    for (int i = threadIdx.x; i < 32 * ITW_LD; i += NT) itw[i] = tb.itw[i];
    if (threadIdx.x == 0) {
        asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(su32(&mbar)) : "memory");
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
        if (blockIdx.x < rows) stage_row(stage, g + blockIdx.x * (int64_t)(M * N), &mbar);
    }
    if (STW) asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
    __syncthreads();
    if (STW) asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
    uint32_t parity = 0;
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31, tid = threadIdx.x;
    if (STW && threadIdx.x >= NT) {
        // ---- store warpgroup: warp k drains TMEM lane quarter k of both compute warpgroups
        asm volatile("setmaxnreg.dec.sync.aligned.u32 56;" ::: "memory");
        const int k = warp - NT / 32;
        const uint32_t ta = tm_base + ((uint32_t)(32 * k) << 16);
        uint32_t rc = 0;  // global round count
        for (int64_t row = blockIdx.x; row < rows; row += gridDim.x) {
            for (int r = 0; r < 4; ++r, ++rc) {
                const uint32_t b = rc & 1;
                stage_wait(&tfull[b], (rc >> 1) & 1);
                asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
#pragma unroll 1
                for (int wg = 0; wg < 2; ++wg) {
                    const int ctid = 128 * wg + 32 * k + lane;  // the compute thread of this lane
                    const int c = ctid & 7, bt = ctid >> 3, p1 = 8 * r + c;
                    float *fr = f + row * (int64_t)L + p1, *hr = hf + row * (int64_t)L + p1;
                    // (measured: this loop fully unrolled with base + immediate addresses, ~1 instead of ~6
                    // instructions per store, runs the kernel at 0.852 ms instead of 0.731 -- store bursts
                    // crowd the compute warps out of the LSU queue; a 32 ns sleep per chunk: 0.746)
#pragma unroll 1
                    for (int cc = 0; cc < 16; ++cc) {  // 8 columns = outputs (hh, j), 4 per chunk
                        float v[8];
                        tm_ld8(ta + 256 * b + 128 * wg + 8 * cc, v);
#pragma unroll
                        for (int i = 0; i < 4; ++i) {
                            const int e = 4 * cc + i, hh = e >> 5, j = e & 31;
                            const int64_t o = (int64_t)R * (bt + 32 * hh + 64 * j);
                            __stcs(fr + o, v[2 * i]);
                            __stcs(hr + o, v[2 * i + 1]);
                        }
                    }
                }
                asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
                mb_arrive(&tempty[b]);
            }
        }
    } else {
    if (STW) asm volatile("setmaxnreg.inc.sync.aligned.u32 200;" ::: "memory");
    uint32_t rcc = 0;  // STW: global round count of the compute side
    // w = e^{+2 pi i m / L}, m in [0, L)
    auto wL = [&](int m) { return pkx::cmul(mk(whi[m >> 8]), mk(wlo[m & 255])); };

    for (int64_t row = blockIdx.x; row < rows; row += gridDim.x) {
        stage_wait(&mbar, parity);
        parity ^= 1;
        // ---- forward: 4096-point FFT of (g0 + i g1), radix 16 x 16 x 16 (Stockham), all threads
        {
            const int b = tid;
            pk x[16];
            float m0 = 0.f, m1 = 0.f;
#pragma unroll
            for (int j = 0; j < 16; ++j) {
                const float a0 = stage[b + 256 * j], a1 = stage[N + b + 256 * j];
                m0 = fmaxf(m0, fabsf(a0));
                m1 = fmaxf(m1, fabsf(a1));
                x[j] = mk(a0, a1);
            }
            m0 = warp_max_nonneg(m0);
            m1 = warp_max_nonneg(m1);
            if (lane == 0) {
                smx[warp][0] = m0;
                smx[warp][1] = m1;
            }
            if (TS && tid == 0) asm volatile("cp.async.bulk.wait_group.read 0;" ::: "memory");
            bar();  // maxima visible; previous row's last reads of the buffers are complete
            if (tid == 0 && row + gridDim.x < rows) {  // stage consumed: fetch the next row
                asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
                stage_row(stage, g + (row + gridDim.x) * (int64_t)(M * N), &mbar);
            }
            m0 = smx[0][0];
            m1 = smx[0][1];
#pragma unroll
            for (int w = 1; w < 8; ++w) {
                m0 = fmaxf(m0, smx[w][0]);
                m1 = fmaxf(m1, smx[w][1]);
            }
            const int E0 = (__float_as_int(m0) >> 23) & 0xff, E1 = (__float_as_int(m1) >> 23) & 0xff;
            const int e0 = E0 == 0 ? 0 : max(-100, min(100, E0 - 126));
            const int e1 = E1 == 0 ? 0 : max(-100, min(100, E1 - 126));
            const pk sc = mk(pow2f(-e0), pow2f(-e1));
#pragma unroll
            for (int j = 0; j < 16; ++j) x[j] = mul(x[j], sc);
            // pass 1: Ls = 1
            dft<16, -1>(x);
#pragma unroll
            for (int j = 0; j < 16; ++j) F[pad4(16 * b + j)] = f2(x[j]);
            bar();
            // pass 2: Ls = 16, twiddle e^{-2 pi i j k / 256} = conj(whi[j k])
            {
                const int k = b & 15;
#pragma unroll
                for (int j = 0; j < 16; ++j) x[j] = mk(F[pad4(b + 256 * j)]);
#pragma unroll
                for (int j = 1; j < 16; ++j) x[j] = pkx::cmul(x[j], pkx::conj(mk(t16[16 * j + k])));
                dft<16, -1>(x);
                bar();
#pragma unroll
                for (int j = 0; j < 16; ++j) F[pad4(16 * (b - k) + k + 16 * j)] = f2(x[j]);
            }
            bar();
            // pass 3: Ls = 256, twiddle e^{-2 pi i j b / 4096} = conj(w^{16 j b})
#pragma unroll
            for (int j = 0; j < 16; ++j) x[j] = mk(F[pad4(b + 256 * j)]);
#pragma unroll
            for (int j = 1; j < 16; ++j) {  // e^{2 pi i j b / 4096} = whi[(j b) >> 4] w16[(j b) & 15]
                const int jb = j * b;
                x[j] = pkx::cmul(x[j], pkx::conj(pkx::cmul(mk(whi[(jb >> 4) & 255]), mk(w16[jb & 15]))));
            }
            dft<16, -1>(x);
#pragma unroll
            for (int j = 0; j < 16; ++j) F[pad4(b + 256 * j)] = f2(x[j]);
            if (tid == 0) {
                ssc[0] = 0.5f * pow2f(e0);
                ssc[1] = 0.5f * pow2f(e1);
            }
        }
        bar();
        // ---- solve: class q has j_q = q - N (elements q - N, q); Z(0) = X(0), Z(k) = 2 X(k)
        {
            const float h0 = ssc[0], h1 = ssc[1];
            for (int q = tid; q <= N / 2; q += NT) {
                const pk zq = mk(F[pad4(q)]), zm = mk(F[pad4((N - q) & (N - 1))]);
                const pk G0 = mul(add(zq, pkx::conj(zm)), bc(h0));
                const pk G1 = mul(rot<-1>(sub(zq, pkx::conj(zm))), bc(h1));
                pk v0, v1;
                if (tb.deriv) {
                    // (1, ik): a(j) = ((j+N) G0 + i G1)/N^2, a(j+N) = (-j G0 - i G1)/N^2, j = q - N
                    const float jn = (float)(q - N), inv = 1.f / ((float)N * (float)N);
                    const pk iG1 = rot<1>(G1);
                    v0 = add(mul(G0, bc((jn + (float)N) * inv)), mul(iG1, bc(inv)));
                    v1 = sub(mul(G0, bc(-jn * inv)), mul(iG1, bc(inv)));
                } else {
                    const float2 *Qq = tb.Qt + q * 4;
                    v0 = add(pkx::cmul(G0, mk(__ldg(Qq + 0))), pkx::cmul(G1, mk(__ldg(Qq + 2))));
                    v1 = add(pkx::cmul(G0, mk(__ldg(Qq + 1))), pkx::cmul(G1, mk(__ldg(Qq + 3))));
                }
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
        // ---- 4 rounds of 8 phases p1 = 8 r + c
        const int c = tid & 7;
        const int bt = tid >> 3;  // pass-1 butterfly (0..31); pass 2 runs bt and bt + 32
        float2 *buf = bufs + c * BUF;
        for (int r = 0; r < 4; ++r) {
            const int p1 = 8 * r + c;
            pk x[64];
            {  // pass 1 (Ls = 1): k' = bt + 32 j; Zin(k') = w^{k' p1} (Z(k') + u Z(k' + S)),
               // w^{k' p1} = w^{bt p1} e^{2 pi i j p1 / 2048} (itw row p1)
                const pk u = mk(u32[p1]);  // e^{2 pi i 2048 p1 / L}
                const pk wb = wL(bt * p1);
#if MCI_HIL_FOLD
                // wb (Z(k') + u Z(k'+S)) as wb Z(k') + (u wb) Z(k'+S): four FMA-class instructions
                // (one multiply, three fused), then the table factor: 6 per input instead of 7
                const pk uw = pkx::cmul(u, wb);
                const float2 wbf = f2(wb), uwf = f2(uw);
                const pk wbr = mk(-wbf.y, wbf.x), uwr = mk(-uwf.y, uwf.x);  // i wb, i u wb
#pragma unroll
                for (int j = 0; j < 64; ++j) {
                    const int kp = bt + 32 * j;
                    const float2 z0 = Z[kp], z1 = Z[kp + S];
                    pk y = mul(wb, bc(z0.x));
                    y = fma(wbr, bc(z0.y), y);
                    y = fma(uw, bc(z1.x), y);
                    y = fma(uwr, bc(z1.y), y);
                    x[j] = pkx::cmul(y, mk(itw[p1 * ITW_LD + j]));
                }
#else
#pragma unroll
                for (int j = 0; j < 64; ++j) {
                    const int kp = bt + 32 * j;
                    const pk s = add(mk(Z[kp]), pkx::cmul(mk(Z[kp + S]), u));
                    x[j] = pkx::cmul(s, pkx::cmul(wb, mk(itw[p1 * ITW_LD + j])));
                }
#endif
                if (bt == 0) {  // k' = 0 also receives k = 2S = K: u^2 Z(K)
                    x[0] = add(x[0], pkx::cmul(mk(Z[K]), mk(whi[(16 * p1) & 255])));  // e^{2 pi i 4096 p1 / L}
                }
            }
            dft<64, 1>(x);
            // TS: the previous round's staging tile has been read by its TMA stores
            if (TS && tid == 0) asm volatile("cp.async.bulk.wait_group.read 0;" ::: "memory");
            bar();  // previous round's pass-2 loads are complete before the buffers are rewritten
#pragma unroll
            for (int j = 0; j < 64; ++j) buf[pad6(64 * bt + j)] = f2(x[j]);
            bar();
            // pass 2 (Ls = 64): radix 32 on butterflies t = bt and bt + 32; outputs p2 = t + 64 j
            float *fr = f + row * (int64_t)L + p1, *hr = hf + row * (int64_t)L + p1;
            const uint32_t tb_ = STW ? tm_base + ((uint32_t)(32 * (warp & 3)) << 16) + 256 * (rcc & 1) +
                                           128 * (warp >> 2)
                                     : 0u;
            if (STW) {  // the store warpgroup has drained this TMEM buffer (two rounds ago)
                stage_wait(&tempty[rcc & 1], ((rcc >> 1) & 1) ^ 1);
                asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
            }
            if constexpr (TS) {
                pk y[2][32];
#pragma unroll
                for (int hh = 0; hh < 2; ++hh)
#pragma unroll
                    for (int j = 0; j < 32; ++j) y[hh][j] = mk(buf[pad6(bt + 32 * hh + 64 * j)]);
                bar();  // every pass-2 load done: the staging tile may overwrite the buffers
#pragma unroll
                for (int hh = 0; hh < 2; ++hh) {
                    const int t = bt + 32 * hh;
#pragma unroll
                    for (int j = 1; j < 32; ++j) y[hh][j] = pkx::cmul(y[hh][j], mk(itw[j * ITW_LD + t]));
                    dft<32, 1>(y[hh]);
#pragma unroll
                    for (int j = 0; j < 32; ++j) {  // output p2 = t + 64 j, phase c of the round
                        const float2 z = f2(y[hh][j]);
                        Sf[(t + 64 * j) * 8 + c] = z.x;
                        Sh[(t + 64 * j) * 8 + c] = z.y;
                    }
                }
                asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
                bar();
                if (tid == 0) {
#pragma unroll 1
                    for (int b = 0; b < 8; ++b) {
                        asm volatile(
                            "cp.async.bulk.tensor.3d.global.shared::cta.bulk_group [%0, {%1, %2, %3}], [%4];" ::"l"(&tmf),
                            "r"(8 * r), "r"(256 * b), "r"((int)row), "r"(su32(Sf + 2048 * b))
                            : "memory");
                        asm volatile(
                            "cp.async.bulk.tensor.3d.global.shared::cta.bulk_group [%0, {%1, %2, %3}], [%4];" ::"l"(&tmh),
                            "r"(8 * r), "r"(256 * b), "r"((int)row), "r"(su32(Sh + 2048 * b))
                            : "memory");
                    }
                    asm volatile("cp.async.bulk.commit_group;" ::: "memory");
                }
                continue;
            }
#pragma unroll
            for (int hh = 0; hh < 2; ++hh) {
                const int t = bt + 32 * hh;
                pk y[32];
#pragma unroll
                for (int j = 0; j < 32; ++j) y[j] = mk(buf[pad6(t + 64 * j)]);
#pragma unroll
                for (int j = 1; j < 32; ++j) y[j] = pkx::cmul(y[j], mk(itw[j * ITW_LD + t]));
                dft<32, 1>(y);
                if (STW) {
#pragma unroll
                    for (int cc = 0; cc < 2; ++cc) {
                        float v[32];
#pragma unroll
                        for (int i = 0; i < 16; ++i) {
                            const float2 z = f2(y[16 * cc + i]);
                            v[2 * i] = z.x;
                            v[2 * i + 1] = z.y;
                        }
                        tm_st32(tb_ + 64 * hh + 32 * cc, v);
                    }
                } else {
#pragma unroll
                    for (int j = 0; j < 32; ++j) {
                        const float2 z = f2(y[j]);
                        const int64_t o = (int64_t)R * (t + 64 * j);
                        __stcs(fr + o, z.x);
                        __stcs(hr + o, z.y);
                    }
                }
            }
            if (STW) {
                asm volatile("tcgen05.wait::st.sync.aligned;" ::: "memory");
                asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
                mb_arrive(&tfull[rcc & 1]);
                ++rcc;
            }
        }
    }
    if (TS && threadIdx.x == 0) asm volatile("cp.async.bulk.wait_group 0;" ::: "memory");
    }  // compute warps
    if (STW) {
        asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
        __syncthreads();
        if (threadIdx.x < 32)
            asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 512;" ::"r"(tm_base) : "memory");
    }
}

// TMA view of an output plane [rows][2048 p2][32 p1] (p = 32 p2 + p1), box 8 phases x 256 p2
static bool encode_out_map(CUtensorMap *tm, void *base, int64_t rows) {
    const auto enc = (PFN_cuTensorMapEncodeTiled_v12000)tensor_map_encoder();
    if (!enc) return false;
    const cuuint64_t dims[3] = {32, 2048, (cuuint64_t)rows};
    const cuuint64_t strides[2] = {32 * 4, (cuuint64_t)hilk::L * 4};
    const cuuint32_t box[3] = {8, 256, 1}, es[3] = {1, 1, 1};
    return enc(tm, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 3, base, dims, strides, box, es, CU_TENSOR_MAP_INTERLEAVE_NONE,
               CU_TENSOR_MAP_SWIZZLE_NONE, CU_TENSOR_MAP_L2_PROMOTION_NONE, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) ==
           CUDA_SUCCESS;
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
    const float2 *base = (const float2 *)ax.rowtab;  // [whi 256][wlo 256][itw 32 x 65]
    tb.whi = base;
    tb.wlo = base + 256;
    tb.itw = base + 512;
    tb.deriv = ax.bank_deriv01;
    const size_t smem = (size_t)(ZLEN + NBUF * BUF + 512 + 32 * ITW_LD) * 8 + M * N * 4 + (16 + 32 + 256) * 8;
    // MCI_HILBERT_VARIANT=1: the 8-warp layout storing directly, 2: TMA tensor stores from a
    // staging tile (A/B); default: store warpgroup
    const int variant = getenv("MCI_HILBERT_VARIANT") ? atoi(getenv("MCI_HILBERT_VARIANT")) : 0;
    const bool stw = variant == 0;
    CUtensorMap tmf, tmh;
    memset(&tmf, 0, sizeof(tmf));
    memset(&tmh, 0, sizeof(tmh));
    const bool ts = variant == 2 && rows < (1ll << 31) && aligned16(f) && aligned16(hf) &&
                    encode_out_map(&tmf, f, rows) && encode_out_map(&tmh, hf, rows);
    auto kern = stw ? mci_hilbert_kernel<1> : ts ? mci_hilbert_kernel<2> : mci_hilbert_kernel<0>;
    cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    if (e != cudaSuccess) return e;
    int dev = 0, nsm = 148;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, dev);
    int64_t grid = nsm;
    if (grid > rows) grid = rows;
    if (n_launches) *n_launches += 1;
    kern<<<(unsigned)grid, NT + (stw ? 128 : 0), smem, st>>>((const float *)g, (float *)f, (float *)hf, rows, tb, tmf,
                                                            tmh);
    return cudaGetLastError();
}

}  // namespace mci
