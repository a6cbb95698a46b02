// Specialised fused MCI row kernel for the batched real-output shape
// (BASELINE.json configs[1]: M = 3 channels, N = 1024, L = 16384, fp32).
//
// Same mathematics as mci_fused.cu (Lemma 1 forward DFT PAPER.md:180-233,
// per-class solve a = D H^{-1} Eq. matrixeqn1, Hermitian-part
// assembly, zero-padded inverse of Eq. DFTexpression).
// B200 layout (the binding resource is the shared-memory/L1 data pipe, so the
// design minimises shared-memory round trips):
//   * CTA = G row groups of 128 threads (4 warps) with named barriers; input
//     rows arrive by TMA bulk copy (cp.async.bulk + mbarrier), the next row is
//     prefetched while the current one is transformed;
//   * forward: two complex 1024-point FFTs (channel pairs (g0,g1), (g2,0)) as
//     two register radix-32 passes (one shared-memory exchange);
//   * per-class solve: Q~ from the plan's table (through L1), or -- for the (f, f', f'') bank --
//     the paper's closed-form inverse of Example 2, exact in
//     fp32 (integer numerators over powers of two);
//   * the solve writes the pre-twiddled inputs of the two inverse FFTs
//     (A: p1 = 0,1 and B: p1 = 2,3; Zin(k) = Y(k)(w^{2ck} + i w^{(2c+1)k}));
//   * inverse: two 4096-point FFTs as two register radix-64 passes; lanes 0-15
//     of every warp run FFT A and lanes 16-31 FFT B on the same butterfly
//     index, so one warp-wide 64-bit store writes 256 contiguous output bytes
//     (A: f[4p2], f[4p2+1]; B: f[4p2+2], f[4p2+3]);
//   * shared buffers use XOR swizzles (conflict-free for both access strides);
//   * all complex arithmetic runs on packed FP32x2 instructions (FADD2/FFMA2/
//     FMUL2, mci_pk.cuh): same FLOP rate as scalar FFMA, half the issue slots.
#include <cstdint>

#include "mci_fft.cuh"
#include "mci_internal.h"
#include "mci_pk.cuh"

#ifndef MCI_ROW_BALANCED
#define MCI_ROW_BALANCED 1  // 0: the divergent q = 0 branch and table loads for q* (A/B)
#endif
#ifndef MCI_ROW_SCALE2
#define MCI_ROW_SCALE2 0  // 1: also scale channel 2 to unit range (A/B; it shares its FFT with no channel)
#endif

namespace mci {

namespace rowk {

constexpr int NT = 128;  // threads per row group

__device__ __forceinline__ uint32_t smem_u32(const void *p) { return (uint32_t)__cvta_generic_to_shared(p); }
__device__ __forceinline__ void mbar_init(uint64_t *bar, uint32_t count) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count) : "memory");
}
__device__ __forceinline__ void mbar_expect_tx(uint64_t *bar, uint32_t bytes) {
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)), "r"(bytes)
                 : "memory");
}
__device__ __forceinline__ void tma_load_1d(void *dst, const void *src, uint32_t bytes, uint64_t *bar) {
    asm volatile(
        "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
            smem_u32(dst)),
        "l"(src), "r"(bytes), "r"(smem_u32(bar))
        : "memory");
}
__device__ __forceinline__ void mbar_wait(uint64_t *bar, uint32_t parity) {
    uint32_t done = 0;
    const uint32_t a = smem_u32(bar);
    while (!done)
        asm volatile(
            "{ .reg .pred p; mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2; selp.u32 %0, 1, 0, p; }"
            : "=r"(done)
            : "r"(a), "r"(parity)
            : "memory");
}
__device__ __forceinline__ void tma_store_1d(void *gdst, const void *ssrc, uint32_t bytes) {
    asm volatile("cp.async.bulk.global.shared::cta.bulk_group [%0], [%1], %2;" ::"l"(gdst), "r"(smem_u32(ssrc)),
                 "r"(bytes)
                 : "memory");
    asm volatile("cp.async.bulk.commit_group;" ::: "memory");
}
__device__ __forceinline__ void tma_store_wait_read() {
    asm volatile("cp.async.bulk.wait_group.read 0;" ::: "memory");
}
__device__ __forceinline__ void group_bar(int id) { asm volatile("bar.sync %0, %1;" ::"r"(id), "r"(NT) : "memory"); }

// paddings (8-byte elements; bank pair = low 4 bits): conflict-free for contiguous
// runs and for the radix-R transposed stores (stride R), and -- unlike XOR
// swizzles -- a constant offset per unrolled index, so no address arithmetic
__device__ __forceinline__ int swz32(int a) { return a + (a >> 5); }  // forward, 1024 -> 1056
__device__ __forceinline__ int swz64(int a) { return a + (a >> 6); }  // inverse, 4096 -> 4160
// 4-warp forward (radix 8 x 8 x 16): no padding is conflict-free for all its strides;
// this XOR swizzle is (brute-force checked), and keeps each 1024-point FFT in 1024 slots
__device__ __forceinline__ int sw3(int a) { return a ^ ((a >> 3) & 15); }

// 2^e as an exact float (|e| <= 100)
__device__ __forceinline__ float pow2f(int e) { return __int_as_float((127 + e) << 23); }

// ---- tensor memory (TMEM) as per-thread read-only tables.  Every table entry the
// kernel reads is a fixed function of the thread's index within its row group, and
// thread tid of every group maps to TMEM lane tid (warp w of a group accesses lanes
// 32 (w % 4) ..), so one copy serves the three groups.  tcgen05.ld runs beside the
// shared-memory pipe (tools/microbench/tmem_ld.cu: >= 370 B/clk/SM at 16 warps),
// which is the kernel's most loaded data path.
constexpr int TM_COLS = 512;
// TM flags (template parameter): which per-thread data live in TMEM
constexpr int TM_SMALL = 1;   // forward-pass and pre-twiddle tables (read through L1 otherwise)
constexpr int TM_ITWF = 2;    // inverse pass-2 twiddles (shared memory otherwise)
constexpr int TM_L2PF = 4;    // the store warpgroup prefetches each group's input two rows ahead into L2
constexpr int TM_STORE = 8;   // outputs, drained by a fourth (store) warpgroup
constexpr int TM_A2 = 32;     // squared pre-twiddles e^{2 pi i 2p / L}: FFT B's inputs = a^2 x FFT A's
constexpr int TM_TS = 64;     // no store warpgroup: outputs staged in the group's (dead) exchange buffers in row
                              // order and written by one 64 KB TMA bulk store per row
// column map; with TM_STORE the outputs take columns 0..383 and the tables move up by 256
constexpr int TM_ITW = 0;    // 126 cols: w_j(t) = e^{+2 pi i j t / 4096}, j = 1..63 (inverse pass 2)
constexpr int TM_FW8 = 128;  // 14 cols: e^{-2 pi i j k / 64}, j = 1..7, k = tid & 7 (forward pass 2)
constexpr int TM_FW3 = 144;  // 30 cols: e^{-2 pi i j bb / 1024}, j = 1..15, bb = tid & 63 (forward pass 3)
constexpr int TM_WP = 176;   // 24 cols: e^{+2 pi i p / L} for p = N - q, q, q + N, q = tid + 128 u (solve)
constexpr int TM_WP2 = 200;  // 24 cols: e^{+2 pi i 2p / L} for the same p (TM_A2)
__device__ __forceinline__ void tm_st8(uint32_t ta, const float *v) {
    asm volatile("tcgen05.st.sync.aligned.32x32b.x8.b32 [%0], {%1,%2,%3,%4,%5,%6,%7,%8};" ::"r"(ta),
                 "f"(v[0]), "f"(v[1]), "f"(v[2]), "f"(v[3]), "f"(v[4]), "f"(v[5]), "f"(v[6]), "f"(v[7])
                 : "memory");
}
// Example 2 closed-form inverse for the (f, f', f'') bank, class q of
// N = 1024, K = 1536, divided by N (d = G/N): r0[l], r1[l] (r2 = (-d2, d1, -d2) is constant).
// Every numerator is an integer < 2^24 and every denominator a power of two: exact in fp32.
__device__ __forceinline__ void ex2_coeffs(int q, float *r0, float *r1) {
    constexpr int N = 1024, K = 1536;
    const float n = (float)(-K + ((q + K) % N));
    const float Nf = (float)N;
    const float d2 = 1.f / (2.f * Nf * Nf * Nf), d1 = 1.f / (Nf * Nf * Nf);
    r0[0] = (2.f * Nf * Nf + 3.f * Nf * n + n * n) * d2;
    r0[1] = -(n * (2.f * Nf + n)) * d1;
    r0[2] = (n * (Nf + n)) * d2;
    r1[0] = (3.f * Nf + 2.f * n) * d2;
    r1[1] = -2.f * (Nf + n) * d1;
    r1[2] = (Nf + 2.f * n) * d2;
}
// load 8 consecutive columns (4 complex entries) and wait; the wait names the
// destination registers so no use can be scheduled before it
__device__ __forceinline__ void tm_ld8(uint32_t ta, float2 *w) {
    float v0, v1, v2, v3, v4, v5, v6, v7;
    asm volatile("tcgen05.ld.sync.aligned.32x32b.x8.b32 {%0,%1,%2,%3,%4,%5,%6,%7}, [%8];"
                 : "=f"(v0), "=f"(v1), "=f"(v2), "=f"(v3), "=f"(v4), "=f"(v5), "=f"(v6), "=f"(v7)
                 : "r"(ta));
    asm volatile("tcgen05.wait::ld.sync.aligned;"
                 : "+f"(v0), "+f"(v1), "+f"(v2), "+f"(v3), "+f"(v4), "+f"(v5), "+f"(v6), "+f"(v7)::"memory");
    w[0] = make_float2(v0, v1);
    w[1] = make_float2(v2, v3);
    w[2] = make_float2(v4, v5);
    w[3] = make_float2(v6, v7);
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
__device__ __forceinline__ void mbar_arrive(uint64_t *bar) {
    asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(smem_u32(bar)) : "memory");
}
__device__ __forceinline__ void tm_ld16(uint32_t ta, float2 *w) {
    float v[16];
    asm volatile(
        "tcgen05.ld.sync.aligned.32x32b.x16.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15}, [%16];"
        : "=f"(v[0]), "=f"(v[1]), "=f"(v[2]), "=f"(v[3]), "=f"(v[4]), "=f"(v[5]), "=f"(v[6]), "=f"(v[7]),
          "=f"(v[8]), "=f"(v[9]), "=f"(v[10]), "=f"(v[11]), "=f"(v[12]), "=f"(v[13]), "=f"(v[14]), "=f"(v[15])
        : "r"(ta));
    asm volatile("tcgen05.wait::ld.sync.aligned;"
                 : "+f"(v[0]), "+f"(v[1]), "+f"(v[2]), "+f"(v[3]), "+f"(v[4]), "+f"(v[5]), "+f"(v[6]), "+f"(v[7]),
                   "+f"(v[8]), "+f"(v[9]), "+f"(v[10]), "+f"(v[11]), "+f"(v[12]), "+f"(v[13]), "+f"(v[14]),
                   "+f"(v[15])::"memory");
#pragma unroll
    for (int i = 0; i < 8; ++i) w[i] = make_float2(v[2 * i], v[2 * i + 1]);
}

}  // namespace rowk

// Device tables built by the plan (fp64-rounded), see mci_plan.cpp.
struct RowTables {
    const float2 *Qt;   // [(N/2+1)][M][M]  H^{-1}/N per class (table mode)
    const float2 *wp;   // [K+1]      e^{+2 pi i p / L}
    const float2 *fw2;  // [32][32]   e^{-2 pi i j k / 1024}     (forward pass 2)
    const float2 *itw;  // [64][64]   e^{+2 pi i j t / 4096}     (inverse pass 2)
    const float2 *fw3;  // [16][64]   e^{-2 pi i j b / 1024}     (4-warp forward pass 3)
    const float2 *fw8;  // [8][8]     e^{-2 pi i j k / 64}       (4-warp forward pass 2)
    int deriv;          // 1: bank is (1, ik, -k^2) -> closed-form Q (Example 2)
};

template <int G, bool QTAB, bool FW4 = false, int TM = 0>
struct RowCfg {
    static constexpr int M = 3, N = 1024, S = 4096, K = 1536, L = 16384;
    static constexpr int NQ = N / 2 + 1;
    static constexpr bool STAGED = G < 3;                   // TMA-staged input rows (G <= 2)
    static constexpr int STAGE_BYTES = STAGED ? M * N * 4 : 0;  // 12 KB
    static constexpr int BUF_ELEMS = S + S / 64;             // padded inverse buffer (4160)
    static constexpr int FWD_ELEMS = N + N / 32;             // padded forward buffer (1056)
    static constexpr int GROUP_BYTES = STAGE_BYTES + (2 * BUF_ELEMS + 8) * 8;  // B offset by 8 elements
    static constexpr int Q_BYTES = 0;  // table-mode Q~ is read through L1 (__ldg)
    static constexpr int FW_TAB = FW4 ? 16 * 64 + 8 * 8 : 32 * 32;  // forward twiddles
    // G = 3 (12 warps) fits 227 KB only with the inverse twiddles (rows j >= 1) alone in
    // shared memory; the pre-twiddle and forward tables are then read through L1
    static constexpr bool SMALL_TAB = G >= 3;
    static constexpr int TAB_BYTES = (TM & rowk::TM_ITWF) ? 0 : SMALL_TAB ? 63 * 64 * 8 : (FW_TAB + 64 * 64 + K + 2) * 8;
    static constexpr int SMEM = G * GROUP_BYTES + Q_BYTES + TAB_BYTES;
    // TM = 3: a fourth warpgroup streams the outputs out of tensor memory
    static constexpr int THREADS = G * 128 + ((TM & rowk::TM_STORE) ? 128 : 0);
};

template <int G, bool QTAB, bool FW4, int TM = 0>
__global__ void __launch_bounds__(RowCfg<G, QTAB, FW4, TM>::THREADS, 1)
    mci_row_kernel(const float *__restrict__ g, float *__restrict__ f, int64_t rows, RowTables tb) {
    using namespace rowk;
    using C = RowCfg<G, QTAB, FW4, TM>;
    static_assert(!C::SMALL_TAB || FW4, "G = 3 uses the 4-warp forward");
    static_assert(!TM || (FW4 && G == 3), "TMEM tables: 3 groups, 4-warp forward");
    constexpr bool TMS = TM & TM_SMALL, TMI = TM & TM_ITWF, PF2 = TM & TM_L2PF, STW = TM & TM_STORE;
    constexpr bool TS = (TM & TM_TS) != 0;
    static_assert(!(TS && STW), "TMA bulk stores replace the store warpgroup");
    static_assert(!(STW && TMI), "the outputs leave no TMEM room for the inverse twiddles");
    static_assert(!PF2 || STW || TS, "the L2 prefetch is issued by the store warpgroup (TS: by the compute threads)");
    constexpr int TB = STW ? 256 : 0;  // table column shift
    constexpr int M = C::M, N = C::N, S = C::S, K = C::K, L = C::L;
    extern __shared__ __align__(128) unsigned char smem[];
    __shared__ __align__(8) uint64_t mbar[G];
    __shared__ float ssup[G][4];
    __shared__ float smx[G][4][3];  // per-warp channel maxima (4-warp forward)
    __shared__ uint32_t tm_base;
    // TM = 3: output hand-off barriers of group gg, kept in the 64-byte gap between its
    // buffers A and B (the 227 KB budget has no room for them in static shared memory)
    auto tm_full = [&](int gg) {
        return reinterpret_cast<uint64_t *>(smem + gg * C::GROUP_BYTES + C::STAGE_BYTES + C::BUF_ELEMS * 8);
    };
    auto tm_empty = [&](int gg) { return tm_full(gg) + 1; };

    const int grp = threadIdx.x / NT;
    const int tid = threadIdx.x % NT;
    const int warp = tid >> 5, lane = tid & 31;
    const int barid = 1 + grp;
    unsigned char *gbase = smem + grp * C::GROUP_BYTES;
    float *stage = reinterpret_cast<float *>(gbase);
    float2 *bufA = reinterpret_cast<float2 *>(gbase + C::STAGE_BYTES);
    float2 *bufB = bufA + C::BUF_ELEMS + 8;  // +8 elements: A and B lanes of a half-warp hit different banks
    float2 *fwd = bufB;  // forward spectra (2 x 1024) alias buffer B
    float2 *fw2 = reinterpret_cast<float2 *>(smem + G * C::GROUP_BYTES + C::Q_BYTES);
    float2 *fw3 = fw2, *fw8 = fw2 + 16 * 64;  // 4-warp forward twiddles (alias fw2)
    // inverse pass-2 twiddles w_j(t) = e^{+2 pi i j t / 4096}, j = 1..63, paired for 128-bit loads:
    // itwp[128 p + 2 t + h] = w_{2p+1+h}(t) for p < 31, itwp[3968 + t] = w_63(t)  (4032 entries)
    float2 *itwp = C::SMALL_TAB ? fw2 : fw2 + C::FW_TAB;
    float2 *wps = itwp + 64 * 64;  // e^{+2 pi i p / L}, p = 0..K (layouts with all tables in smem)
    // table reads: shared memory, or L1 (__ldg) in the G = 3 layout
    auto ld_wp = [&](int p) { return C::SMALL_TAB ? __ldg(tb.wp + p) : wps[p]; };
    auto ld_fw3 = [&](int i) { return C::SMALL_TAB ? __ldg(tb.fw3 + i) : fw3[i]; };
    auto ld_fw8 = [&](int i) { return C::SMALL_TAB ? __ldg(tb.fw8 + i) : fw8[i]; };

    // ---- one-time setup
    if constexpr (TM) {
        if (threadIdx.x < 32) {
            asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(smem_u32(&tm_base)),
                         "n"(TM_COLS)
                         : "memory");
            asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;" ::: "memory");
        }
        asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
        __syncthreads();
        asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
        if ((TMS || TMI) && threadIdx.x < NT) {  // group 0 writes lane tid of the shared tables
            const int tt = threadIdx.x;
            const uint32_t ta = tm_base + ((uint32_t)(32 * (tt >> 5)) << 16);
            const int t2 = 16 * (tt >> 5) + ((tt & 31) >> 1);  // inverse butterfly of this lane
            float v[8];
#pragma unroll 1
            for (int c = 0; TMI && c < 128; c += 8) {  // inverse pass-2 twiddles, j = 1 + c/2 ..
#pragma unroll
                for (int i = 0; i < 4; ++i) {
                    const int j = 1 + c / 2 + i;
                    const float2 w = j <= 63 ? tb.itw[j * 64 + t2] : make_float2(0.f, 0.f);
                    v[2 * i] = w.x;
                    v[2 * i + 1] = w.y;
                }
                tm_st8(ta + TM_ITW + c, v);
            }
#pragma unroll 1
            for (int c = 0; TMS && c < 16; c += 8) {  // forward pass-2 twiddles
#pragma unroll
                for (int i = 0; i < 4; ++i) {
                    const int j = 1 + c / 2 + i;
                    const float2 w = j <= 7 ? tb.fw8[j * 8 + (tt & 7)] : make_float2(0.f, 0.f);
                    v[2 * i] = w.x;
                    v[2 * i + 1] = w.y;
                }
                tm_st8(ta + TB + TM_FW8 + c, v);
            }
#pragma unroll 1
            for (int c = 0; TMS && c < 32; c += 8) {  // forward pass-3 twiddles
#pragma unroll
                for (int i = 0; i < 4; ++i) {
                    const int j = 1 + c / 2 + i;
                    const float2 w = j <= 15 ? tb.fw3[j * 64 + (tt & 63)] : make_float2(0.f, 0.f);
                    v[2 * i] = w.x;
                    v[2 * i + 1] = w.y;
                }
                tm_st8(ta + TB + TM_FW3 + c, v);
            }
#pragma unroll 1
            for (int c = 0; TMS && c < 32; c += 8) {  // pre-twiddles of the solve outputs (entry 3u + e)
#pragma unroll
                for (int i = 0; i < 4; ++i) {
                    const int idx = c / 2 + i, u = idx / 3, e = idx % 3;
                    const int q = tt + 128 * u;
                    const int pp = e == 0 ? (N - q) & (2 * N - 1) : e == 1 ? q : q + N;  // q = 0: e = 0 -> p = N
                    const float2 w = u < 4 ? tb.wp[pp] : make_float2(0.f, 0.f);
                    v[2 * i] = w.x;
                    v[2 * i + 1] = w.y;
                }
                tm_st8(ta + TB + TM_WP + c, v);
            }
#pragma unroll 1
            for (int c = 0; (TM & TM_A2) && c < 24; c += 8) {  // their squares, in double precision
#pragma unroll
                for (int i = 0; i < 4; ++i) {
                    const int idx = c / 2 + i, u = idx / 3, e = idx % 3;
                    const int q = tt + 128 * u;
                    const int pp = e == 0 ? (N - q) & (2 * N - 1) : e == 1 ? q : q + N;
                    double sn, cs;
                    sincospi(4.0 * pp / L, &sn, &cs);
                    v[2 * i] = (float)cs;
                    v[2 * i + 1] = (float)sn;
                }
                tm_st8(ta + TB + TM_WP2 + c, v);
            }
            asm volatile("tcgen05.wait::st.sync.aligned;" ::: "memory");
        }
    }
    for (int i = threadIdx.x; !TMI && i < 31 * 128 + 64; i += G * NT) {
        const int pp = i >> 7, r = i & 127;
        itwp[i] = i < 31 * 128 ? tb.itw[(2 * pp + 1 + (r & 1)) * 64 + (r >> 1)] : tb.itw[63 * 64 + (i - 31 * 128)];
    }
    if constexpr (C::SMALL_TAB) {
    } else if constexpr (FW4) {
        for (int i = threadIdx.x; i < 16 * 64; i += G * NT) fw3[i] = tb.fw3[i];
        for (int i = threadIdx.x; i < 8 * 8; i += G * NT) fw8[i] = tb.fw8[i];
    } else {
        for (int i = threadIdx.x; i < 32 * 32; i += G * NT) fw2[i] = tb.fw2[i];
    }
    if constexpr (!C::SMALL_TAB) {
        for (int i = threadIdx.x; i <= K; i += G * NT) wps[i] = tb.wp[i];
    }
    if (tid == 0 && grp < G) mbar_init(&mbar[grp], 1);
    if (STW && threadIdx.x < G) {
        mbar_init(tm_full(threadIdx.x), NT);
        mbar_init(tm_empty(threadIdx.x), NT);
    }
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    if constexpr (TM) asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
    __syncthreads();
    if constexpr (TM) asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
    const uint32_t tmA = TM ? tm_base + ((uint32_t)(32 * warp) << 16) : 0u;  // this thread's TMEM lane
    const int64_t gid = (int64_t)blockIdx.x * G + grp;
    const int64_t gstride = (int64_t)gridDim.x * G;
    uint32_t phase = 0;
    if (C::STAGED && tid == 0 && gid < rows) {
        mbar_expect_tx(&mbar[grp], C::STAGE_BYTES);
        tma_load_1d(stage, g + gid * (int64_t)(M * N), C::STAGE_BYTES, &mbar[grp]);
    }

    // forward FFTs run on two warps per group; group 0 uses warps 0-1 and group 1
    // warps 2-3 so the two groups' forward phases land on different SM sub-partitions
    const int fw = warp - 2 * (grp & 1);  // 0 / 1 for the forward warps
    const bool fwd_warp = fw == 0 || fw == 1;
    // inverse FFT lane mapping: even lanes FFT A, odd lanes FFT B, same butterfly t,
    // so every half-warp output store covers 128 contiguous bytes
    const int h = lane & 1;
    const int t = 16 * warp + (lane >> 1);

    uint32_t opar = 0;  // TM = 3: parity of this group's output hand-off
    if (STW && grp == G) {
        // ---- store warpgroup: drains each group's finished row from TMEM (lane = the
        //      computing thread, columns 128 g + 2 j, 2 j + 1 = its output j) with the
        //      compute warps' coalesced store pattern, so output stores never stall them
        asm volatile("setmaxnreg.dec.sync.aligned.u32 32;" ::: "memory");
        const uint32_t ta = tm_base + ((uint32_t)(32 * warp) << 16);
        // TM_L2PF: 96 lanes x 128 B = one 12 KB input row into L2, two rows ahead of its group
        auto l2pf = [&](int64_t r) {
            if (r < rows && tid < M * N * 4 / 128)
                asm volatile("prefetch.global.L2::evict_last [%0];" ::"l"(g + r * (int64_t)(M * N) + 32 * tid));
        };
        if constexpr (PF2) {
            for (int gg = 0; gg < G; ++gg) l2pf((int64_t)blockIdx.x * G + gg + gstride);
        }
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
                    tm_ld8(ta + 128 * gg + 8 * c, w);
#pragma unroll
                    for (int i = 0; i < 4; ++i) __stcs(fo + 2 * (t + 64 * (4 * c + i)) + h, w[i]);
                    // pace the drain: a short sleep between the four-store bursts leaves the LSU to the
                    // compute warps (measured 1.260 -> 1.253 ms; 80 ns and longer fall behind: 1.288;
                    // a fully unrolled, burstier drain 1.315; finer x4 / x2 loads 1.290 / 1.315)
                    __nanosleep(32);
                }
                asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
                mbar_arrive(tm_empty(gg));
                if constexpr (PF2) l2pf(r + 2 * gstride);
            }
            if (!any) break;
        }
    } else {
    if constexpr (STW) asm volatile("setmaxnreg.inc.sync.aligned.u32 160;" ::: "memory");
    for (int64_t row = gid; row < rows; row += gstride) {
        using namespace pkx;
        if constexpr (TS) {
            // the previous row's bulk store has read the buffers (its first writer comes after the next
            // barrier); the row two ahead goes to L2 (96 lanes x 128 B)
            if (tid == 0) tma_store_wait_read();
            if (PF2 && tid < M * N * 4 / 128 && row + 2 * gstride < rows)
                asm volatile("prefetch.global.L2::evict_last [%0];" ::"l"(g + (row + 2 * gstride) * (int64_t)(M * N) + 32 * tid));
        }
        if constexpr (C::STAGED) {
            mbar_wait(&mbar[grp], phase);
            phase ^= 1;
        }

        // ---- forward, 4-warp variant: both 1024-point FFTs as radix 8 x 8 x 16 Stockham
        //      passes over all 128 threads (half the serial work per thread of the 2-warp
        //      variant); pass 1 reads the staged rows, 2 -> buffer A, 3 -> buffer B.
        if constexpr (FW4) {
            const int b = tid;
            {  // pass 1: radix 8, Ls = 1, butterfly b of both FFTs
                pk x0[8], x1[8];
                float m0 = 0.f, m1 = 0.f, m2 = 0.f;
#pragma unroll
                for (int j = 0; j < 8; ++j) {
                    float a0, a1, a2;
                    if constexpr (C::STAGED) {
                        a0 = stage[b + 128 * j];
                        a1 = stage[N + b + 128 * j];
                        a2 = stage[2 * N + b + 128 * j];
                    } else {  // streaming loads (evict-first: keep L1 for the tables)
                        const float *src = g + row * (int64_t)(M * N);
                        a0 = __ldcs(src + b + 128 * j);
                        a1 = __ldcs(src + N + b + 128 * j);
                        a2 = __ldcs(src + 2 * N + b + 128 * j);
                    }
                    x0[j] = mk(a0, a1);
                    x1[j] = mk(a2, 0.f);
                    m0 = fmaxf(m0, fabsf(a0));
                    m1 = fmaxf(m1, fabsf(a1));
                    if constexpr (MCI_ROW_SCALE2) m2 = fmaxf(m2, fabsf(a2));
                }
                m0 = warp_max_nonneg(m0);
                m1 = warp_max_nonneg(m1);
                if constexpr (MCI_ROW_SCALE2) m2 = warp_max_nonneg(m2);
                if (lane == 0) {
                    smx[grp][warp][0] = m0;
                    smx[grp][warp][1] = m1;
                    if constexpr (MCI_ROW_SCALE2) smx[grp][warp][2] = m2;
                }
                group_bar(barid);  // maxima visible; previous row's reads of buffers A/B complete
                // channel 2 is alone in its FFT (g2 + 0 i): the FFT is linear and no other channel's
                // rounding can leak into it, so it needs no scaling (R10 is about channels sharing one
                // complex FFT): e[2] = 0 saves its maxima and eight multiplies per thread
                int e[3] = {0, 0, 0};
#pragma unroll
                for (int m = 0; m < (MCI_ROW_SCALE2 ? 3 : 2); ++m) {
                    const float mm = fmaxf(fmaxf(smx[grp][0][m], smx[grp][1][m]), fmaxf(smx[grp][2][m], smx[grp][3][m]));
                    const int E = (__float_as_int(mm) >> 23) & 0xff;
                    e[m] = E == 0 ? 0 : max(-100, min(100, E - 126));
                }
                if (tid == 0) {
#pragma unroll
                    for (int m = 0; m < 3; ++m) ssup[grp][m] = pow2f(e[m]);
                }
                const pk sc0 = mk(pow2f(-e[0]), pow2f(-e[1]));
                const float sc1 = pow2f(-e[2]);
#pragma unroll
                for (int j = 0; j < 8; ++j) {
                    x0[j] = pkx::mul(x0[j], sc0);
                    if constexpr (MCI_ROW_SCALE2) x1[j] = pkx::mul(x1[j], bc(sc1));
                }
                pkx::dft<8, -1>(x0);
                pkx::dft<8, -1>(x1);
#pragma unroll
                for (int j = 0; j < 8; ++j) {
                    bufB[sw3(8 * b + j)] = f2(x0[j]);
                    bufB[1024 + sw3(8 * b + j)] = f2(x1[j]);
                }
            }
            group_bar(barid);
            if (C::STAGED && tid == 0 && row + gstride < rows) {  // staged input consumed: prefetch the next row
                asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
                mbar_expect_tx(&mbar[grp], C::STAGE_BYTES);
                tma_load_1d(stage, g + (row + gstride) * (int64_t)(M * N), C::STAGE_BYTES, &mbar[grp]);
            }
            {  // pass 2: radix 8, Ls = 8, B -> A
                const int k = b & 7;
                float2 w8[8];
                if constexpr (TMS) tm_ld16(tmA + TB + TM_FW8, w8);
#pragma unroll
                for (int c = 0; c < 2; ++c) {
                    pk x[8];
#pragma unroll
                    for (int j = 0; j < 8; ++j) x[j] = mk(bufB[c * 1024 + sw3(b + 128 * j)]);
#pragma unroll
                    for (int j = 1; j < 8; ++j) x[j] = pkx::cmul(x[j], mk(TMS ? w8[j - 1] : ld_fw8(j * 8 + k)));
                    pkx::dft<8, -1>(x);
#pragma unroll
                    for (int j = 0; j < 8; ++j) bufA[c * 1024 + sw3(8 * (b - k) + k + 8 * j)] = f2(x[j]);
                }
            }
            group_bar(barid);
            {  // pass 3: radix 16, Ls = 64, A -> B; FFT c = tid / 64
                const int c = tid >> 6, bb = tid & 63;
                pk x[16];
#pragma unroll
                for (int j = 0; j < 16; ++j) x[j] = mk(bufA[c * 1024 + sw3(bb + 64 * j)]);
                float2 w3[16];
                if constexpr (TMS) {
                    tm_ld16(tmA + TB + TM_FW3, w3);
                    tm_ld16(tmA + TB + TM_FW3 + 16, w3 + 8);
                }
#pragma unroll
                for (int j = 1; j < 16; ++j) x[j] = pkx::cmul(x[j], mk(TMS ? w3[j - 1] : ld_fw3(j * 64 + bb)));
                pkx::dft<16, -1>(x);
#pragma unroll
                for (int j = 0; j < 16; ++j) bufB[c * 1024 + sw3(bb + 64 * j)] = f2(x[j]);
            }
            group_bar(barid);
        } else {
            // ---- forward: two register radix-32 passes; FFT c = fw on the channel pair
            //      (g_{2c}, g_{2c+1}); channels scaled to unit range by exact powers of two
            //      (avoids cross-channel rounding leakage when |f''| >> |f|)
            {
                const int c = fw, i = lane;
                float2 *F = fwd + (c & 1) * C::FWD_ELEMS;
                pk x[32];
                if (fwd_warp) {  // pass 1: radix 32, Ls = 1, from the staged rows
                    const float *src = C::STAGED ? stage : g + row * (int64_t)(M * N);
                    const float *g0 = src + (2 * c) * N;
                    const float *g1 = src + (2 * c + 1) * N;
                    float m0 = 0.f, m1 = 0.f;
    #pragma unroll
                    for (int j = 0; j < 32; ++j) {
                        const float re = g0[i + 32 * j];
                        const float im = c == 0 ? g1[i + 32 * j] : 0.f;
                        x[j] = mk(re, im);
                        m0 = fmaxf(m0, fabsf(re));
                        m1 = fmaxf(m1, fabsf(im));
                    }
    #pragma unroll
                    for (int o = 16; o; o >>= 1) {
                        m0 = fmaxf(m0, __shfl_xor_sync(0xffffffffu, m0, o));
                        m1 = fmaxf(m1, __shfl_xor_sync(0xffffffffu, m1, o));
                    }
                    const int E0 = (__float_as_int(m0) >> 23) & 0xff, E1 = (__float_as_int(m1) >> 23) & 0xff;
                    const int e0 = E0 == 0 ? 0 : max(-100, min(100, E0 - 126));
                    const int e1 = E1 == 0 ? 0 : max(-100, min(100, E1 - 126));
                    const pk sc = mk(pow2f(-e0), pow2f(-e1));
                    if (lane == 0) {
                        ssup[grp][2 * c] = pow2f(e0);
                        ssup[grp][2 * c + 1] = pow2f(e1);
                    }
    #pragma unroll
                    for (int j = 0; j < 32; ++j) x[j] = pkx::mul(x[j], sc);
                    pkx::dft<32, -1>(x);
                }
                group_bar(barid);  // previous row's reads of buffers A/B are complete
                if (fwd_warp) {
    #pragma unroll
                    for (int j = 0; j < 32; ++j) F[swz32(32 * i + j)] = f2(x[j]);
                }
                group_bar(barid);
                if (C::STAGED && tid == 0 && row + gstride < rows) {  // staged input consumed: prefetch
                    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
                    mbar_expect_tx(&mbar[grp], C::STAGE_BYTES);
                    tma_load_1d(stage, g + (row + gstride) * (int64_t)(M * N), C::STAGE_BYTES, &mbar[grp]);
                }
                if (fwd_warp) {  // pass 2: radix 32, Ls = 32, in place on own positions
    #pragma unroll
                    for (int j = 0; j < 32; ++j) x[j] = mk(F[swz32(i + 32 * j)]);
    #pragma unroll
                    for (int j = 1; j < 32; ++j) x[j] = pkx::cmul(x[j], mk(fw2[j * 32 + i]));
                    pkx::dft<32, -1>(x);
    #pragma unroll
                    for (int j = 0; j < 32; ++j) F[swz32(i + 32 * j)] = f2(x[j]);
                }
                group_bar(barid);
            }
        }

        // ---- solve.  M = 3: for 0 < q < N/2 the class is j_q = q - N with elements
        //      q - N, q, q + N; the self-mirror classes q = 0 and q* = N/2 are done by
        //      thread 0 with the Hermitian-part averaging.
        pk zq[5][2], zm[5][2];
#pragma unroll
        for (int u = 0; u < 5; ++u) {
            const int q = u < 4 ? tid + 128 * u : N / 2;
            const int qm = (N - q) & (N - 1);
            if (u < 4 || tid == 0) {
#pragma unroll
                for (int c = 0; c < 2; ++c) {
                    if constexpr (FW4) {
                        zq[u][c] = mk(bufB[c * 1024 + sw3(q)]);
                        zm[u][c] = mk(bufB[c * 1024 + sw3(qm)]);
                    } else {
                        zq[u][c] = mk(fwd[c * C::FWD_ELEMS + swz32(q)]);
                        zm[u][c] = mk(fwd[c * C::FWD_ELEMS + swz32(qm)]);
                    }
                }
            }
        }
        float hs[3];  // 2^e_m / 2 (the 1/2 of the channel-pair unpacking folded in)
#pragma unroll
        for (int m = 0; m < 3; ++m) hs[m] = 0.5f * ssup[grp][m];
        group_bar(barid);  // forward spectra read: buffer B may now be overwritten

        float2 wq[12];  // TMEM mode: pre-twiddles of this thread's solve outputs (entry 3u + e)
        if constexpr (TMS) {
            tm_ld8(tmA + TB + TM_WP, wq);
            tm_ld8(tmA + TB + TM_WP + 8, wq + 4);
            tm_ld8(tmA + TB + TM_WP + 16, wq + 8);
        }
        float2 wq2[12];  // TM_A2: a^2 for the same outputs
        if constexpr ((TM & TM_A2) != 0) {
            tm_ld8(tmA + TB + TM_WP2, wq2);
            tm_ld8(tmA + TB + TM_WP2 + 8, wq2 + 4);
            tm_ld8(tmA + TB + TM_WP2 + 16, wq2 + 8);
        }
        // emitm: emit with an explicit mirror slot pm (no p > 0 branch): the caller passes S - p, or
        // the never-read slot 2048 (inside the zero-padding band) for p = 0
        auto emitm = [&](int p, int pm, pk X, float2 wa, float2 wa2) {
            const pk a = mk(wa), a2 = mk(wa2);
            const pk P1 = pkx::cmul(X, a);
            const pk A = add_rot<1>(X, P1);
            bufA[swz64(p)] = f2(A);
            bufB[swz64(p)] = f2(pkx::cmul(A, a2));
            const pk Am = add_rot<1>(pkx::conj(X), pkx::conj(P1));
            bufA[swz64(pm)] = f2(Am);
            bufB[swz64(pm)] = f2(pkx::cmul(Am, pkx::conj(a2)));
        };
        auto emit = [&](int p, pk X, float2 wa, float2 wa2) {
            const pk a = mk(TMS ? wa : ld_wp(p));
            const pk P1 = pkx::cmul(X, a);
            if constexpr ((TM & TM_A2) != 0) {
                // FFT B's inputs are a^2 times FFT A's: P2 + i P3 = a^2 (X + i P1), and the
                // mirrored conj(P2) + i conj(P3) = conj(a^2) (conj X + i conj P1)
                const pk a2 = mk(wa2);
                const pk A = add_rot<1>(X, P1);
                bufA[swz64(p)] = f2(A);
                bufB[swz64(p)] = f2(pkx::cmul(A, a2));
                if (p > 0) {
                    const pk Am = add_rot<1>(pkx::conj(X), pkx::conj(P1));
                    bufA[swz64(S - p)] = f2(Am);
                    bufB[swz64(S - p)] = f2(pkx::cmul(Am, pkx::conj(a2)));
                }
            } else {
                const pk P2 = pkx::cmul(P1, a);
                const pk P3 = pkx::cmul(P2, a);
                bufA[swz64(p)] = f2(add_rot<1>(X, P1));  // X + i P1
                bufB[swz64(p)] = f2(add_rot<1>(P2, P3));
                if (p > 0) {  // k' = S - p: conj(X) + i conj(P1)
                    bufA[swz64(S - p)] = f2(add_rot<1>(pkx::conj(X), pkx::conj(P1)));
                    bufB[swz64(S - p)] = f2(add_rot<1>(pkx::conj(P2), pkx::conj(P3)));
                }
            }
        };
        auto solve = [&](const pk *zqu, const pk *zmu, int q, pk *v) {
            // channel-pair unpacking: G_{2c} = (Z[q] + conj Z[-q])/2, G_{2c+1} = (Z[q] - conj Z[-q])/(2i)
            const pk g0 = pkx::mul(add(zqu[0], pkx::conj(zmu[0])), bc(hs[0]));
            const pk g1 = pkx::mul(rot<-1>(sub(zqu[0], pkx::conj(zmu[0]))), bc(hs[1]));
            const pk g2 = pkx::mul(add(zqu[1], pkx::conj(zmu[1])), bc(hs[2]));
            if constexpr (QTAB) {
                const float2 *Qq = tb.Qt + q * 9;
#pragma unroll
                for (int l = 0; l < 3; ++l) {
                    pk acc = pkx::cmul(g0, mk(__ldg(Qq + l)));
                    acc = add(acc, pkx::cmul(g1, mk(__ldg(Qq + 3 + l))));
                    v[l] = add(acc, pkx::cmul(g2, mk(__ldg(Qq + 6 + l))));
                }
            } else {
                // Example 2, paper's L = N, n = j_q; divided by N (d = G/N).
                // Every numerator is an integer < 2^24 and every denominator a power of
                // two, so these entries are exact in fp32.
                const float Nf = (float)N;
                const float d2 = 1.f / (2.f * Nf * Nf * Nf), d1 = 1.f / (Nf * Nf * Nf);
                float r0[3], r1[3];
                ex2_coeffs(q, r0, r1);
                const float r2[3] = {-d2, d1, -d2};
                const pk ig1 = rot<1>(g1);  // i G1
#pragma unroll
                for (int l = 0; l < 3; ++l)  // v = G0 r0 + i G1 r1 + G2 r2
                    v[l] = pkx::fma(g2, bc(r2[l]), pkx::fma(ig1, bc(r1[l]), pkx::mul(g0, bc(r0[l]))));
            }
        };
#pragma unroll
        for (int u = 0; u < 4; ++u) {
            const int q = tid + 128 * u;
            pk v[3];
            solve(zq[u], zm[u], q, v);
            if constexpr (MCI_ROW_BALANCED && TMS && (TM & TM_A2) != 0) {
                // no divergent branch for q = 0 (thread 0, u = 0): its three outputs are selected into the
                // regular pattern -- p = N - q and q + N both become N and carry (a(N) + conj a(-N))/2
                // (the same value written twice), p = q = 0 carries Re a(0) and its mirror goes to the
                // never-read slot 2048 -- so warp 0 does the same work as the other warps of its group
                // (they waited for it at the next barrier: 4 % of the compute warps' samples)
                pk Xa = pkx::conj(v[0]), Xb = v[1], Xc = v[2];
                int pm = S - q;
                if (u == 0) {
                    const bool is0 = q == 0;
                    const pk avg = pkx::mul(add(v[2], Xa), bc(0.5f));
                    Xa.v = is0 ? avg.v : Xa.v;
                    Xc.v = is0 ? avg.v : Xc.v;
                    Xb.v = is0 ? mk(f2(v[1]).x, 0.f).v : Xb.v;
                    pm = is0 ? 2048 : pm;
                }
                emitm(N - q, S - N + q, Xa, wq[3 * u], wq2[3 * u]);
                emitm(q, pm, Xb, wq[3 * u + 1], wq2[3 * u + 1]);
                emitm(q + N, S - N - q, Xc, wq[3 * u + 2], wq2[3 * u + 2]);
            } else if (q != 0) {
                emit(N - q, pkx::conj(v[0]), wq[3 * u], wq2[3 * u]);
                emit(q, v[1], wq[3 * u + 1], wq2[3 * u + 1]);
                emit(q + N, v[2], wq[3 * u + 2], wq2[3 * u + 2]);
            } else {  // q = 0: elements -N, 0, N; X[0] = Re a(0), X[N] = (a(N) + conj a(-N))/2
                emit(0, mk(f2(v[1]).x, 0.f), wq[3 * u + 1], wq2[3 * u + 1]);
                emit(N, pkx::mul(add(v[2], pkx::conj(v[0])), bc(0.5f)), wq[3 * u + 2], wq2[3 * u + 2]);
            }
        }
        if (tid == 0) {  // q* = N/2: elements -3N/2 = -K, -N/2, N/2
            pk v[3];
            solve(zq[4], zm[4], N / 2, v);
            if constexpr (MCI_ROW_BALANCED && L == 16 * N && K == 3 * N / 2) {
                // a(K) = e^{2 pi i 6/64}, a(N/2) = e^{2 pi i 2/64} and their squares: compile-time constants
                // (the table loads were two L1/L2 round trips on warp 0's critical path every row)
                const float2 aK = make_float2((float)cl::cos64(6), (float)cl::sin64(6));
                const float2 aK2 = make_float2((float)cl::cos64(12), (float)cl::sin64(12));
                const float2 aH = make_float2((float)cl::cos64(2), (float)cl::sin64(2));
                const float2 aH2 = make_float2((float)cl::cos64(4), (float)cl::sin64(4));
                emit(K, pkx::mul(pkx::conj(v[0]), bc(0.5f)), aK, aK2);
                emit(N / 2, pkx::mul(add(v[2], pkx::conj(v[1])), bc(0.5f)), aH, aH2);
            } else {
            const float2 aK = __ldg(tb.wp + K), aH = __ldg(tb.wp + N / 2);
            emit(K, pkx::mul(pkx::conj(v[0]), bc(0.5f)), aK, f2(pkx::cmul(mk(aK), mk(aK))));
            emit(N / 2, pkx::mul(add(v[2], pkx::conj(v[1])), bc(0.5f)), aH, f2(pkx::cmul(mk(aH), mk(aH))));
            }
        }
        group_bar(barid);

        // ---- inverse pass 1: radix 64, Ls = 1.  Lane pair (2s, 2s+1) runs FFTs A and B
        //      on butterfly t; zero-padding inputs k' in (K, S-K) are not read.
        float2 *buf = h ? bufB : bufA;
        pk x[64];
#pragma unroll
        for (int j = 0; j < 64; ++j) {
            const int kp = t + 64 * j;
            if (j < 24 || j >= 40) x[j] = mk(buf[swz64(kp)]);
            else if (j == 24) x[j] = (t == 0) ? mk(buf[swz64(kp)]) : mk(0.f, 0.f);
            else x[j] = mk(0.f, 0.f);
        }
        group_bar(barid);
        // inputs j = 25..39 (k' in (K, S-K)) are structurally zero: pruned from the first stage
        pkx::dftz<64, 1, ((1ull << 40) - 1) & ~((1ull << 25) - 1)>(x);
#pragma unroll
        for (int j = 0; j < 64; ++j) buf[swz64(64 * t + j)] = f2(x[j]);
        group_bar(barid);
        // ---- inverse pass 2: radix 64, Ls = 64; twiddles w4096^{j t} = it1[j&7] * it2[j>>3]
#pragma unroll
        for (int j = 0; j < 64; ++j) x[j] = mk(buf[swz64(t + 64 * j)]);
        if constexpr (TMI) {
#pragma unroll
            for (int c = 0; c < 8; ++c) {  // twiddles j = 8c+1 .. 8c+8 (j <= 63)
                float2 w[8];
                tm_ld16(tmA + TM_ITW + 16 * c, w);
#pragma unroll
                for (int i = 0; i < 8; ++i)
                    if (8 * c + 1 + i <= 63) x[8 * c + 1 + i] = pkx::cmul(x[8 * c + 1 + i], mk(w[i]));
            }
        } else {
#pragma unroll
            for (int p2 = 0; p2 < 31; ++p2) {
                const float4 w2 = *reinterpret_cast<const float4 *>(itwp + 128 * p2 + 2 * t);
                x[2 * p2 + 1] = pkx::cmul(x[2 * p2 + 1], mk(w2.x, w2.y));
                x[2 * p2 + 2] = pkx::cmul(x[2 * p2 + 2], mk(w2.z, w2.w));
            }
            x[63] = pkx::cmul(x[63], mk(itwp[31 * 128 + t]));
        }
        pkx::dft<64, 1>(x);
        // outputs p2 = t + 64 j: A -> f[4p2], f[4p2+1]; B -> f[4p2+2], f[4p2+3]
        // (each half-warp store covers 128 contiguous bytes)
        float2 *fo = reinterpret_cast<float2 *>(f + row * (int64_t)L);
#pragma unroll
        if constexpr (STW) {  // hand the row to the store warpgroup through TMEM
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
        } else if constexpr (TS) {
            // every thread's pass-2 loads are complete (their values are in x): the group's 64 KB region
            // [bufA .. bufB) becomes the row's output in memory order, (A.x, A.y, B.x, B.y) per p2
            group_bar(barid);
            float2 *so = reinterpret_cast<float2 *>(gbase);
#pragma unroll
            for (int j = 0; j < 64; ++j) so[2 * (t + 64 * j) + h] = f2(x[j]);
            asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
            group_bar(barid);
            if (tid == 0) tma_store_1d(fo, so, L * 4);
        } else {
#pragma unroll
            for (int j = 0; j < 64; ++j) {
                    __stcs(fo + 2 * (t + 64 * j) + h, f2(x[j]));
            }
        }
    }
    if (TS && tid == 0) asm volatile("cp.async.bulk.wait_group 0;" ::: "memory");
    }  // compute warpgroups
    if constexpr (TM) {
        asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
        __syncthreads();
        if (threadIdx.x < 32)
            asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tm_base), "n"(TM_COLS)
                         : "memory");
    }
}

// ---------------------------------------------------------------------------------------
template <int G, bool QTAB, bool FW4, int TM = 0>
static cudaError_t row_launch_t(const RowTables &tb, int64_t rows, const float *g, float *f, cudaStream_t st) {
    using C = RowCfg<G, QTAB, FW4, TM>;
    auto kern = mci_row_kernel<G, QTAB, FW4, TM>;
    cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, C::SMEM);
    if (e != cudaSuccess) return e;
    int dev = 0, nsm = 148, occ = 1;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, dev);
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, kern, C::THREADS, C::SMEM);
    if (occ < 1) occ = 1;
    int64_t grid = (int64_t)nsm * occ;
    const int64_t need = (rows + G - 1) / G;
    if (grid > need) grid = need;
    kern<<<(unsigned)grid, C::THREADS, C::SMEM, st>>>(g, f, rows, tb);
    return cudaGetLastError();
}

bool row_supported(const Axis1D &ax) {
    return ax.dtype == MCI_F32 && !ax.analytic && ax.M == 3 && ax.N == 1024 && ax.S == 4096 && ax.R == 4;
}

cudaError_t launch_row(const Axis1D &ax, const void *rowtab, int64_t rows, const void *g, void *f, cudaStream_t st,
                       int *n_launches) {
    if (rows <= 0) return cudaSuccess;
    const float2 *base = (const float2 *)rowtab;
    RowTables tb;
    tb.Qt = (const float2 *)ax.Qt;
    // layout written by mci_plan.cpp: [wp: K+1][fw2: 32x32][itw: 64x64]
    tb.deriv = ax.bank_deriv012;
    tb.wp = base;
    tb.fw2 = tb.wp + (ax.K + 1);
    tb.itw = tb.fw2 + 32 * 32;
    tb.fw3 = tb.itw + 64 * 64;
    tb.fw8 = tb.fw3 + 16 * 64;
    if (n_launches) *n_launches += 1;
    const float *gg = (const float *)g;
    float *ff = (float *)f;
    switch (ax.row_variant) {  // A/B variants (plan-time MCI_ROW_VARIANT); 0 is the tuned default
    case 1:  // 2 groups (8 warps), 2-warp forward
        return tb.deriv ? row_launch_t<2, false, false>(tb, rows, gg, ff, st)
                        : row_launch_t<2, true, false>(tb, rows, gg, ff, st);
    case 2:  // 2 groups, 4-warp forward, all tables in shared memory
        return tb.deriv ? row_launch_t<2, false, true>(tb, rows, gg, ff, st)
                        : row_launch_t<2, true, true>(tb, rows, gg, ff, st);
    case 3:  // 3 groups, 4-warp forward, all per-thread twiddle tables in tensor memory
        return tb.deriv ? row_launch_t<3, false, true, rowk::TM_SMALL | rowk::TM_ITWF>(tb, rows, gg, ff, st)
                        : row_launch_t<3, true, true, rowk::TM_SMALL | rowk::TM_ITWF>(tb, rows, gg, ff, st);
    case 5:  // 3 compute groups + a store warpgroup draining the outputs from tensor memory
        return tb.deriv ? row_launch_t<3, false, true, rowk::TM_STORE>(tb, rows, gg, ff, st)
                        : row_launch_t<3, true, true, rowk::TM_STORE>(tb, rows, gg, ff, st);
    case 4:  // the default without the a^2 form of FFT B's inputs
        return tb.deriv ? row_launch_t<3, false, true, rowk::TM_STORE | rowk::TM_SMALL | rowk::TM_L2PF>(tb, rows, gg, ff, st)
                        : row_launch_t<3, true, true, rowk::TM_STORE | rowk::TM_SMALL | rowk::TM_L2PF>(tb, rows, gg, ff, st);
    case 6:  // 3 compute groups + the store warpgroup, no L2 prefetch
        return tb.deriv ? row_launch_t<3, false, true, rowk::TM_STORE | rowk::TM_SMALL>(tb, rows, gg, ff, st)
                        : row_launch_t<3, true, true, rowk::TM_STORE | rowk::TM_SMALL>(tb, rows, gg, ff, st);
    case 7:  // variant 0 with the forward and pre-twiddle tables in tensor memory
        return tb.deriv ? row_launch_t<3, false, true, rowk::TM_SMALL>(tb, rows, gg, ff, st)
                        : row_launch_t<3, true, true, rowk::TM_SMALL>(tb, rows, gg, ff, st);
    case 8:  // 3 groups (12 warps), 4-warp forward, untiled inputs, inverse twiddles in shared memory
        return tb.deriv ? row_launch_t<3, false, true>(tb, rows, gg, ff, st)
                        : row_launch_t<3, true, true>(tb, rows, gg, ff, st);
    case 9:  // no store warpgroup: row-order staging in the exchange buffers + one TMA bulk store per row
        return tb.deriv ? row_launch_t<3, false, true, rowk::TM_SMALL | rowk::TM_L2PF | rowk::TM_A2 | rowk::TM_TS>(tb, rows, gg, ff, st)
                        : row_launch_t<3, true, true, rowk::TM_SMALL | rowk::TM_L2PF | rowk::TM_A2 | rowk::TM_TS>(tb, rows, gg, ff, st);
    case 10:  // variant 9 with the inverse pass-2 twiddles in the tensor memory the hand-off no longer needs
        return tb.deriv ? row_launch_t<3, false, true, rowk::TM_SMALL | rowk::TM_ITWF | rowk::TM_L2PF | rowk::TM_A2 | rowk::TM_TS>(tb, rows, gg, ff, st)
                        : row_launch_t<3, true, true, rowk::TM_SMALL | rowk::TM_ITWF | rowk::TM_L2PF | rowk::TM_A2 | rowk::TM_TS>(tb, rows, gg, ff, st);
    default:  // 3 compute groups + the store warpgroup (outputs from TMEM, input rows into L2
              // two rows ahead); forward and pre-twiddle tables in TMEM; FFT B's inputs = a^2 x A's
        return tb.deriv ? row_launch_t<3, false, true, rowk::TM_STORE | rowk::TM_SMALL | rowk::TM_L2PF | rowk::TM_A2>(tb, rows, gg, ff, st)
                        : row_launch_t<3, true, true, rowk::TM_STORE | rowk::TM_SMALL | rowk::TM_L2PF | rowk::TM_A2>(tb, rows, gg, ff, st);
    }
}

}  // namespace mci
