// Warp-per-line MCI kernel for short real-output lines (the 2D passes of
// BASELINE.json configs[4]: M = 2 channels, N = 512 samples, L = 2048 outputs).
//
// Same mathematics as mci_fused.cu (Lemma 1 forward DFT PAPER.md:180-233,
// per-class solve Eq. matrixeqn1, Hermitian-part assembly,
// zero-padded inverse of Eq. DFTexpression).  One warp owns
// one line at a time, so there are no block barriers, only __syncwarp:
//   * forward: one complex 512-point FFT of (g0 + i g1) (channels scaled to unit
//     range by exact powers of two), three radix-8 passes (two butterflies per lane);
//   * solve: 257 classes (j_q = q - N, elements q - N and q; self-mirror
//     classes q = 0 and N/2), Q~ from shared memory;
//   * inverse: S = 1024 = 2K (the window [-K, K] aliases only at k' = K),
//     R = 2: one complex FFT gives f[2 p2] + i f[2 p2 + 1]; two radix-32
//     passes; lane i writes float2 at p2 = i + 32 j (256 contiguous bytes);
//   * packed FP32x2 arithmetic (mci_pk.cuh), XOR-swizzled warp-private buffers.
// Lines are addressed with RowAddr, so the same kernel serves 1D batches and
// both passes of the separable 2D transform (strided samples).  In the 2D passes
// (TILED) a CTA's 16 lines are adjacent in memory: the next tile [2][16][512] is
// copied by 4-byte cp.async (transposed into a conflict-free [2][16][516] stage)
// while the current one is transformed (one 16-warp CTA per SM: warp buffers,
// stage and tables fill the 227 KB).  The per-lane pre-twiddles and inverse
// pass-2 twiddles are read from tensor memory (a copy per lane quarter), off the
// shared-memory pipe that bounds the kernel; for the (1, ik) bank the solve uses
// the closed-form inverse instead of the Q~ table.
#include <cuda.h>
#include <cudaTypedefs.h>

#include <algorithm>
#include <cstdint>
#include <cstdio>
#include <cstdlib>
#include <cstring>

#include "mci_internal.h"
#include "mci_pk.cuh"

namespace mci {

namespace linek {
constexpr int N = 512, S = 1024, L = 2048, K = 512, NQ = N / 2 + 1;
// paddings (conflict-free for the access strides used, constant offsets per index)
__device__ __forceinline__ int sw3(int a) { return a + (a >> 4); }  // forward 512 -> 544
__device__ __forceinline__ int sw5(int a) { return a + (a >> 5); }  // inverse 1024 -> 1056
// warp buffer stride: = 2 (mod 32) floats, so the tile write-out of the transposed-store
// mode (thread (py, c) reads lines 4c..4c+3 at float py) hits 32 distinct banks
constexpr int BUF = S + S / 32 + 1;
constexpr int SP = N + 2;  // stage row stride = 2 (mod 32): the transposed cp.async (lines l, l + 8 of a warp) hits 32 banks
__device__ __forceinline__ float pow2f(int e) { return __int_as_float((127 + e) << 23); }
// TM: per-lane tables in tensor memory (the kernel is bound by the shared-memory pipe).
// Every warp's lane l reads the same values, so each lane quarter holds a copy:
// columns 0..31: pre-twiddles e^{2 pi i p / L} for p = N - q, q (q = lane + 32 u, entry 2u + e);
// columns 32..93: inverse pass-2 twiddles e^{2 pi i j lane / 1024}, j = 1..31.
constexpr int TM_COLS = 256, TMW = 0, TMI = 32, TMEM_TOTAL_COLS = 512;
__device__ __forceinline__ uint32_t s32(const void *p) { return (uint32_t)__cvta_generic_to_shared(p); }
__device__ __forceinline__ void tst8(uint32_t ta, const float *v) {
    asm volatile("tcgen05.st.sync.aligned.32x32b.x8.b32 [%0], {%1,%2,%3,%4,%5,%6,%7,%8};" ::"r"(ta), "f"(v[0]),
                 "f"(v[1]), "f"(v[2]), "f"(v[3]), "f"(v[4]), "f"(v[5]), "f"(v[6]), "f"(v[7])
                 : "memory");
}
__device__ __forceinline__ void tld16(uint32_t ta, float2 *w) {
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
}  // namespace linek

struct LineTables {
    const float2 *Qt;   // [NQ][2][2] H^{-1}/N per class
    const float2 *wp;   // [K+1] e^{+2 pi i p / L}
    const float2 *fwt;  // [32][16] e^{-2 pi i j k / 512} (plan layout; the 8 x 8 x 8 forward derives its twiddles from wp)
    const float2 *iw;   // [32][32] e^{+2 pi i j k / 1024}
    int deriv;          // 1: bank is (1, ik) -> closed-form inverse, no Q~ reads
};

// TST (2D passes; TILED, or untiled with PF): the tile's 16 output lines leave transposed, as
// f[(l0 / D0) L D0 + p D0 + (l0 % D0) + w] (row p of the 16 lines is 64 contiguous bytes),
// through the warp buffers; the row pass then reads contiguous lines.
// PF (contiguous lines, untiled; with TILED it selects the G16 gather below): the next line's two channel rows are copied by 16-byte
// cp.async into the warp's own buffer while the current line's inverse finishes.
// TMA (TILED with PF): the [m][n][16 lines] tile arrives by four tensor-map box loads
// (cp.async.bulk.tensor, 16 lines x 256 samples each, 64-byte swizzle = the G16 chunk XOR)
// issued by one thread on an mbarrier, instead of 8 cp.async per thread through the LSU.
template <int WARPS, bool TILED, bool TM = false, bool TST = false, bool PF = false, bool TMA = false>
__global__ void __launch_bounds__(WARPS * 32, WARPS >= 16 ? 1 : 2) mci_line_kernel(const float *__restrict__ g, float *__restrict__ f,
                                                              int64_t lines, RowAddr ra, LineTables tb,
                                                              const __grid_constant__ CUtensorMap tmap) {
    using namespace linek;
    using namespace pkx;
    extern __shared__ __align__(16) unsigned char smem[];
    // CT (tiled, tensor-memory tables, 8 warps): compact shared memory -- no copies of Q~
    // (read through L1), of the pre-twiddles or of the inverse twiddles (both in TMEM) -- so
    // two CTAs fit per SM and one's tile write-out overlaps the other's transforms
    constexpr bool CT = TILED && TM && WARPS == 8;
    float2 *Qs = reinterpret_cast<float2 *>(smem);  // NQ*4
    float2 *wps = Qs + NQ * 4;                      // K+1 (+1 pad)
    float2 *fwt = CT ? Qs : wps + K + 2;            // 512
    float2 *iw = fwt + 512;                         // 1024
    // (measured: running the untiled TST CTA as two independent 8-warp halves with 8-line
    // tiles and named barriers was slower, 0.33 -> 0.39 ms per 65,536 lines)
    constexpr int TW = WARPS;  // lines per tile
    // CT: buffer stride = 2 (mod 16) float2 for the 8-line write-out mapping
    constexpr int BUFS = CT ? BUF + 1 : BUF;
    float2 *bufs = CT ? fwt + 512 : iw + 1024;      // WARPS x BUFS
    // TILED: [2][WARPS][SP]; TMA: [2][N][16] at a 1024-byte boundary (the swizzle pattern is
    // a function of the shared-memory address bits)
    // (the boundary is reached by adding an offset to the shared-memory pointer: rounding the pointer
    // through uintptr_t loses its address space and turns every stage read into a generic LD)
    unsigned char *stage0 = (unsigned char *)(bufs + WARPS * BUFS);
    float *stage = reinterpret_cast<float *>(
        TMA ? stage0 + ((1024u - ((uint32_t)__cvta_generic_to_shared(stage0) & 1023u)) & 1023u) : stage0);
    __shared__ __align__(8) uint64_t tbar;  // TMA: tile landed (expect_tx)
    // TMA on the untiled prefetch path (BULK): each warp's next line arrives by two 1D bulk copies
    // (cp.async.bulk, one per channel row) on the warp's own mbarrier instead of 8 cp.async per lane
    constexpr bool BULK = TMA && PF && !TILED && !TST;
    __shared__ __align__(8) uint64_t lbar[BULK ? WARPS : 1];
    if (!CT) {
        for (int i = threadIdx.x; i < NQ * 4; i += WARPS * 32) Qs[i] = tb.Qt[i];
        for (int i = threadIdx.x; i <= K; i += WARPS * 32) wps[i] = tb.wp[i];
    }
    // forward 8 x 8 x 8 twiddles, from the plan's e^{+2 pi i p / L} by quarter turns (exact):
    // fwt[64 (j-1) + b] = W512^{j b} (j = 1..7, b < 64), fwt[448 + 8 (j-1) + k] = W64^{j k} (k < 8)
    for (int i = threadIdx.x; i < 448 + 56; i += WARPS * 32) {
        const int r = i < 448 ? ((((i >> 6) + 1) * (i & 63)) & 511) : ((8 * (((i - 448) >> 3) + 1) * ((i - 448) & 7)) & 511);
        const int q = r >> 7;
        const float2 w = tb.wp[4 * (r & 127)];  // e^{+2 pi i (r mod 128) / 512}
        const float2 v = make_float2(w.x, -w.y);
        fwt[i] = q == 0 ? v : q == 1 ? make_float2(v.y, -v.x) : q == 2 ? make_float2(-v.x, -v.y) : make_float2(-v.y, v.x);
    }
    // inverse pass-2 twiddles re-laid as pairs for 128-bit loads:
    // iw[64 p + 2 i + h] = iw_{2p+1+h}(i) (p < 15), iw[960 + i] = iw_31(i)
    for (int i = threadIdx.x; !CT && i < 15 * 64 + 32; i += WARPS * 32)
        iw[i] = i < 960 ? tb.iw[(2 * (i >> 6) + 1 + (i & 1)) * 32 + ((i & 63) >> 1)] : tb.iw[31 * 32 + (i - 960)];
    __shared__ uint32_t tm_base;
    if (TM) {
        if (threadIdx.x < 32) {
            asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(s32(&tm_base)),
                         "n"(TM_COLS)
                         : "memory");
            asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;" ::: "memory");
        }
        asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
        __syncthreads();
        asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
        if (threadIdx.x < 128) {  // warps 0-3 fill their lane quarter (all quarters identical)
            const int ln = threadIdx.x & 31;
            const uint32_t ta = tm_base + ((uint32_t)(32 * (threadIdx.x >> 5)) << 16);
            float v[8];
#pragma unroll 1
            for (int c = 0; c < 32; c += 8) {
#pragma unroll
                for (int i = 0; i < 4; ++i) {
                    const int idx = c / 2 + i, u = idx >> 1, e = idx & 1, q = ln + 32 * u;
                    const float2 w = tb.wp[e ? q : N - q];
                    v[2 * i] = w.x;
                    v[2 * i + 1] = w.y;
                }
                tst8(ta + TMW + c, v);
            }
#pragma unroll 1
            for (int c = 0; c < 64; c += 8) {
#pragma unroll
                for (int i = 0; i < 4; ++i) {
                    const int j = 1 + c / 2 + i;
                    const float2 w = j <= 31 ? tb.iw[j * 32 + ln] : make_float2(0.f, 0.f);
                    v[2 * i] = w.x;
                    v[2 * i + 1] = w.y;
                }
                tst8(ta + TMI + c, v);
            }
            asm volatile("tcgen05.wait::st.sync.aligned;" ::: "memory");
        }
        asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
    }
    __syncthreads();
    if (TM) asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
    auto ldQ = [&](int i) { return CT ? __ldg(tb.Qt + i) : Qs[i]; };
    auto ldwp = [&](int i) { return CT ? __ldg(tb.wp + i) : wps[i]; };
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    float2 *buf = bufs + warp * BUFS;
    const uint32_t tmA = TM ? tm_base + ((uint32_t)(32 * (warp & 3)) << 16) : 0u;

    // TILED (2D passes): WARPS consecutive lines are adjacent in memory (s0 = 1) while
    // samples are strided.  Tile tl = [2][WARPS][N] is fetched by 4-byte cp.async: element
    // e = (m, n, l) (l fastest: 8 lanes read one 32-byte sector) lands at stage[(m WARPS + l) SP + n].
    const int64_t ntiles = (lines + WARPS - 1) / WARPS;
    // line -> element offset; the launcher guarantees lines < 2^31, so the quotients are
    // 32-bit (a 64-bit division is a long emulated sequence, measured ~8 % of the issue slots)
    const uint32_t uD0 = (uint32_t)ra.D0, uD1 = (uint32_t)ra.D1;
    auto line_base = [&](uint32_t l) -> int64_t {
        const uint32_t a = l / uD0, r0 = l - a * uD0, b = a / uD1, r1 = a - b * uD1;
        return (int64_t)b * ra.s2 + (int64_t)r1 * ra.s1 + (int64_t)r0 * ra.s0;
    };
    auto tile_base = [&](int64_t t) { return line_base((uint32_t)(t * WARPS)); };
    // G16 (TILED with PF set): the tile is gathered by 16-byte cp.async into [m][n][16 lines]
    // rows of 64 B whose 16-byte chunks are XOR-swizzled by (n >> 1) & 3 (8 copies per
    // thread instead of 32); a warp's column reads are then 4-way bank conflicted
    constexpr bool G16 = TILED && PF;
    constexpr int CPR = TW / 4;  // 16-byte chunks per stage row (TW lines)
    auto g16_idx = [](int m, int n, int l) {
        return (m * N + n) * TW + ((((l >> 2) ^ (TW == 16 ? (n >> 1) : 0)) & (CPR - 1)) << 2) + (l & 3);
    };
    auto fetch_tile = [&](int64_t t, int64_t tb0) {
        if constexpr (TMA) {
            if (threadIdx.x == 0 && t < ntiles) {
                const uint32_t l0 = (uint32_t)(t * WARPS), a = l0 / uD0, x0 = l0 - a * uD0, c4 = a / uD1,
                               c3 = a - c4 * uD1;
                const uint32_t bar = s32(&tbar);
                // the stage was read through the generic proxy (CTA barrier before this call)
                asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
                asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(bar),
                             "r"((uint32_t)(2 * N * TW * 4))
                             : "memory");
#pragma unroll
                for (int m = 0; m < 2; ++m)
#pragma unroll
                    for (int hh = 0; hh < 2; ++hh)
                        asm volatile(
                            "cp.async.bulk.tensor.5d.shared::cluster.global.tile.mbarrier::complete_tx::bytes"
                            " [%0], [%1, {%2, %3, %4, %5, %6}], [%7];" ::"r"(s32(stage + (m * N + hh * 256) * TW)),
                            "l"(&tmap), "r"(x0), "r"(hh * 256), "r"(m), "r"(c3), "r"(c4), "r"(bar)
                            : "memory");
            }
            (void)tb0;
            return;
        }
        if (G16) {
            if (t < ntiles) {
#pragma unroll
                for (int i = 0; i < 8; ++i) {
                    const int q = threadIdx.x + WARPS * 32 * i, c = q & (CPR - 1), n = (q / CPR) & (N - 1),
                              m = q / (CPR * N);
                    const uint32_t dst = (uint32_t)__cvta_generic_to_shared(stage + g16_idx(m, n, 4 * c));
                    asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"(dst),
                                 "l"(g + tb0 + m * ra.cs + (int64_t)n * ra.ss + 4 * c)
                                 : "memory");
                }
            }
        } else if (t < ntiles && WARPS * 32 == 32 * 16) {
            // 32 elements per thread: line l = tid & 15, samples n = (tid >> 4) + 32 i, channel m;
            // addresses advance by constant strides (no per-element index arithmetic)
            const int l = threadIdx.x & 15, n0 = threadIdx.x >> 4;
            const float *s0 = g + tb0 + l + (int64_t)n0 * ra.ss;
            const int64_t step = 32 * ra.ss;
            const uint32_t d0 = (uint32_t)__cvta_generic_to_shared(stage + l * SP + n0);
#pragma unroll
            for (int m = 0; m < 2; ++m) {
                const float *sp = s0 + m * ra.cs;
                const uint32_t dm = d0 + (uint32_t)(m * WARPS * SP * 4);
#pragma unroll
                for (int i = 0; i < 16; ++i)
                    asm volatile("cp.async.ca.shared.global [%0], [%1], 4;" ::"r"(dm + 128u * i), "l"(sp + i * step)
                                 : "memory");
            }
        } else if (t < ntiles) {
            const float *src = g + tb0;
#pragma unroll 4
            for (int e = threadIdx.x; e < 2 * N * WARPS; e += WARPS * 32) {
                const int l = e % WARPS, n = (e / WARPS) % N, m = e / (WARPS * N);
                const uint32_t dst = (uint32_t)__cvta_generic_to_shared(stage + (m * WARPS + l) * SP + n);
                asm volatile("cp.async.ca.shared.global [%0], [%1], 4;" ::"r"(dst),
                             "l"(src + m * ra.cs + (int64_t)n * ra.ss + l)
                             : "memory");
            }
        }
        asm volatile("cp.async.commit_group;" ::: "memory");
    };
    // PF: stage = floats [0, 2N) of the warp buffer, 16-byte aligned (BUF is odd); with TST
    // the buffer carries the outputs, so the stage is a separate [WARPS][2N] region
    float *pstage = (TST && !TILED) ? stage + warp * 2 * N : reinterpret_cast<float *>(buf + (warp & 1));
    auto prefetch_line = [&](int64_t ln) {
        if constexpr (BULK) {
            if (ln < lines && lane == 0) {
                const float *src = g + line_base((uint32_t)ln);
                const uint32_t bar = s32(&lbar[warp]);
                asm volatile("fence.proxy.async.shared::cta;" ::: "memory");  // the buffer was read generically
                asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(bar), "r"(2 * N * 4)
                             : "memory");
#pragma unroll
                for (int m = 0; m < 2; ++m)
                    asm volatile(
                        "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
                            s32(pstage + m * N)),
                        "l"(src + m * ra.cs), "r"(N * 4), "r"(bar)
                        : "memory");
            }
            return;
        }
        if (ln < lines) {
            const float *src = g + line_base((uint32_t)ln);
            const uint32_t d = (uint32_t)__cvta_generic_to_shared(pstage);
#pragma unroll
            for (int i = 0; i < 8; ++i) {
                const int c = lane + 32 * i, m = c >> 7, n = 4 * (c & 127);
                asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"(d + 16u * c), "l"(src + m * ra.cs + n)
                             : "memory");
            }
        }
        asm volatile("cp.async.commit_group;" ::: "memory");
    };
    uint32_t lph = 0;  // BULK: parity of the warp's line barrier
    if constexpr (BULK) {
        if (lane == 0) {
            asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(s32(&lbar[warp])) : "memory");
            asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
        }
        __syncwarp();
    }
    if constexpr (PF && !TILED) prefetch_line((int64_t)blockIdx.x * WARPS + warp);
    uint32_t tph = 0;  // TMA: parity of the tile barrier
    if constexpr (TMA && TILED) {
        if (threadIdx.x == 0) {
            asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(s32(&tbar)) : "memory");
            asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
        }
        __syncthreads();
    }
    // TILED: D0 % WARPS == 0, so a tile's lines share the outer indices: base = tile base + warp s0
    int64_t tbase = 0;
    if constexpr (TILED) {
        if ((int64_t)blockIdx.x < ntiles) tbase = tile_base(blockIdx.x);
        fetch_tile(blockIdx.x, tbase);
    }
    // tile tl = lines tl TW .. + TW - 1; warp -> (half, index): line = blockIdx.x WARPS + warp
    // + k gridDim.x WARPS in every mode
    constexpr int NH = WARPS / TW;
    for (int64_t tl = (int64_t)blockIdx.x * NH + warp / TW; tl < (TILED ? ntiles : (lines + TW - 1) / TW);
         tl += (int64_t)gridDim.x * NH) {
        const int64_t line = tl * TW + warp % TW;
        const int64_t base = TILED ? tbase + warp * ra.s0 : line_base((uint32_t)line);
        const float *g0 = g + base, *g1 = g + base + ra.cs;
        pk x[16];
        float m0 = 0.f, m1 = 0.f;
        if constexpr (TILED) {
            if constexpr (TMA) {
                uint32_t done = 0;
                while (!done)
                    asm volatile(
                        "{ .reg .pred p; mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2; selp.u32 %0, 1, 0, p; }"
                        : "=r"(done)
                        : "r"(s32(&tbar)), "r"(tph)
                        : "memory");
                tph ^= 1u;
            } else {
                asm volatile("cp.async.wait_group 0;" ::: "memory");
                __syncthreads();  // tile tl has landed
            }
            if (line < lines) {
#pragma unroll
                for (int j = 0; j < 16; ++j) {
                    const int n = lane + 32 * j;
                    const float a = G16 ? stage[g16_idx(0, n, warp)] : stage[warp * SP + n];
                    const float b = G16 ? stage[g16_idx(1, n, warp)] : stage[(WARPS + warp) * SP + n];
                    m0 = fmaxf(m0, fabsf(a));
                    m1 = fmaxf(m1, fabsf(b));
                    x[j] = mk(a, b);
                }
            }
            __syncthreads();  // stage consumed: fetch the CTA's next tile while this one is transformed
            if (tl + gridDim.x < ntiles) tbase = tile_base(tl + gridDim.x);
            fetch_tile(tl + gridDim.x, tbase);
            if (line >= lines) continue;
            __syncwarp();  // previous line's reads of buf are complete
        } else if constexpr (PF) {
            if (line >= lines) continue;
            if constexpr (BULK) {
                uint32_t done = 0;
                while (!done)
                    asm volatile(
                        "{ .reg .pred p; mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2; selp.u32 %0, 1, 0, p; }"
                        : "=r"(done)
                        : "r"(s32(&lbar[warp])), "r"(lph)
                        : "memory");
                lph ^= 1u;
            } else {
                asm volatile("cp.async.wait_group 0;" ::: "memory");
            }
            __syncwarp();  // this line's rows have landed in the warp buffer
#pragma unroll
            for (int j = 0; j < 16; ++j) {
                const int n = lane + 32 * j;
                const float a = pstage[n], b = pstage[N + n];
                m0 = fmaxf(m0, fabsf(a));
                m1 = fmaxf(m1, fabsf(b));
                x[j] = mk(a, b);
            }
            __syncwarp();  // stage read: the forward pass may overwrite the buffer
            if constexpr (TST) prefetch_line(line + (int64_t)gridDim.x * WARPS);  // separate stage
        } else {
            if (line >= lines) continue;
            __syncwarp();  // previous line's reads of buf are complete
#pragma unroll
            for (int j = 0; j < 16; ++j) {
                const int64_t n = lane + 32 * j;
                const float a = __ldg(g0 + n * ra.ss), b = __ldg(g1 + n * ra.ss);
                m0 = fmaxf(m0, fabsf(a));
                m1 = fmaxf(m1, fabsf(b));
                x[j] = mk(a, b);
            }
        }
        m0 = warp_max_nonneg(m0);
        m1 = warp_max_nonneg(m1);
        const int E0 = (__float_as_int(m0) >> 23) & 0xff, E1 = (__float_as_int(m1) >> 23) & 0xff;
        const int e0 = E0 == 0 ? 0 : max(-100, min(100, E0 - 126));
        const int e1 = E1 == 0 ? 0 : max(-100, min(100, E1 - 126));
        {  // ---- forward: 512 = 8 x 8 x 8 (Stockham DIT), butterflies b = lane and lane + 32 on
           // every lane in every pass; pass p reads b + 64 j and writes (b / Ls) 8 Ls + b % Ls + Ls k.
           // XOR swizzles keep the 64-bit accesses of each half-warp on 16 bank pairs:
           // s1 (pass-1 output, region buf[512..1023]) for the stride-8 writes and stride-1 reads,
           // s2 (pass-2 output, buf[0..511]) for the (b / 8, b % 8) writes; pass 3 writes the
           // natural-order spectrum with sw3 for the solve.
            auto s1 = [](int a) { return a ^ ((a >> 4) & 15); };
            auto s2 = [](int a) { return a ^ (((a >> 6) & 1) << 3); };
            float2 *R1 = buf + 512;
            const pk sc = mk(pow2f(-e0), pow2f(-e1));
            pk u[8], v[8];
#pragma unroll
            for (int j = 0; j < 8; ++j) {  // n = lane + 64 j (b = lane), lane + 32 + 64 j (b = lane + 32)
                u[j] = mul(x[2 * j], sc);
                v[j] = mul(x[2 * j + 1], sc);
            }
            dft<8, -1>(u);
            dft<8, -1>(v);
#pragma unroll
            for (int k = 0; k < 8; ++k) {  // pass 1 (Ls = 1): outputs 8 b + k
                R1[s1(8 * lane + k)] = f2(u[k]);
                R1[s1(8 * (lane + 32) + k)] = f2(v[k]);
            }
            __syncwarp();
            const int k1 = lane & 7;
#pragma unroll
            for (int j = 0; j < 8; ++j) {  // pass 2 (Ls = 8): twiddle W64^{j (b % 8)}
                u[j] = mk(R1[s1(lane + 64 * j)]);
                v[j] = mk(R1[s1(lane + 32 + 64 * j)]);
            }
#pragma unroll
            for (int j = 1; j < 8; ++j) {
                const pk w = mk(fwt[448 + 8 * (j - 1) + k1]);
                u[j] = pkx::cmul(u[j], w);
                v[j] = pkx::cmul(v[j], w);
            }
            dft<8, -1>(u);
            dft<8, -1>(v);
            const int o2 = 64 * (lane >> 3) + k1;
#pragma unroll
            for (int k = 0; k < 8; ++k) {
                buf[s2(o2 + 8 * k)] = f2(u[k]);
                buf[s2(256 + o2 + 8 * k)] = f2(v[k]);
            }
            __syncwarp();
#pragma unroll
            for (int j = 0; j < 8; ++j) {  // pass 3 (Ls = 64): twiddle W512^{j b}, outputs b + 64 k
                u[j] = mk(buf[s2(lane + 64 * j)]);
                v[j] = mk(buf[s2(lane + 32 + 64 * j)]);
            }
#pragma unroll
            for (int j = 1; j < 8; ++j) {
                u[j] = pkx::cmul(u[j], mk(fwt[64 * (j - 1) + lane]));
                v[j] = pkx::cmul(v[j], mk(fwt[64 * (j - 1) + lane + 32]));
            }
            dft<8, -1>(u);
            dft<8, -1>(v);
            __syncwarp();  // pass-3 reads done: the natural-order writes overlap them
#pragma unroll
            for (int k = 0; k < 8; ++k) {
                buf[sw3(lane + 64 * k)] = f2(u[k]);
                buf[sw3(lane + 32 + 64 * k)] = f2(v[k]);
            }
        }
        __syncwarp();
        pk y[32];

        // ---- solve: classes q = lane + 32 u (u < 8) and q = N/2 (lane 0)
        pk zq[9], zm[9];
#pragma unroll
        for (int u = 0; u < 9; ++u) {
            const int q = u < 8 ? lane + 32 * u : N / 2;
            if (u < 8 || lane == 0) {
                zq[u] = mk(buf[sw3(q)]);
                zm[u] = mk(buf[sw3((N - q) & (N - 1))]);
            }
        }
        __syncwarp();  // forward spectrum read: buf becomes the inverse input
        const float h0 = 0.5f * pow2f(e0), h1 = 0.5f * pow2f(e1);
        auto solve = [&](int u, int q, pk &v0, pk &v1) {
            const pk G0 = mul(add(zq[u], pkx::conj(zm[u])), bc(h0));
            const pk G1 = mul(rot<-1>(sub(zq[u], pkx::conj(zm[u]))), bc(h1));
            if (tb.deriv) {
                // (1, ik): H_j = [[1, ij], [1, i(j+N)]], det = iN, so with d = G/N
                // a(j) = ((j+N) G0 + i G1)/N^2, a(j+N) = (-j G0 - i G1)/N^2, j = q - N
                // (integers times 2^-18: exact in fp32)
                const float jn = (float)(q - N), inv = 1.f / ((float)N * (float)N);
                const pk iG1 = rot<1>(G1);
                v0 = add(mul(G0, bc((jn + (float)N) * inv)), mul(iG1, bc(inv)));
                v1 = sub(mul(G0, bc(-jn * inv)), mul(iG1, bc(inv)));
            } else {
                const int Qq = q * 4;  // [m][l]
                v0 = add(pkx::cmul(G0, mk(ldQ(Qq + 0))), pkx::cmul(G1, mk(ldQ(Qq + 2))));
                v1 = add(pkx::cmul(G0, mk(ldQ(Qq + 1))), pkx::cmul(G1, mk(ldQ(Qq + 3))));
            }
        };
        // inverse input (p1 = 0, 1 share one FFT): Zin(k) = Y(k)(1 + i w^k), w = e^{2 pi i/L}
        float2 wq[16];  // TM: pre-twiddles of this lane's solve outputs (entry 2u + e)
        if constexpr (TM) {
            tld16(tmA + TMW, wq);
            tld16(tmA + TMW + 16, wq + 8);
        }
        auto emit = [&](int p, pk X, float2 wa) {
            const pk P = pkx::cmul(X, mk(TM ? wa : ldwp(p)));
            buf[sw5(p)] = f2(add_rot<1>(X, P));
            buf[sw5(S - p)] = f2(add_rot<1>(pkx::conj(X), pkx::conj(P)));
        };
#pragma unroll
        for (int u = 0; u < 8; ++u) {
            const int q = lane + 32 * u;
            pk v0, v1;
            solve(u, q, v0, v1);
            if (q != 0) {  // elements q - N (-> X[N - q] = conj v0) and q (-> X[q] = v1)
                emit(N - q, pkx::conj(v0), wq[2 * u]);
                emit(q, v1, wq[2 * u + 1]);
            } else {  // q = 0: X[0] = Re a(0); position K = N aliases +-K at k' = K
                const float2 a0 = f2(v1);
                buf[sw5(0)] = make_float2(a0.x, a0.x);  // X + iX, X real
                const pk XK = mul(pkx::conj(v0), bc(0.5f));  // X[K] = conj a(-K)/2
                const pk P = pkx::cmul(XK, mk(TM ? wq[2 * u] : ldwp(K)));
                buf[sw5(K)] = f2(add(add_rot<1>(XK, P), add_rot<1>(pkx::conj(XK), pkx::conj(P))));
            }
        }
        if (lane == 0) {  // q = N/2: elements -N/2, N/2 -> X[N/2] = (a(N/2) + conj a(-N/2))/2
            pk v0, v1;
            solve(8, N / 2, v0, v1);
            emit(N / 2, mul(add(v1, pkx::conj(v0)), bc(0.5f)), ldwp(N / 2));
        }
        __syncwarp();

        // ---- inverse pass 1 (radix 32, Ls = 1)
#pragma unroll
        for (int j = 0; j < 32; ++j) y[j] = mk(buf[sw5(lane + 32 * j)]);
        __syncwarp();
        dft<32, 1>(y);
#pragma unroll
        for (int j = 0; j < 32; ++j) buf[sw5(32 * lane + j)] = f2(y[j]);
        __syncwarp();
        // ---- pass 2 (Ls = 32)
#pragma unroll
        for (int j = 0; j < 32; ++j) y[j] = mk(buf[sw5(lane + 32 * j)]);
        if constexpr (PF && !TILED && !TST) {
            __syncwarp();  // buffer read: the next line's rows may land in it
            prefetch_line(line + (int64_t)gridDim.x * WARPS);
        }
        if constexpr (TM) {
#pragma unroll
            for (int c = 0; c < 4; ++c) {  // twiddles j = 8c+1 .. 8c+8 (j <= 31)
                float2 w[8];
                tld16(tmA + TMI + 16 * c, w);
#pragma unroll
                for (int i = 0; i < 8; ++i)
                    if (8 * c + 1 + i <= 31) y[8 * c + 1 + i] = pkx::cmul(y[8 * c + 1 + i], mk(w[i]));
            }
        } else {
#pragma unroll
            for (int p2 = 0; p2 < 15; ++p2) {
                const float4 w2 = *reinterpret_cast<const float4 *>(iw + 64 * p2 + 2 * lane);
                y[2 * p2 + 1] = pkx::cmul(y[2 * p2 + 1], mk(w2.x, w2.y));
                y[2 * p2 + 2] = pkx::cmul(y[2 * p2 + 2], mk(w2.z, w2.w));
            }
            y[31] = pkx::cmul(y[31], mk(iw[960 + lane]));
        }
        dft<32, 1>(y);
        if constexpr (TST) {
            // lines % WARPS == 0 (launcher), so every warp of the tile gets here
            __syncwarp();  // pass-2 reads of buf are complete
#pragma unroll
            for (int j = 0; j < 32; ++j) buf[lane + 32 * j] = f2(y[j]);  // f[2 p2 + e] at float 2 p2 + e
            // (32-bit quotient as in line_base: lines < 2^31; the 64-bit division here was an emulated
            // sequence of ~100 instructions per thread and tile on the write-out's critical path)
            const uint32_t l0 = (uint32_t)(tl * TW), lq = l0 / uD0;
            float *ob = f + (int64_t)lq * L * ra.D0 + (l0 - lq * uD0);
            {
                __syncthreads();  // the tile's 16 lines are in the warp buffers
                // thread (c, p2): lines 4c..4c+3 of rows 2 p2, 2 p2 + 1 (one 64-bit read per line).
                // 16 lines: c = tid & 3, buffer stride = 1 (mod 16) float2; 8 lines: c = bit 3 of
                // tid, stride = 2 (mod 16): either way a half-warp's reads hit 16 bank pairs
                const int c = TW == 16 ? (threadIdx.x & 3) : ((threadIdx.x >> 3) & 1);
                const int p20 = TW == 16 ? (threadIdx.x >> 2) : ((threadIdx.x & 7) + 8 * (threadIdx.x >> 4));
#pragma unroll 2
                for (int p2 = p20; p2 < L / 2; p2 += WARPS * 32 / CPR) {
                    const float2 u0 = bufs[(4 * c + 0) * BUFS + p2], u1 = bufs[(4 * c + 1) * BUFS + p2];
                    const float2 u2 = bufs[(4 * c + 2) * BUFS + p2], u3 = bufs[(4 * c + 3) * BUFS + p2];
                    __stcs(reinterpret_cast<float4 *>(ob + (2 * p2) * ra.D0) + c, make_float4(u0.x, u1.x, u2.x, u3.x));
                    __stcs(reinterpret_cast<float4 *>(ob + (2 * p2 + 1) * ra.D0) + c, make_float4(u0.y, u1.y, u2.y, u3.y));
                }
                __syncthreads();  // warp buffers free for the next tile
            }
        } else {
            float2 *fo = reinterpret_cast<float2 *>(f + line * (int64_t)L);
#pragma unroll
            for (int j = 0; j < 32; ++j) __stcs(fo + lane + 32 * j, f2(y[j]));
        }
    }
    if (TM) {
        asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
        __syncthreads();
        if (threadIdx.x < 32)
            asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tm_base), "n"(TM_COLS)
                         : "memory");
    }
}

// cuTensorMapEncodeTiled through the runtime's driver entry point (no libcuda link dependency);
// resolved once, thread-safely (function-local static), nullptr when unavailable
void *tensor_map_encoder() {
    static void *const fn = [] {
        void *p = nullptr;
        cudaDriverEntryPointQueryResult q;
        if (cudaGetDriverEntryPointByVersion("cuTensorMapEncodeTiled", &p, 12000, cudaEnableDefault, &q) != cudaSuccess ||
            q != cudaDriverEntryPointSuccess) {
            cudaGetLastError();
            p = nullptr;
        }
        return p;
    }();
    return fn;
}

// Tensor map of the tiled 2D pass input: dims (innermost first) line-in-block x (D0, stride 1),
// sample n (N, stride ss), channel m (2, stride cs), block a1 (D1, stride s1), block b (stride s2),
// fp32; box 16 lines x 256 samples x 1 x 1 x 1, 64-byte swizzle (16-byte chunk c of 64-byte
// row n stored at chunk c ^ ((n >> 1) & 3), the layout of the G16 gather).  The driver entry
// point comes through the runtime (no libcuda link dependency).
static bool encode_tile_map(CUtensorMap *tm, const void *g, const RowAddr &ra, int64_t lines, int N) {
    const auto enc = (PFN_cuTensorMapEncodeTiled_v12000)tensor_map_encoder();
    if (!enc) return false;
    if (ra.s0 != 1 || ra.D0 % 16 != 0 || lines % (ra.D0 * ra.D1) != 0) return false;
    const int64_t nb = lines / (ra.D0 * ra.D1);
    if (ra.D0 >= (1ll << 31) || nb >= (1ll << 31) || ra.D1 >= (1ll << 31)) return false;
    auto okst = [](int64_t s) { return s > 0 && (s * 4) % 16 == 0 && s * 4 < (1ll << 40); };
    const int64_t s1 = ra.D1 > 1 ? ra.s1 : 4, s2 = nb > 1 ? ra.s2 : 4;
    if (!okst(ra.ss) || !okst(ra.cs) || !okst(s1) || !okst(s2)) return false;
    const cuuint64_t dims[5] = {(cuuint64_t)ra.D0, (cuuint64_t)N, 2, (cuuint64_t)ra.D1, (cuuint64_t)nb};
    const cuuint64_t strides[4] = {(cuuint64_t)ra.ss * 4, (cuuint64_t)ra.cs * 4, (cuuint64_t)s1 * 4, (cuuint64_t)s2 * 4};
    const cuuint32_t box[5] = {16, 256, 1, 1, 1}, es[5] = {1, 1, 1, 1, 1};
    return enc(tm, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 5, const_cast<void *>(g), dims, strides, box, es,
               CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_64B, CU_TENSOR_MAP_L2_PROMOTION_L2_128B,
               CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) == CUDA_SUCCESS;
}

bool line_supported(const Axis1D &ax) {
    return ax.dtype == MCI_F32 && !ax.analytic && ax.M == 2 && ax.N == 512 && ax.L == 2048 && ax.S == 1024;
}

size_t line_table_elems(const Axis1D &ax) { return (ax.K + 1) + 512 + 1024; }

bool line_tstore_ok(const Axis1D &ax, const RowAddr &ra, int64_t lines, const void *g, const void *f) {
    if (getenv("MCI_2D_TSTORE") && atoi(getenv("MCI_2D_TSTORE")) == 0) return false;
    const bool tiled_in = ra.s0 == 1 && ra.ss != 1 && ra.ss % 4 == 0;  // adjacent lines, strided samples
    const bool contig_in = ra.ss == 1 && ra.s0 % 4 == 0 &&              // contiguous lines (prefetched)
                           !(getenv("MCI_LINE_PF") && atoi(getenv("MCI_LINE_PF")) == 0);
    return line_supported(ax) && (tiled_in || contig_in) && ra.D0 % 16 == 0 && lines % 16 == 0 &&
           (((uintptr_t)g) & 15) == 0 && (((uintptr_t)f) & 15) == 0 && ra.cs % 4 == 0 && ra.s1 % 4 == 0 &&
           ra.s2 % 4 == 0;
}

cudaError_t launch_line(const Axis1D &ax, const RowAddr &ra, int64_t lines, const void *g, void *f, cudaStream_t st,
                        int *n_launches, bool tstore) {
    if (lines <= 0) return cudaSuccess;
    if (tstore && !line_tstore_ok(ax, ra, lines, g, f)) return cudaErrorInvalidValue;
    if (lines >= ((int64_t)1 << 31) - 64) return cudaErrorInvalidValue;  // 32-bit line quotients
    LineTables tb;
    tb.Qt = (const float2 *)ax.Qt;
    const float2 *base = (const float2 *)ax.rowtab;  // [wp K+1][fwt 32x16][iw 32x32]
    tb.wp = base;
    tb.fwt = tb.wp + (ax.K + 1);
    tb.iw = tb.fwt + 512;
    tb.deriv = ax.bank_deriv01;
    const bool tiled = ra.s0 == 1 && ra.ss != 1 && ra.D0 % 16 == 0 &&
                       (((uintptr_t)g) & 15) == 0 && ra.cs % 4 == 0 && ra.ss % 4 == 0 && ra.s1 % 4 == 0 &&
                       ra.s2 % 4 == 0;
    // contiguous 16-byte-aligned lines: cp.async prefetch of the next line (MCI_LINE_PF=0: direct loads)
    const bool pf = !tiled && ra.ss == 1 && (((uintptr_t)g) & 15) == 0 && ra.cs % 4 == 0 && ra.s0 % 4 == 0 &&
                    ra.s1 % 4 == 0 && ra.s2 % 4 == 0 && !(getenv("MCI_LINE_PF") && atoi(getenv("MCI_LINE_PF")) == 0);
    // tiled or transposed-store: one 16-warp CTA per SM (a tile = 16 lines); else two 8-warp CTAs
    const bool tstore_c = tstore && !tiled;  // untiled transposed store (prefetched contiguous lines)
    if (tstore_c && !pf) return cudaErrorInvalidValue;
    // tiled passes: 16-byte gather into a swizzled [m][n][16] stage (config 5: 0.808 -> 0.775
    // ms); MCI_LINE_G16=0: 4-byte transposing cp.async into [m][l][SP] (A/B)
    const bool g16 = tiled && !(getenv("MCI_LINE_G16") && atoi(getenv("MCI_LINE_G16")) == 0);
    // default: per-lane pre-twiddle and inverse pass-2 twiddle tables in tensor memory;
    // MCI_LINE_VARIANT=1: all tables in shared memory, 2: tensor memory on the tiled path only (A/B)
    const int lv = getenv("MCI_LINE_VARIANT") ? atoi(getenv("MCI_LINE_VARIANT")) : 0;
    const bool tm = lv == 0 || (lv == 2 && tiled);
    // MCI_LINE_CT8=1 (A/B): tiled transposed-store pass as two 8-warp CTAs per SM (8-line tiles,
    // compact shared memory), so one CTA's write-out overlaps the other's transforms
    const bool ct8 = tstore && tiled && g16 && tm && getenv("MCI_LINE_CT8") && atoi(getenv("MCI_LINE_CT8")) == 1;
    const int WARPS = ct8 ? 8 : (tiled || tstore) ? 16 : 8;
    // tiled 16-line transposed-store pass: the tile gather by TMA tensor-map box loads
    // (MCI_LINE_TMA=0: the 16-byte cp.async gather, A/B)
    CUtensorMap tmap;
    memset(&tmap, 0, sizeof(tmap));
    // untiled prefetched lines: the next line by TMA bulk copies (MCI_LINE_TMA=0: 16-byte cp.async)
    const bool bulk = pf && !(getenv("MCI_LINE_TMA") && atoi(getenv("MCI_LINE_TMA")) == 0) && ra.cs % 4 == 0;
    const bool tma = tiled && g16 && tm && !ct8 && !(getenv("MCI_LINE_TMA") && atoi(getenv("MCI_LINE_TMA")) == 0) &&
                     encode_tile_map(&tmap, g, ra, lines, linek::N);
    auto kern = ct8 ? mci_line_kernel<8, true, true, true, true>
                : tma ? (tstore ? mci_line_kernel<16, true, true, true, true, true> : mci_line_kernel<16, true, true, false, true, true>)
                : tstore_c ? (tm ? mci_line_kernel<16, false, true, true, true> : mci_line_kernel<16, false, false, true, true>)
                : (tstore && g16) ? (tm ? mci_line_kernel<16, true, true, true, true> : mci_line_kernel<16, true, false, true, true>)
                : tstore  ? (tm ? mci_line_kernel<16, true, true, true> : mci_line_kernel<16, true, false, true>)
                : (tiled && g16) ? (tm ? mci_line_kernel<16, true, true, false, true> : mci_line_kernel<16, true, false, false, true>)
                : tiled ? (tm ? mci_line_kernel<16, true, true> : mci_line_kernel<16, true, false>)
                : pf    ? (tm ? (bulk ? mci_line_kernel<8, false, true, false, true, true> : mci_line_kernel<8, false, true, false, true>)
                              : mci_line_kernel<8, false, false, false, true>)
                        : (tm ? mci_line_kernel<8, false, true> : mci_line_kernel<8, false, false>);
    const size_t smem = ct8 ? (size_t)(512 + WARPS * (linek::BUF + 1)) * 8 + (size_t)2 * WARPS * linek::SP * 4
                            : (size_t)(linek::NQ * 4 + linek::K + 2 + 512 + 1024 + WARPS * linek::BUF) * 8 +
                                  (tiled ? (size_t)2 * WARPS * linek::SP * 4 : tstore_c ? (size_t)WARPS * 2 * linek::N * 4 : 0) +
                                  (tma ? 1024 : 0);  // TMA: the stage starts at a 1024-byte boundary
    cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    if (e != cudaSuccess) return e;
    int dev = 0, nsm = 148, occ = 1;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, dev);
    cudaFuncSetAttribute(kern, cudaFuncAttributePreferredSharedMemoryCarveout, (int)cudaSharedmemCarveoutMaxShared);
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, kern, WARPS * 32, smem);
    if (getenv("MCI_DEBUG")) {
        cudaFuncAttributes fa;
        cudaFuncGetAttributes(&fa, kern);
        int occ0 = 0;
        cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ0, kern, WARPS * 32, 0);
        size_t avail = 0;
        const cudaError_t ea = cudaOccupancyAvailableDynamicSMemPerBlock(&avail, kern, 2, WARPS * 32);
        if (ea != cudaSuccess) fprintf(stderr, "mci: avail query: %s\n", cudaGetErrorString(ea));
        cudaGetLastError();
        fprintf(stderr, "mci: line kernel warps=%d tiled=%d tstore=%d pf=%d smem=%zu occ=%d occ(smem0)=%d regs=%d static=%zu local=%zu avail2=%zu\n",
                WARPS, (int)tiled, (int)tstore, (int)pf, smem, occ, occ0, fa.numRegs, fa.sharedSizeBytes, fa.localSizeBytes, avail);
    }
    if (occ < 1) occ = 1;
    if (tm && WARPS == 8) {  // (also the CT8 tiled pass)
        // the occupancy query reports one CTA per SM for a kernel that allocates tensor memory;
        // two 8-warp CTAs fit (2 x 256 of the 512 TMEM columns, 2 x 92 KB shared memory, 2 x 32K
        // registers) and run (measured: 0.217 -> 0.202 ms per 65,536 contiguous lines)
        occ = std::max(occ, std::min(linek::TMEM_TOTAL_COLS / linek::TM_COLS, (int)(233472 / (smem + 1024))));
    }
    if (getenv("MCI_LINE_OCC")) occ = atoi(getenv("MCI_LINE_OCC"));  // A/B: CTAs per SM in the grid
    int64_t grid = (int64_t)nsm * occ;
    const int64_t need = (lines + WARPS - 1) / WARPS;
    if (grid > need) grid = need;
    if (n_launches) *n_launches += 1;
    kern<<<(unsigned)grid, WARPS * 32, smem, st>>>((const float *)g, (float *)f, lines, ra, tb, tmap);
    return cudaGetLastError();
}

}  // namespace mci
