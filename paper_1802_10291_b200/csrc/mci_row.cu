// Specialised fused MCI row kernel for the batched real-output shape
// (BASELINE.json configs[1]: M = 3 channels f, f', f'', N = 1024, L = 16384).
//
// Same mathematics as mci_fused.cu (Lemma 1 forward DFT PAPER.md:180-233,
// per-class solve a = D H^{-1} Eq. matrixeqn1, Hermitian-part
// assembly, zero-padded inverse of Eq. DFTexpression), laid
// out for B200:
//   * CTA = G independent row groups of 256 threads (named barriers), sharing
//     one shared-memory copy of the per-class inverse tables Q~;
//   * input rows arrive by TMA bulk copy (cp.async.bulk + mbarrier), the next
//     row is prefetched while the current one is transformed;
//   * forward: two complex 1024-point FFTs (channel pairs), radix 8/8/16;
//   * the solve writes the pre-twiddled inputs of both inverse FFTs directly
//     (Zin_c(k) = Y(k) T_c(k), T_c = w^{2ck} + i w^{(2c+1)k}, w = e^{2 pi i/L});
//   * inverse: two 4096-point FFTs, three register radix-16 passes, 16 points
//     per thread, padded shared-memory exchanges (conflict-free);
//   * the last pass hands results straight to 128-bit streaming stores:
//     thread t owns p2 = t + 256 j and writes f[4 p2 .. 4 p2 + 3].
#include <cstdint>

#include "mci_fft.cuh"
#include "mci_internal.h"

namespace mci {

namespace rowk {

constexpr int NT = 256;

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
__device__ __forceinline__ void group_bar(int id) {
    asm volatile("bar.sync %0, %1;" ::"r"(id), "r"(NT) : "memory");
}

__device__ __forceinline__ int pad16(int a) { return a + (a >> 4); }
__device__ __forceinline__ int pad8(int a) { return a + (a >> 3); }

}  // namespace rowk

// Device tables built by the plan (fp64-rounded), see mci_plan.cpp build_row_tables().
struct RowTables {
    const float2 *Qt;   // [(N/2+1)][M][M]  H^{-1}/N per class
    const float2 *wp;   // [K+1]  e^{+2 pi i p / L}
    const float2 *ft2;  // [8][8]    e^{-2 pi i j k / 64}
    const float2 *ft3;  // [16][64]  e^{-2 pi i j k / 1024}
    const float2 *it2;  // [16][16]  e^{+2 pi i j k / 256}
    const float2 *it3;  // [4][256]  e^{+2 pi i 2^e t / 4096}, e = 0..3
};

template <int M, int N, int S, int NPI, int G>
struct RowCfg {
    static constexpr int K = M * N / 2;
    static constexpr int L = 2 * NPI * S;
    static constexpr int NPAIR = (M + 1) / 2;
    static constexpr int NQ = N / 2 + 1;
    static constexpr int FWD_STRIDE = N + N / 8;        // padded forward buffer per pair
    static constexpr int INV_STRIDE = S + S / 16;       // padded inverse buffer
    static constexpr int STAGE_BYTES = M * N * 4;
    // per-group shared layout (bytes)
    static constexpr int OFF_STAGE = 0;
    static constexpr int OFF_BUF = STAGE_BYTES;                       // NPI... inverse buffers (8B each)
    static constexpr int NBUF = NPI < 2 ? 2 : NPI;                    // forward aliases buffer 1
    static constexpr int GROUP_BYTES = STAGE_BYTES + NBUF * INV_STRIDE * 8;
    static constexpr int Q_BYTES = NQ * M * M * 8;
    static constexpr int TAB_BYTES = (8 * 8 + 16 * 64 + 16 * 16) * 8;
    static constexpr int SMEM = G * GROUP_BYTES + Q_BYTES + TAB_BYTES;
    static_assert(N == 1024 && S == 4096, "specialised for N=1024, S=4096");
    static_assert(NPAIR == 2, "two channel pairs (M = 3 or 4)");
    static_assert(S > 2 * K, "no alias bin at K");
    static_assert(2 * FWD_STRIDE <= INV_STRIDE, "forward buffers alias one inverse buffer");
};

template <int M, int N, int S, int NPI, int G>
__global__ void __launch_bounds__(G * rowk::NT, 1)
    mci_row_kernel(const float *__restrict__ g, float *__restrict__ f, int64_t rows, RowTables tb) {
    using namespace rowk;
    using C = RowCfg<M, N, S, NPI, G>;
    constexpr int K = C::K, L = C::L;
    extern __shared__ __align__(128) unsigned char smem[];
    __shared__ __align__(8) uint64_t mbar[G];
    __shared__ float red[G][NT / 32][4];

    const int grp = threadIdx.x / NT;
    const int t = threadIdx.x % NT;
    const int barid = 1 + grp;
    unsigned char *gbase = smem + grp * C::GROUP_BYTES;
    float *stage = reinterpret_cast<float *>(gbase + C::OFF_STAGE);
    float2 *bufA = reinterpret_cast<float2 *>(gbase + C::OFF_BUF);
    float2 *bufB = bufA + C::INV_STRIDE;
    float2 *fwd = bufB;  // forward spectra alias buffer B
    float2 *Qs = reinterpret_cast<float2 *>(smem + G * C::GROUP_BYTES);
    float2 *ft2 = reinterpret_cast<float2 *>(smem + G * C::GROUP_BYTES + C::Q_BYTES);
    float2 *ft3 = ft2 + 64;
    float2 *it2 = ft3 + 16 * 64;

    // ---- one-time setup: shared tables, per-thread pass-3 twiddle bases, barriers
    for (int i = threadIdx.x; i < C::NQ * M * M; i += G * NT) Qs[i] = tb.Qt[i];
    for (int i = threadIdx.x; i < 64; i += G * NT) ft2[i] = tb.ft2[i];
    for (int i = threadIdx.x; i < 16 * 64; i += G * NT) ft3[i] = tb.ft3[i];
    for (int i = threadIdx.x; i < 16 * 16; i += G * NT) it2[i] = tb.it2[i];
    const float2 b1 = tb.it3[t], b2 = tb.it3[256 + t], b4 = tb.it3[512 + t], b8 = tb.it3[768 + t];
    if (t == 0) mbar_init(&mbar[grp], 1);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    __syncthreads();

    const int64_t gid = (int64_t)blockIdx.x * G + grp;
    const int64_t gstride = (int64_t)gridDim.x * G;
    uint32_t phase = 0;
    if (t == 0 && gid < rows) {
        mbar_expect_tx(&mbar[grp], C::STAGE_BYTES);
        tma_load_1d(stage, g + gid * (int64_t)(M * N), C::STAGE_BYTES, &mbar[grp]);
    }

    for (int64_t row = gid; row < rows; row += gstride) {
        mbar_wait(&mbar[grp], phase);
        phase ^= 1;

        // ---- per-channel max |g| -> exact power-of-two scale (see mci_fused.cu)
        {
            float mx[4] = {0.f, 0.f, 0.f, 0.f};
#pragma unroll
            for (int m = 0; m < M; ++m) {
                const float4 v = reinterpret_cast<const float4 *>(stage + m * N)[t];
                mx[m] = fmaxf(fmaxf(fabsf(v.x), fabsf(v.y)), fmaxf(fabsf(v.z), fabsf(v.w)));
#pragma unroll
                for (int o = 16; o; o >>= 1) mx[m] = fmaxf(mx[m], __shfl_xor_sync(0xffffffffu, mx[m], o));
            }
            if ((t & 31) == 0)
#pragma unroll
                for (int m = 0; m < M; ++m) red[grp][t >> 5][m] = mx[m];
        }
        group_bar(barid);  // also: previous row's reads of bufA/bufB are complete
        // exact power-of-two scales: max|g_m| = f 2^e, f in [0.5, 1); multiply by 2^-e before
        // packing, by 2^e after unpacking (bit-built powers of two, no rounding)
        float sdn[4], sup[4];
#pragma unroll
        for (int m = 0; m < 4; ++m) {
            float v = 0.f;
            if (m < M)
#pragma unroll
                for (int w = 0; w < NT / 32; ++w) v = fmaxf(v, red[grp][w][m]);
            const int E = (__float_as_int(v) >> 23) & 0xff;
            const int e = E == 0 ? 0 : max(-100, min(100, E - 126));
            sdn[m] = __int_as_float((127 - e) << 23);
            sup[m] = __int_as_float((127 + e) << 23);
        }

        // ---- forward pass F1: radix 8, Ls = 1 (reads the staged rows, applies the scales)
        {
            const int c = t >> 7, i = t & 127;
            const float *g0 = stage + (2 * c) * N;
            const float *g1 = stage + (2 * c + 1) * N;
            const float s0 = c ? sdn[2] : sdn[0], s1 = c ? sdn[3] : sdn[1];
            float2 x[8];
#pragma unroll
            for (int j = 0; j < 8; ++j) {
                const float re = g0[i + 128 * j];
                const float im = (2 * c + 1 < M) ? g1[i + 128 * j] : 0.f;
                x[j] = make_float2(re * s0, im * s1);
            }
            dft<8, -1>(x);
            float2 *F = fwd + c * C::FWD_STRIDE;
#pragma unroll
            for (int j = 0; j < 8; ++j) F[pad8(8 * i + j)] = x[j];
        }
        group_bar(barid);
        // the staged input has been consumed: prefetch the next row
        if (t == 0 && row + gstride < rows) {
            asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
            mbar_expect_tx(&mbar[grp], C::STAGE_BYTES);
            tma_load_1d(stage, g + (row + gstride) * (int64_t)(M * N), C::STAGE_BYTES, &mbar[grp]);
        }
        // ---- F2: radix 8, Ls = 8
        {
            const int c = t >> 7, i = t & 127, k = i & 7;
            float2 *F = fwd + c * C::FWD_STRIDE;
            float2 x[8];
#pragma unroll
            for (int j = 0; j < 8; ++j) x[j] = F[pad8(i + 128 * j)];
            group_bar(barid);
#pragma unroll
            for (int j = 1; j < 8; ++j) x[j] = cmul(x[j], ft2[j * 8 + k]);
            dft<8, -1>(x);
#pragma unroll
            for (int j = 0; j < 8; ++j) F[pad8((i - k) * 8 + k + 8 * j)] = x[j];
        }
        group_bar(barid);
        // ---- F3: radix 16, Ls = 64 (in place on own positions)
        if (t < 128) {
            const int c = t >> 6, i = t & 63;
            float2 *F = fwd + c * C::FWD_STRIDE;
            float2 x[16];
#pragma unroll
            for (int j = 0; j < 16; ++j) x[j] = F[pad8(i + 64 * j)];
#pragma unroll
            for (int j = 1; j < 16; ++j) x[j] = cmul(x[j], ft3[j * 64 + i]);
            dft<16, -1>(x);
#pragma unroll
            for (int j = 0; j < 16; ++j) F[pad8(i + 64 * j)] = x[j];
        }
        group_bar(barid);

        // ---- solve (M = 3: j_q = q - N for 0 < q < N/2, elements q - N, q, q + N).
        // Thread t owns classes t and t + 256; thread 0 also the two self-mirror
        // classes q = 0 and q* = N/2 (Hermitian-part averaging).
        static_assert(M == 3, "solve specialised for M = 3");
        float2 zq[3][2], zm[3][2];
#pragma unroll
        for (int u = 0; u < 3; ++u) {
            const int q = (u < 2) ? t + 256 * u : N / 2;
            const int qm = (N - q) & (N - 1);
            if (u < 2 || t == 0) {
#pragma unroll
                for (int c = 0; c < 2; ++c) {
                    zq[u][c] = fwd[c * C::FWD_STRIDE + pad8(q)];
                    zm[u][c] = fwd[c * C::FWD_STRIDE + pad8(qm)];
                }
            }
        }
        group_bar(barid);  // forward spectra read: buffer B may now be overwritten

        // write the pre-twiddled inputs of both inverse FFTs for position p with
        // value X = X[p]:  Zin_A(k) = X (1 + i w^k), Zin_B(k) = X (w^2k + i w^3k),
        // and the mirrored k' = S - p with conj(X) (Hermitian spectrum).
        auto emit = [&](int p, float2 X) {
            const float2 a = __ldg(tb.wp + p);
            const float2 P1 = cmul(X, a);
            bufA[pad16(p)] = make_float2(X.x - P1.y, X.y + P1.x);
            if (p > 0) bufA[pad16(S - p)] = make_float2(X.x + P1.y, -X.y + P1.x);
            if constexpr (NPI == 2) {
                const float2 P2 = cmul(P1, a);
                const float2 P3 = cmul(P2, a);
                bufB[pad16(p)] = make_float2(P2.x - P3.y, P2.y + P3.x);
                if (p > 0) bufB[pad16(S - p)] = make_float2(P2.x + P3.y, -P2.y + P3.x);
            }
        };
        auto solve = [&](int u, int q, float2 *v) {
            float2 gm[3];
#pragma unroll
            for (int m = 0; m < 3; ++m) {
                const float2 a = zq[u][m >> 1], b = cconj(zm[u][m >> 1]);
                const float2 w = (m & 1) ? make_float2(0.5f * (a.y - b.y), -0.5f * (a.x - b.x))
                                         : make_float2(0.5f * (a.x + b.x), 0.5f * (a.y + b.y));
                gm[m] = make_float2(w.x * sup[m], w.y * sup[m]);
            }
            const float2 *Qq = Qs + q * 9;
#pragma unroll
            for (int l = 0; l < 3; ++l) {
                float2 acc = make_float2(0.f, 0.f);
#pragma unroll
                for (int m = 0; m < 3; ++m) {
                    const float2 qv = Qq[m * 3 + l];
                    acc.x = fmaf(gm[m].x, qv.x, fmaf(-gm[m].y, qv.y, acc.x));
                    acc.y = fmaf(gm[m].x, qv.y, fmaf(gm[m].y, qv.x, acc.y));
                }
                v[l] = acc;
            }
        };
#pragma unroll
        for (int u = 0; u < 2; ++u) {
            const int q = t + 256 * u;
            float2 v[3];
            solve(u, q, v);
            if (q != 0) {
                emit(N - q, cconj(v[0]));
                emit(q, v[1]);
                emit(q + N, v[2]);
            } else {  // q = 0: elements -N, 0, N
                emit(0, make_float2(v[1].x, 0.f));
                emit(N, make_float2(0.5f * (v[2].x + v[0].x), 0.5f * (v[2].y - v[0].y)));
            }
        }
        if (t == 0) {  // q* = N/2: elements -3N/2 = -K, -N/2, N/2
            float2 v[3];
            solve(2, N / 2, v);
            emit(K, make_float2(0.5f * v[0].x, -0.5f * v[0].y));
            emit(N / 2, make_float2(0.5f * (v[2].x + v[1].x), 0.5f * (v[2].y - v[1].y)));
        }
        group_bar(barid);

        // ---- inverse FFTs: three radix-16 passes, A and B interleaved around barriers
        float2 xa[16], xb[16];
        // I1 loads (Ls = 1): zero-padding positions (K, S-K) are not read
#pragma unroll
        for (int j = 0; j < 16; ++j) {
            const int kp = t + 256 * j;
            const bool nz = (kp <= K) || (kp >= S - K);
            xa[j] = nz ? bufA[pad16(kp)] : make_float2(0.f, 0.f);
        }
        group_bar(barid);
        dft<16, 1>(xa);
#pragma unroll
        for (int j = 0; j < 16; ++j) bufA[pad16(16 * t + j)] = xa[j];
        if constexpr (NPI == 2) {
#pragma unroll
            for (int j = 0; j < 16; ++j) {
                const int kp = t + 256 * j;
                const bool nz = (kp <= K) || (kp >= S - K);
                xb[j] = nz ? bufB[pad16(kp)] : make_float2(0.f, 0.f);
            }
        }
        group_bar(barid);
        // I2 (Ls = 16): twiddles w256^{j k}, k = t & 15
        const int k2 = t & 15;
        if constexpr (NPI == 2) {
            dft<16, 1>(xb);
#pragma unroll
            for (int j = 0; j < 16; ++j) bufB[pad16(16 * t + j)] = xb[j];
        }
#pragma unroll
        for (int j = 0; j < 16; ++j) xa[j] = bufA[pad16(t + 256 * j)];
        group_bar(barid);
#pragma unroll
        for (int j = 1; j < 16; ++j) xa[j] = cmul(xa[j], it2[j * 16 + k2]);
        dft<16, 1>(xa);
#pragma unroll
        for (int j = 0; j < 16; ++j) bufA[pad16((t - k2) * 16 + k2 + 16 * j)] = xa[j];
        if constexpr (NPI == 2) {
#pragma unroll
            for (int j = 0; j < 16; ++j) xb[j] = bufB[pad16(t + 256 * j)];
        }
        group_bar(barid);
        if constexpr (NPI == 2) {
#pragma unroll
            for (int j = 1; j < 16; ++j) xb[j] = cmul(xb[j], it2[j * 16 + k2]);
            dft<16, 1>(xb);
#pragma unroll
            for (int j = 0; j < 16; ++j) bufB[pad16((t - k2) * 16 + k2 + 16 * j)] = xb[j];
        }
        // I3 (Ls = 256): twiddles w4096^{j t} from the per-thread bases b1, b2, b4, b8
        float2 tw[16];
        tw[1] = b1; tw[2] = b2; tw[4] = b4; tw[8] = b8;
        tw[3] = cmul(b2, b1);
        tw[5] = cmul(b4, b1); tw[6] = cmul(b4, b2); tw[7] = cmul(b4, tw[3]);
#pragma unroll
        for (int j = 1; j < 8; ++j) tw[8 + j] = cmul(b8, tw[j]);
#pragma unroll
        for (int j = 0; j < 16; ++j) xa[j] = bufA[pad16(t + 256 * j)];
#pragma unroll
        for (int j = 1; j < 16; ++j) xa[j] = cmul(xa[j], tw[j]);
        dft<16, 1>(xa);
        float *frow = f + row * (int64_t)L;
        if constexpr (NPI == 2) {
            group_bar(barid);
#pragma unroll
            for (int j = 0; j < 16; ++j) xb[j] = bufB[pad16(t + 256 * j)];
#pragma unroll
            for (int j = 1; j < 16; ++j) xb[j] = cmul(xb[j], tw[j]);
            dft<16, 1>(xb);
#pragma unroll
            for (int j = 0; j < 16; ++j)
                __stcs(reinterpret_cast<float4 *>(frow) + (t + 256 * j), make_float4(xa[j].x, xa[j].y, xb[j].x, xb[j].y));
        } else {
#pragma unroll
            for (int j = 0; j < 16; ++j)
                __stcs(reinterpret_cast<float2 *>(frow) + (t + 256 * j), xa[j]);
        }
    }
}

// ---------------------------------------------------------------------------------------
template <int M, int NPI, int G>
static cudaError_t row_launch_t(const RowTables &tb, int64_t rows, const float *g, float *f, cudaStream_t st) {
    using C = RowCfg<M, 1024, 4096, NPI, G>;
    auto kern = mci_row_kernel<M, 1024, 4096, NPI, G>;
    cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, C::SMEM);
    if (e != cudaSuccess) return e;
    int dev = 0, nsm = 148;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, dev);
    int64_t grid = nsm;
    const int64_t need = (rows + G - 1) / G;
    if (grid > need) grid = need;
    kern<<<(unsigned)grid, G * rowk::NT, C::SMEM, st>>>(g, f, rows, tb);
    return cudaGetLastError();
}

bool row_supported(const Axis1D &ax) {
    return ax.dtype == MCI_F32 && !ax.analytic && ax.N == 1024 && ax.S == 4096 && ax.M == 3 &&
           (ax.R == 2 || ax.R == 4) && ax.S > 2 * ax.K;
}

cudaError_t launch_row(const Axis1D &ax, const void *rowtab, int64_t rows, const void *g, void *f, cudaStream_t st,
                       int *n_launches) {
    if (rows <= 0) return cudaSuccess;
    const float2 *base = (const float2 *)rowtab;
    RowTables tb;
    tb.Qt = (const float2 *)ax.Qt;
    // layout written by mci_plan.cpp: [wp: K+1][ft2: 64][ft3: 1024][it2: 256][it3: 1024]
    tb.wp = base;
    tb.ft2 = tb.wp + (ax.K + 1);
    tb.ft3 = tb.ft2 + 64;
    tb.it2 = tb.ft3 + 1024;
    tb.it3 = tb.it2 + 256;
    if (n_launches) *n_launches += 1;
    const float *gg = (const float *)g;
    float *ff = (float *)f;
    return ax.R == 4 ? row_launch_t<3, 2, 2>(tb, rows, gg, ff, st) : row_launch_t<3, 1, 2>(tb, rows, gg, ff, st);
}

}  // namespace mci
