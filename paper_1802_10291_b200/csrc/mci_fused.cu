// Fused per-row MCI kernel (sm_100a): one CTA streams whole rows
//   load M channel rows -> forward DFT per channel (Lemma 1)
//   -> per-class solve a = D H^{-1} (Eq. matrixeqn1)
//   -> Hermitian-part assembly X[0..K] (real output Re T_N f)
//   -> zero-pad + inverse FFT to L points (Eq. DFTexpression)
//   -> store f (and Hf via the analytic spectrum, Example 4 PAPER.md:436-464).
//
// Inverse transform layout (B200 design, not the paper's): L = R*S with
// S >= 2K (real) or S >= K (analytic).  Output index p = R*p2 + p1 is the S-point
// inverse DFT over k' = k mod S of W_{p1}(k) = Y(k) e^{2 pi i k p1/L}: a pruned
// first decimation-in-frequency stage (the other R-1 inputs of every radix-R
// butterfly are zero-padding).  In real mode two p1 share one complex FFT
// (f_{p1a} + i f_{p1b}); in analytic mode z = f + i Hf at one p1.
// All arithmetic in T (float or double); twiddles from fp64-rounded tables.
#include <algorithm>
#include <cstdio>
#include <cstdlib>

#include "mci_fft.cuh"
#include "mci_internal.h"

namespace mci {

template <typename T> struct FusedArgs {
    int M, N, K, L, R, analytic, G;
    int64_t rows;
    RowAddr ra;
    const T *g;
    T *f, *hf;
    const cv<T> *Qt;
    const cv<T> *twF;
    int64_t TW;
    const cv<T> *twLhi, *twLlo;
    int LOB;  // log2 of the low table size
};

template <typename T> __device__ __forceinline__ cv<T> twL(const FusedArgs<T> &a, int64_t m) {
    m &= (int64_t)a.L - 1;
    cv<T> h = __ldg(a.twLhi + (m >> a.LOB));
    cv<T> l = __ldg(a.twLlo + (m & ((1 << a.LOB) - 1)));
    return cmul(h, l);
}

template <typename T> __device__ __forceinline__ void store_run(T *dst, const T *v, int n) {
    // n consecutive values starting at dst; vectorise when aligned
    if constexpr (sizeof(T) == 4) {
        if (n % 4 == 0 && ((uintptr_t)dst & 15) == 0) {
            for (int j = 0; j < n; j += 4)
                *reinterpret_cast<float4 *>(dst + j) = make_float4(v[j], v[j + 1], v[j + 2], v[j + 3]);
            return;
        }
        if (n % 2 == 0 && ((uintptr_t)dst & 7) == 0) {
            for (int j = 0; j < n; j += 2) *reinterpret_cast<float2 *>(dst + j) = make_float2(v[j], v[j + 1]);
            return;
        }
    } else {
        if (n % 2 == 0 && ((uintptr_t)dst & 15) == 0) {
            for (int j = 0; j < n; j += 2) *reinterpret_cast<double2 *>(dst + j) = make_double2(v[j], v[j + 1]);
            return;
        }
    }
    for (int j = 0; j < n; ++j) dst[j] = v[j];
}

template <typename T, int S, int NT>
__global__ void __launch_bounds__(NT) mci_fused_kernel(const FusedArgs<T> a) {
    using V = cv<T>;
    extern __shared__ __align__(16) unsigned char smem_raw[];
    V *X = reinterpret_cast<V *>(smem_raw);
    const int K = a.K, N = a.N, M = a.M, R = a.R, L = a.L;
    const int xsz = (K + 2) & ~1;
    V *slots = X + xsz;
    const int npair = (M + 1) / 2;
    V *zA = slots;
    V *zB = slots + npair * N;
    const int ns = a.analytic ? a.G : (R > 1 ? R / 2 : 1);
    const int tid = threadIdx.x;
    __shared__ T red[NT / 32];
    __shared__ int escale[8];

    for (int64_t row = blockIdx.x; row < a.rows; row += gridDim.x) {
        // ---- 1. load channel rows as complex pairs z_c = g_{2c} + i g_{2c+1}
        const RowAddr &ra = a.ra;
        const int64_t base = (row / (ra.D0 * ra.D1)) * ra.s2 + ((row / ra.D0) % ra.D1) * ra.s1 + (row % ra.D0) * ra.s0;
        // Two real channels share one complex FFT; channels of very different
        // magnitude (f vs f'' ~ K^2 f) would leak rounding error into each other,
        // so each channel is first scaled by an exact power of two to unit range
        // and the scale is undone after unpacking (no rounding is introduced).
        for (int c = 0; c < npair; ++c) {
            T m0 = 0, m1 = 0;
            for (int n = tid; n < N; n += NT) {
                T re = __ldg(a.g + base + (int64_t)(2 * c) * ra.cs + (int64_t)n * ra.ss);
                T im = (2 * c + 1 < M) ? __ldg(a.g + base + (int64_t)(2 * c + 1) * ra.cs + (int64_t)n * ra.ss) : T(0);
                zA[c * N + n] = V{re, im};
                m0 = fmax(m0, fabs(re));
                m1 = fmax(m1, fabs(im));
            }
            m0 = block_max<NT>(m0, red);
            m1 = block_max<NT>(m1, red);
            if (tid == 0) {
                int e0 = 0, e1 = 0;
                if (m0 > 0) frexp(m0, &e0);
                if (m1 > 0) frexp(m1, &e1);
                escale[2 * c] = e0;
                escale[2 * c + 1] = e1;
            }
        }
        __syncthreads();
        for (int idx = tid; idx < npair * N; idx += NT) {
            const int c = idx / N;
            V z = zA[idx];
            zA[idx] = V{ldexp(z.x, -escale[2 * c]), ldexp(z.y, -escale[2 * c + 1])};
        }
        __syncthreads();
        // ---- 2. forward DFT of every pair, G_c[q] = sum_n z_c[n] e^{-2 pi i q n/N}
        V *Z = block_fft_rt<T, -1>(zA, zB, N, npair, N, a.twF, a.TW);
        // ---- 3. per-class solve and Hermitian-part assembly
        for (int q = tid; q <= N / 2; q += NT) {
            const int qm = (N - q) & (N - 1);
            const int jq = -K + (((q + K) % N) + N) % N;  // j_q in [-K, -K+N), j_q = q mod N
            V v[8];
#pragma unroll
            for (int l = 0; l < 8; ++l) v[l] = V{0, 0};
            for (int m = 0; m < M; ++m) {
                V zc = Z[(m >> 1) * N + q], zm = cconj(Z[(m >> 1) * N + qm]);
                V gm = (m & 1) ? V{(T)0.5 * (zc.y - zm.y), (T)-0.5 * (zc.x - zm.x)}   // (zc - zm)/(2i)
                               : V{(T)0.5 * (zc.x + zm.x), (T)0.5 * (zc.y + zm.y)};   // (zc + zm)/2
                gm = V{ldexp(gm.x, escale[m]), ldexp(gm.y, escale[m])};
                const V *qrow = a.Qt + ((int64_t)q * M + m) * M;
                for (int l = 0; l < M && l < 8; ++l) v[l] = cadd(v[l], cmul(gm, __ldg(qrow + l)));
            }
            const bool selfm = (q == 0) || (2 * q == N);
            for (int l = 0; l < M; ++l) {
                const int k = jq + l * N;
                if (!selfm) {
                    if (k > 0) X[k] = v[l];
                    else X[-k] = cconj(v[l]);
                } else {
                    // X[p] = (a(p) + conj a(-p))/2 within the class (a = 0 out of band)
                    const int lm = (-k - jq);
                    const bool neg_in = (lm >= 0) && (lm % N == 0) && (lm / N < M);
                    if (k >= 0 || !neg_in) {
                        const int p = k >= 0 ? k : -k;
                        V ap = V{0, 0}, an = V{0, 0};
                        const int lp = p - jq, ln = -p - jq;
                        if (lp >= 0 && lp % N == 0 && lp / N < M) ap = v[lp / N];
                        if (ln >= 0 && ln % N == 0 && ln / N < M) an = v[ln / N];
                        X[p] = V{(T)0.5 * (ap.x + an.x), (T)0.5 * (ap.y - an.y)};
                    }
                }
            }
        }
        __syncthreads();
        // ---- 4. pre-twiddle, inverse FFTs, stores
        const int S2 = S;
        const int ngroups = a.analytic ? (R / ns) : 1;
        for (int grp = 0; grp < ngroups; ++grp) {
            for (int idx = tid; idx < ns * S2; idx += NT) {
                const int c = idx / S2, kp = idx - c * S2;
                V acc = V{0, 0};
                if (!a.analytic) {
                    const int pa = 2 * c, pb = 2 * c + 1;
#pragma unroll
                    for (int w = 0; w < 2; ++w) {
                        const int k = w == 0 ? kp : kp - S2;
                        if (k > K || k < -K) continue;
                        const int ak = k >= 0 ? k : -k;
                        V y = X[ak];
                        if (k < 0) y = cconj(y);
                        V ta = twL(a, (int64_t)ak * pa), tb = twL(a, (int64_t)ak * pb);
                        if (k < 0) { ta = cconj(ta); tb = cconj(tb); }
                        V wa = cmul(y, ta);
                        V wb = (pb < R) ? cmul(y, tb) : V{0, 0};
                        acc = cadd(acc, V{wa.x - wb.y, wa.y + wb.x});  // wa + i wb
                    }
                } else {
                    const int p1 = grp * ns + c;
#pragma unroll
                    for (int w = 0; w < 2; ++w) {
                        const int k = kp + w * S2;
                        if (k > K) continue;
                        V z = X[k];
                        if (k > 0) z = cscale(z, (T)2);
                        acc = cadd(acc, cmul(z, twL(a, (int64_t)k * p1)));
                    }
                }
                slots[idx] = acc;
            }
            __syncthreads();
            for (int c = 0; c < ns; ++c) block_fft_ct<T, S, 1, 1, NT, 1>(slots + c * S, S, a.twF, a.TW);
            // copy-out
            T *frow = a.f + row * (int64_t)L;
            if (!a.analytic) {
                for (int p2 = tid; p2 < S2; p2 += NT) {
                    T vals[32];
                    for (int c = 0; c < ns; ++c) {
                        V z = slots[c * S2 + p2];
                        vals[2 * c] = z.x;
                        vals[2 * c + 1] = z.y;
                    }
                    store_run<T>(frow + (int64_t)R * p2, vals, R);
                }
            } else {
                T *hrow = a.hf + row * (int64_t)L;
                for (int p2 = tid; p2 < S2; p2 += NT) {
                    T vf[16], vh[16];
                    for (int c = 0; c < ns; ++c) {
                        V z = slots[c * S2 + p2];
                        vf[c] = z.x;
                        vh[c] = z.y;
                    }
                    store_run<T>(frow + (int64_t)R * p2 + grp * ns, vf, ns);
                    store_run<T>(hrow + (int64_t)R * p2 + grp * ns, vh, ns);
                }
            }
            __syncthreads();
        }
    }
}

// ---------------------------------------------------------------------------------------
static int pick_threads(int64_t S) { return S >= 4096 ? 256 : (S >= 1024 ? 128 : 64); }

static int ns_of(const Axis1D &ax) {
    if (ax.analytic) return (int)(ax.R < 2 ? ax.R : 2);
    return ax.R > 1 ? (int)(ax.R / 2) : 1;
}

size_t fused_smem_bytes(const Axis1D &ax) {
    const size_t vs = ax.dtype == MCI_F64 ? 16 : 8;
    const int64_t xsz = (ax.K + 2) & ~1LL;
    const int64_t npair = (ax.M + 1) / 2;
    int64_t slots = (int64_t)ns_of(ax) * ax.S;
    if (2 * npair * ax.N > slots) slots = 2 * npair * ax.N;
    return (size_t)(xsz + slots) * vs;
}

bool fused_supported(const Axis1D &ax) {
    if (ax.S < 16 || ax.S > 8192 || ax.N > 8192 || ax.M > 8) return false;
    if (!ax.analytic && ax.R > 32) return false;
    return fused_smem_bytes(ax) <= 200 * 1024;
}

template <typename T, int S, int NT>
static cudaError_t launch_t(const Axis1D &ax, const RowAddr &ra, int64_t rows, const void *g, void *f, void *hf,
                           cudaStream_t st) {
    FusedArgs<T> a;
    a.M = ax.M; a.N = (int)ax.N; a.K = (int)ax.K; a.L = (int)ax.L; a.R = (int)ax.R;
    a.analytic = ax.analytic; a.G = ns_of(ax);
    a.rows = rows; a.ra = ra;
    a.g = (const T *)g; a.f = (T *)f; a.hf = (T *)hf;
    a.Qt = (const cv<T> *)ax.Qt; a.twF = (const cv<T> *)ax.twF; a.TW = ax.TW;
    a.twLhi = (const cv<T> *)ax.twLhi; a.twLlo = (const cv<T> *)ax.twLlo;
    a.LOB = ilog2c(ax.LO);
    const size_t smem = fused_smem_bytes(ax);
    auto kern = mci_fused_kernel<T, S, NT>;
    cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    if (e != cudaSuccess) return e;
    int dev = 0, nsm = 148, occ = 1;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, dev);
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, kern, NT, smem);
    if (occ < 1) occ = 1;
    // Analytic (f + i Hf) rows write f[R p2 + p1] in partial 32-byte sectors that are
    // completed by later p1 groups of the same row; bound the rows in flight so the
    // partially written output (rows x 8 L bytes) stays L2-resident (126 MB).
    if (ax.analytic) {
        const int64_t row_bytes = 8 * ax.L;
        const int64_t max_rows = (64ll << 20) / row_bytes;
        if ((int64_t)nsm * occ > max_rows) occ = (int)std::max<int64_t>(1, max_rows / nsm);
    }
    if (const char *e = getenv("MCI_FUSED_CTAS_PER_SM")) occ = std::max(1, atoi(e));
    int64_t grid = (int64_t)nsm * occ;
    if (grid > rows) grid = rows;
    kern<<<(unsigned)grid, NT, smem, st>>>(a);
    return cudaGetLastError();
}

template <typename T>
static cudaError_t dispatch_S(const Axis1D &ax, const RowAddr &ra, int64_t rows, const void *g, void *f, void *hf,
                              cudaStream_t st) {
    switch (ax.S) {
    case 16: return launch_t<T, 16, 64>(ax, ra, rows, g, f, hf, st);
    case 32: return launch_t<T, 32, 64>(ax, ra, rows, g, f, hf, st);
    case 64: return launch_t<T, 64, 64>(ax, ra, rows, g, f, hf, st);
    case 128: return launch_t<T, 128, 64>(ax, ra, rows, g, f, hf, st);
    case 256: return launch_t<T, 256, 64>(ax, ra, rows, g, f, hf, st);
    case 512: return launch_t<T, 512, 64>(ax, ra, rows, g, f, hf, st);
    case 1024: return launch_t<T, 1024, 128>(ax, ra, rows, g, f, hf, st);
    case 2048: return launch_t<T, 2048, 128>(ax, ra, rows, g, f, hf, st);
    case 4096: return launch_t<T, 4096, 256>(ax, ra, rows, g, f, hf, st);
    case 8192: return launch_t<T, 8192, 256>(ax, ra, rows, g, f, hf, st);
    }
    return cudaErrorInvalidValue;
}

cudaError_t launch_fused(const Axis1D &ax, const RowAddr &ra, int64_t rows, const void *g, void *f, void *hf,
                         cudaStream_t st, int *n_launches) {
    if (rows <= 0) return cudaSuccess;
    (void)pick_threads;
    if (n_launches) *n_launches += 1;
    if (ax.dtype == MCI_F64) return dispatch_S<double>(ax, ra, rows, g, f, hf, st);
    return dispatch_S<float>(ax, ra, rows, g, f, hf, st);
}

}  // namespace mci
