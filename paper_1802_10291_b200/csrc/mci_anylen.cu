// MCI for arbitrary sample and output lengths: any N >= 2,
// any L with L % N == 0 and L >= M N, even or odd M N.  The paper's SISR images
// need this (low-resolution widths 107, 120, 160, 166, 170 = 321..510 / 3,
// PAPER.md:896-931) and so do Examples 1-2's odd bands.
//
// Mathematics (same steps as mci_fused.cu, generalised):
//   band k in [K1, K1 + MN), K1 = -floor(MN/2) (odd MN: the symmetric band);
//   forward DFT of each channel (Lemma 1), channels paired into
//   complex FFTs after exact power-of-two scaling;
//   per-class solve a(j_q + l N) = sum_m G_m[q] Q~_q[m][l] for every class q in [0, N)
//   (Eq. matrixeqn1), j_q = the element of [K1, K1 + N) = q (mod N);
//   Hermitian part Xf(k) = (a(k) + conj a(-k)) / 2 (a = 0 out of band), so that
//   Re T_N f(t) = sum_k Xf(k) e^{ikt};
//   inverse DFT of length L of Xf placed at k mod L (the k = +-L/2 pair of an even
//   band with L = MN folds onto one bin) -> real f; for Hf the one-sided spectrum
//   Z(0) = Xf(0), Z(k) = 2 Xf(k) (Example 4) gives z = f + i Hf.
// FFTs: runtime mixed-radix Stockham passes in shared memory (radix 4, 2, 3, 5 and 7
// codelets; any other prime factor p as a direct p-point pass parallel over its
// outputs), twiddles from the plan's fp64-rounded root tables.  One CTA per row.
#include <cstdint>

#include "mci_fft.cuh"
#include "mci_internal.h"

namespace mci {

template <typename T> struct AnyArgs {
    int M, N, L, K1, Kmax, MN, analytic;
    AnyRadix rn, rl;  // radix plans of the forward (N) and inverse (L) transforms
    int64_t rows;
    RowAddr ra;
    const T *g;
    T *f, *hf;
    const cv<T> *Q;    // [N][M][M]  H_{j_q}^{-1}[m][l] / N for every class q
    const cv<T> *twN;  // [N] e^{-2 pi i m / N}
    const cv<T> *twL;  // [L] e^{+2 pi i m / L}
};

namespace anyk {

template <typename V> __device__ __forceinline__ V crot(V a, int s) {  // a * (s i)
    return s > 0 ? V{-a.y, a.x} : V{a.y, -a.x};
}

// one Stockham pass of radix r over `cnt` transforms of length n stored with stride n:
// butterfly b in [0, n/r), k = b mod Ls: x_j = in[b + j n/r] * w^{j k}, w = root^(n/(Ls r)),
// out[(b - k) r + k + j Ls] = DFT_r(x)_j.  `root(m)` = e^{s 2 pi i m / n}.
template <typename T, int NT>
__device__ void stockham_pass(const cv<T> *in, cv<T> *out, int n, int cnt, int r, int Ls, int s, const cv<T> *root) {
    using V = cv<T>;
    const int nb = n / r, tws = n / (Ls * r);
    if (r <= 7 && r != 6) {
        for (int idx = threadIdx.x; idx < cnt * nb; idx += NT) {
            const int c = idx / nb, b = idx - c * nb, k = b % Ls;
            const V *src = in + (int64_t)c * n;
            V *dst = out + (int64_t)c * n;
            V x[7];
            for (int j = 0; j < r; ++j) {
                V v = src[b + j * nb];
                if (j && k) v = cmul(v, __ldg(root + (int64_t)j * k * tws % n));
                x[j] = v;
            }
            V y[7];
            if (r == 2) {
                y[0] = cadd(x[0], x[1]);
                y[1] = csub(x[0], x[1]);
            } else if (r == 4) {
                const V t0 = cadd(x[0], x[2]), t1 = csub(x[0], x[2]), t2 = cadd(x[1], x[3]), t3 = csub(x[1], x[3]);
                y[0] = cadd(t0, t2);
                y[2] = csub(t0, t2);
                y[1] = cadd(t1, crot(t3, s));
                y[3] = csub(t1, crot(t3, s));
            } else if (r == 3) {
                const T h = (T)0.86602540378443864676;  // sqrt(3)/2
                const V t1 = cadd(x[1], x[2]);
                const V t2 = V{x[0].x - (T)0.5 * t1.x, x[0].y - (T)0.5 * t1.y};
                const V t3 = cscale(crot(csub(x[1], x[2]), s), h);
                y[0] = cadd(x[0], t1);
                y[1] = cadd(t2, t3);
                y[2] = csub(t2, t3);
            } else if (r == 1) {
                y[0] = x[0];
            } else {  // 5, 7: direct with the root table, w_r^{jm} = root(j m n / r)
                for (int m = 0; m < r; ++m) {
                    V acc = x[0];
                    for (int j = 1; j < r; ++j) acc = cadd(acc, cmul(x[j], __ldg(root + (int64_t)((j * m) % r) * nb)));
                    y[m] = acc;
                }
            }
            for (int j = 0; j < r; ++j) dst[(b - k) * r + k + j * Ls] = y[j];
        }
    } else {  // any other radix: direct r-point pass, parallel over (butterfly, output)
        for (int idx = threadIdx.x; idx < cnt * n; idx += NT) {
            const int c = idx / n, rem = idx - c * n, b = rem / r, m = rem - b * r, k = b % Ls;
            const V *src = in + (int64_t)c * n;
            V acc = V{0, 0};
            for (int j = 0; j < r; ++j) {
                V v = src[b + j * nb];
                // twiddle w^{j k} times the DFT kernel w_r^{j m}: one root of index (j (k tws + m nb)) mod n
                const int64_t e = ((int64_t)j * ((int64_t)k * tws + (int64_t)m * nb)) % n;
                acc = cadd(acc, cmul(v, __ldg(root + e)));
            }
            out[(int64_t)c * n + (b - k) * r + k + m * Ls] = acc;
        }
    }
}

// full transform: returns the buffer holding the result (a or b)
template <typename T, int NT>
__device__ cv<T> *fft_any(cv<T> *a, cv<T> *b, int n, int cnt, const AnyRadix &pl, int s, const cv<T> *root) {
    int Ls = 1;
    for (int i = 0; i < pl.n; ++i) {
        stockham_pass<T, NT>(a, b, n, cnt, pl.r[i], Ls, s, root);
        __syncthreads();
        Ls *= pl.r[i];
        cv<T> *t = a;
        a = b;
        b = t;
    }
    return a;
}

}  // namespace anyk

template <typename T, int NT>
__global__ void __launch_bounds__(NT) mci_anylen_kernel(const AnyArgs<T> a) {
    using V = cv<T>;
    using namespace anyk;
    extern __shared__ __align__(16) unsigned char smem_raw[];
    const int M = a.M, N = a.N, L = a.L, MN = a.MN, K1 = a.K1, Kmax = a.Kmax;
    const int npair = (M + 1) / 2;
    const int bl = max(npair * N, L);
    V *b0 = reinterpret_cast<V *>(smem_raw);
    V *b1 = b0 + bl;
    V *A = b1 + bl;  // a(k), k = K1 .. K1 + MN - 1
    __shared__ T red[NT / 32];
    __shared__ int escale[8];
    const int tid = threadIdx.x;
    for (int64_t row = blockIdx.x; row < a.rows; row += gridDim.x) {
        const RowAddr &ra = a.ra;
        const int64_t base = (row / (ra.D0 * ra.D1)) * ra.s2 + ((row / ra.D0) % ra.D1) * ra.s1 + (row % ra.D0) * ra.s0;
        // ---- load channel pairs z_c = g_{2c} + i g_{2c+1}, per-channel exact power-of-two scaling
        for (int c = 0; c < npair; ++c) {
            T m0 = 0, m1 = 0;
            for (int n = tid; n < N; n += NT) {
                const T re = __ldg(a.g + base + (int64_t)(2 * c) * ra.cs + (int64_t)n * ra.ss);
                const T im = (2 * c + 1 < M) ? __ldg(a.g + base + (int64_t)(2 * c + 1) * ra.cs + (int64_t)n * ra.ss) : T(0);
                b0[c * N + n] = V{re, im};
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
            const V z = b0[idx];
            b0[idx] = V{ldexp(z.x, -escale[2 * c]), ldexp(z.y, -escale[2 * c + 1])};
        }
        __syncthreads();
        // ---- forward DFTs G_c[q] = sum_n z_c[n] e^{-2 pi i q n / N}
        V *Z = fft_any<T, NT>(b0, b1, N, npair, a.rn, -1, a.twN);
        // ---- per-class solve for every class q: a(j_q + l N), j_q = K1 + ((q - K1) mod N)
        for (int q = tid; q < N; q += NT) {
            const int qm = q == 0 ? 0 : N - q;
            const int jq = K1 + (int)((((int64_t)q - K1) % N + N) % N);
            V v[8];
#pragma unroll
            for (int l = 0; l < 8; ++l) v[l] = V{0, 0};
            for (int m = 0; m < M; ++m) {
                const V zc = Z[(m >> 1) * N + q], zm = cconj(Z[(m >> 1) * N + qm]);
                V gm = (m & 1) ? V{(T)0.5 * (zc.y - zm.y), (T)-0.5 * (zc.x - zm.x)}  // (zc - zm) / (2i)
                               : V{(T)0.5 * (zc.x + zm.x), (T)0.5 * (zc.y + zm.y)};  // (zc + zm) / 2
                gm = V{ldexp(gm.x, escale[m]), ldexp(gm.y, escale[m])};
                const V *qrow = a.Q + ((int64_t)q * M + m) * M;
                for (int l = 0; l < M; ++l) v[l] = cadd(v[l], cmul(gm, __ldg(qrow + l)));
            }
            for (int l = 0; l < M; ++l) A[jq + l * N - K1] = v[l];
        }
        __syncthreads();
        // ---- inverse input: bin i of the length-L transform
        //      real:     sum over k = i (mod L), |k| <= Kmax, of Xf(k) = (a(k) + conj a(-k)) / 2
        //      analytic: Xf(0) at i = 0, 2 Xf(i) for 0 < i <= Kmax
        auto af = [&](int k) { return (k >= K1 && k < K1 + MN) ? A[k - K1] : V{0, 0}; };
        auto xf = [&](int k) {
            const V p = af(k), m = cconj(af(-k));
            return V{(T)0.5 * (p.x + m.x), (T)0.5 * (p.y + m.y)};
        };
        for (int i = tid; i < L; i += NT) {
            V z = V{0, 0};
            if (!a.analytic) {
                if (i <= Kmax) z = xf(i);
                if (i > 0 && L - i <= Kmax) z = cadd(z, xf(i - L));
            } else {
                if (i == 0) z = xf(0);
                else if (i <= Kmax) z = cscale(xf(i), (T)2);
            }
            b0[i] = z;
        }
        __syncthreads();
        V *out = fft_any<T, NT>(b0, b1, L, 1, a.rl, +1, a.twL);
        T *frow = a.f + row * (int64_t)L;
        T *hrow = a.analytic ? a.hf + row * (int64_t)L : nullptr;
        for (int p = tid; p < L; p += NT) {
            const V z = out[p];
            frow[p] = z.x;
            if (hrow) hrow[p] = z.y;
        }
        __syncthreads();
    }
}

size_t anylen_smem_bytes(const Axis1D &ax) {
    const size_t vs = ax.dtype == MCI_F64 ? 16 : 8;
    const int64_t npair = (ax.M + 1) / 2;
    const int64_t bl = std::max<int64_t>(npair * ax.N, ax.L);
    return (size_t)(2 * bl + (int64_t)ax.M * ax.N) * vs;
}

bool anylen_supported(const Axis1D &ax) {
    return ax.M <= 8 && ax.N <= 65536 && ax.L <= (1 << 22) && anylen_smem_bytes(ax) <= 200 * 1024;
}

template <typename T>
static cudaError_t anylen_launch_t(const Axis1D &ax, const RowAddr &ra, int64_t rows, const void *g, void *f, void *hf,
                                   cudaStream_t st) {
    constexpr int NT = 256;
    AnyArgs<T> a;
    a.M = ax.M; a.N = (int)ax.N; a.L = (int)ax.L; a.MN = (int)(ax.M * ax.N);
    a.K1 = (int)ax.K1; a.Kmax = (int)(-ax.K1); a.analytic = ax.analytic;
    a.rn = ax.radN; a.rl = ax.radL;
    a.rows = rows; a.ra = ra;
    a.g = (const T *)g; a.f = (T *)f; a.hf = (T *)hf;
    a.Q = (const cv<T> *)ax.Qt;
    a.twN = (const cv<T> *)ax.twF;
    a.twL = (const cv<T> *)ax.twLhi;
    const size_t smem = anylen_smem_bytes(ax);
    auto kern = mci_anylen_kernel<T, NT>;
    cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    if (e != cudaSuccess) return e;
    int dev = 0, nsm = 148, occ = 1;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, dev);
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, kern, NT, smem);
    int64_t grid = (int64_t)nsm * (occ < 1 ? 1 : occ);
    if (grid > rows) grid = rows;
    kern<<<(unsigned)grid, NT, smem, st>>>(a);
    return cudaGetLastError();
}

cudaError_t launch_anylen(const Axis1D &ax, const RowAddr &ra, int64_t rows, const void *g, void *f, void *hf,
                          cudaStream_t st, int *n_launches) {
    if (rows <= 0) return cudaSuccess;
    if (n_launches) *n_launches += 1;
    return ax.dtype == MCI_F64 ? anylen_launch_t<double>(ax, ra, rows, g, f, hf, st)
                               : anylen_launch_t<float>(ax, ra, rows, g, f, hf, st);
}

}  // namespace mci
