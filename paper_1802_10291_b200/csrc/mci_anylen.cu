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
// FFTs: runtime mixed-radix Stockham passes in shared memory (compile-time radix 4, 2,
// 3, 5 and 7 codelets; the largest prime factor p > 16 by Bluestein's chirp-z transform
// through two power-of-two FFTs of length M >= 2p - 1; other primes as a direct p-point
// pass parallel over its outputs, root index advanced without division), root tables (fp64-rounded) and
// Q~ staged in shared memory.  A warp owns a row (8 rows per CTA, warp-synchronous)
// when its working set is small, else a 256-thread CTA does.
#include <algorithm>
#include <cstdint>
#include <cstdlib>

#include "mci_fft.cuh"
#include "mci_internal.h"

namespace mci {

struct AnyErrSys {
    SysDev s[8];
};

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
    int qsm;           // Q~ copied to shared memory (else read through L1)
    int offgrid;       // evaluate at the points tp[0 .. npts) instead of the L grid (NEXT-3)
    int cplx;          // complex f (NEXT-3 C2C): g, f complex (V), T_N f without real part
    int resid;         // consistency residual per row into f[row] (NEXT-4)
    SysDev sys[8];
    const T *tp;
    int npts;
};

namespace anyk {

// b_m(k) of a built-in system (fp64): 1, (ik)^order, -i sgn k, e^{ik tau} (mci_plan.cpp sys_multiplier)
__device__ __forceinline__ double2 bmul(const SysDev &s, int64_t k) {
    if (s.kind == MCI_SYS_IDENTITY) return make_double2(1.0, 0.0);
    if (s.kind == MCI_SYS_DERIVATIVE) {
        double2 v = make_double2(1.0, 0.0);
        const double kd = (double)k;
        for (int i = 0; i < s.order; ++i) v = make_double2(-v.y * kd, v.x * kd);
        return v;
    }
    if (s.kind == MCI_SYS_HILBERT) return make_double2(0.0, k > 0 ? -1.0 : (k < 0 ? 1.0 : 0.0));
    double sn, cs;  // delay
    sincos(fmod((double)k * s.tau, 6.283185307179586476925286766559), &sn, &cs);
    return make_double2(cs, sn);
}

template <typename V> __device__ __forceinline__ V crot(V a, int s) {  // a * (s i)
    return s > 0 ? V{-a.y, a.x} : V{a.y, -a.x};
}

// x / d and x mod d for 0 <= x < 2^22 without an integer division: float reciprocal, one
// correction step (|x inv - x/d| < 1)
struct FDiv {
    int d;
    float inv;
    __device__ __forceinline__ explicit FDiv(int d_) : d(d_), inv(1.f / (float)d_) {}
    __device__ __forceinline__ int div(int x, int &rem) const {
        int q = (int)((float)x * inv);
        int r = x - q * d;
        if (r < 0) { --q; r += d; }
        else if (r >= d) { ++q; r -= d; }
        rem = r;
        return q;
    }
};

// Row group of G threads: one warp (G = 32, warp-synchronous) or the whole CTA.
template <int G> __device__ __forceinline__ void gsync() {
    if constexpr (G == 32) __syncwarp();
    else __syncthreads();
}

// in-register DFT of compile-time size R in {2, 3, 4, 5, 7}; w_R^m = root[m nb] (root table of the
// transform, e^{s 2 pi i m / n}, nb = n / R) for the 5- and 7-point kernels
template <typename T, int R>
__device__ __forceinline__ void dft_small(cv<T> *x, int s, const cv<T> *root, int nb) {
    using V = cv<T>;
    if constexpr (R == 2) {
        const V t = x[0];
        x[0] = cadd(t, x[1]);
        x[1] = csub(t, x[1]);
    } else if constexpr (R == 4) {
        const V t0 = cadd(x[0], x[2]), t1 = csub(x[0], x[2]), t2 = cadd(x[1], x[3]), t3 = csub(x[1], x[3]);
        x[0] = cadd(t0, t2);
        x[2] = csub(t0, t2);
        x[1] = cadd(t1, crot(t3, s));
        x[3] = csub(t1, crot(t3, s));
    } else if constexpr (R == 3) {
        const T h = (T)0.86602540378443864676;  // sqrt(3)/2
        const V t1 = cadd(x[1], x[2]);
        const V t2 = V{x[0].x - (T)0.5 * t1.x, x[0].y - (T)0.5 * t1.y};
        const V t3 = cscale(crot(csub(x[1], x[2]), s), h);
        x[0] = cadd(x[0], t1);
        x[1] = cadd(t2, t3);
        x[2] = csub(t2, t3);
    } else {
        V w[R];
#pragma unroll
        for (int m = 0; m < R; ++m) w[m] = root[m * nb];
        V y[R];
#pragma unroll
        for (int m = 0; m < R; ++m) {
            V acc = x[0];
#pragma unroll
            for (int j = 1; j < R; ++j) acc = cadd(acc, cmul(x[j], w[(j * m) % R]));
            y[m] = acc;
        }
#pragma unroll
        for (int m = 0; m < R; ++m) x[m] = y[m];
    }
}

// one Stockham pass of radix R over `cnt` transforms of length n stored with stride n:
// butterfly b in [0, n/R), k = b mod Ls: x_j = in[b + j n/R] w^{j k}, w = root^(n/(Ls R)),
// out[(b - k) R + k + j Ls] = DFT_R(x)_j.  root(m) = e^{s 2 pi i m / n} (shared memory).
// PAD: the root table is stored padded (entry e at e + e / 16), which spreads the strided
// twiddle reads k * tws of a warp over the banks (the Bluestein power-of-two transforms)
template <typename T, int R, int G, bool PAD = false>
__device__ __forceinline__ void pass_r(const cv<T> *in, cv<T> *out, int n, int cnt, int Ls, int s, const cv<T> *root,
                                       int lane) {
    using V = cv<T>;
    const int nb = n / R, tws = n / (Ls * R);
    const FDiv fl(Ls);
    for (int c = 0; c < cnt; ++c)
    for (int b = lane; b < nb; b += G) {
        int k;
        fl.div(b, k);  // k = b mod Ls
        const V *src = in + c * n;
        V x[R];
        const int d = k * tws;  // < n
        int e = 0;
#pragma unroll
        for (int j = 0; j < R; ++j) {
            x[j] = src[b + j * nb];
            if (j) {
                e += d;
                if (e >= n) e -= n;
                if (k) x[j] = cmul(x[j], root[PAD ? e + (e >> 4) : e]);
            }
        }
        dft_small<T, R>(x, s, root, nb);
        V *dst = out + c * n + (b - k) * R + k;
#pragma unroll
        for (int j = 0; j < R; ++j) dst[j * Ls] = x[j];
    }
}

// any other (prime) radix r: direct r-point pass.  A thread computes U consecutive outputs
// m0 .. m0+U-1 of one butterfly, so each input is loaded once for U outputs: the kernel
// root of output m0 + t is W^{j d} (W^{j nb})^t with d = k tws + m0 nb (the twiddle w^{jk}
// and the DFT kernel w_r^{j m} combined, index advanced without division), i.e. one table
// load and U - 1 multiplications per input instead of U loads (the pass is bound by
// shared-memory bandwidth).
template <typename T, int G>
__device__ void pass_direct(const cv<T> *in, cv<T> *out, int n, int cnt, int r, int Ls, const cv<T> *root, int lane) {
    using V = cv<T>;
    constexpr int U = 4;
    const int nb = n / r, tws = n / (Ls * r), mbk = (r + U - 1) / U;
    const FDiv fm(mbk), fl(Ls);
    for (int c = 0; c < cnt; ++c)
    for (int rem = lane; rem < nb * mbk; rem += G) {
        int mb, k;
        const int b = fm.div(rem, mb);
        const int m0 = mb * U;
        fl.div(b, k);
        const V *src = in + c * n + b;
        int d = k * tws + m0 * nb;  // < 2 n
        if (d >= n) d -= n;
        V acc[U];
#pragma unroll
        for (int t = 0; t < U; ++t) acc[t] = src[0];
        int e = 0, f = 0;  // e = j d mod n, f = j nb mod n
        for (int j = 1; j < r; ++j) {
            e += d;
            if (e >= n) e -= n;
            f += nb;
            if (f >= n) f -= n;
            const V x = src[j * nb], st = root[f];
            V w = root[e];
#pragma unroll
            for (int t = 0; t < U; ++t) {
                acc[t] = cadd(acc[t], cmul(x, w));
                if (t + 1 < U) w = cmul(w, st);
            }
        }
        V *dst = out + c * n + (b - k) * r + k;
#pragma unroll
        for (int t = 0; t < U; ++t)
            if (m0 + t < r) dst[(m0 + t) * Ls] = acc[t];
    }
}

// Bluestein (chirp-z) state of one transform: tables and the group's two M-point buffers
template <typename T> struct Blue {
    int p = 0, M = 0;
    const cv<T> *c, *H, *wm, *wp;  // chirp [p], H^ [M] (1/M folded in), e^{-2 pi i m/M}, e^{+2 pi i m/M}
    cv<T> *t0, *t1;
};

template <typename T, int G>
__device__ cv<T> *fft_pow2(cv<T> *a, cv<T> *b, int n, int s, const cv<T> *root, int lane) {
    int Ls = 1;
    while (Ls < n) {
        if (n / Ls >= 4) {
            pass_r<T, 4, G, true>(a, b, n, 1, Ls, s, root, lane);
            Ls *= 4;
        } else {
            pass_r<T, 2, G, true>(a, b, n, 1, Ls, s, root, lane);
            Ls *= 2;
        }
        gsync<G>();
        cv<T> *t = a;
        a = b;
        b = t;
    }
    return a;
}

// radix-p pass by Bluestein: X_m = c_m (a (*) h)_m, a_j = x_j c_j (x twiddled), h = conj c,
// as two M-point FFTs and a pointwise product with H^ = FFT(h)/M; butterflies one at a time
template <typename T, int G>
__device__ void pass_bluestein(const cv<T> *in, cv<T> *out, int n, int cnt, int Ls, const cv<T> *root, const Blue<T> &bl,
                               int lane) {
    using V = cv<T>;
    const int p = bl.p, M = bl.M, nb = n / p, tws = n / (Ls * p);
    for (int c = 0; c < cnt; ++c)
    for (int b = 0; b < nb; ++b) {
        const int k = b % Ls;
        const V *src = in + c * n;
        const int d = k * tws;                         // twiddle index step (< n)
        int e = (int)(((int64_t)lane * d) % n);        // index of element i = lane
        const int dG = (int)(((int64_t)G * d) % n);    // advance per G elements
        for (int i = lane; i < M; i += G) {
            V v = V{0, 0};
            if (i < p) {
                v = src[b + i * nb];
                if (e) v = cmul(v, root[e]);
                v = cmul(v, bl.c[i]);
            }
            bl.t0[i] = v;
            e += dG;
            if (e >= n) e -= n;
        }
        gsync<G>();
        V *R = fft_pow2<T, G>(bl.t0, bl.t1, M, -1, bl.wm, lane);
        for (int i = lane; i < M; i += G) R[i] = cmul(R[i], bl.H[i]);
        gsync<G>();
        V *R2 = fft_pow2<T, G>(R, R == bl.t0 ? bl.t1 : bl.t0, M, +1, bl.wp, lane);
        V *dst = out + c * n + (b - k) * p + k;
        for (int m = lane; m < p; m += G) dst[m * Ls] = cmul(R2[m], bl.c[m]);
        gsync<G>();
    }
}

// full transform; returns the buffer holding the result (a or b)
template <typename T, int G>
__device__ cv<T> *fft_any(cv<T> *a, cv<T> *b, int n, int cnt, const AnyRadix &pl, int s, const cv<T> *root,
                          const Blue<T> &bl, int lane) {
    int Ls = 1;
    for (int i = 0; i < pl.n; ++i) {
        const int r = pl.r[i];
        if (r == bl.p) {
            pass_bluestein<T, G>(a, b, n, cnt, Ls, root, bl, lane);
            gsync<G>();
            Ls *= r;
            cv<T> *t = a;
            a = b;
            b = t;
            continue;
        }
        switch (r) {
        case 2: pass_r<T, 2, G>(a, b, n, cnt, Ls, s, root, lane); break;
        case 3: pass_r<T, 3, G>(a, b, n, cnt, Ls, s, root, lane); break;
        case 4: pass_r<T, 4, G>(a, b, n, cnt, Ls, s, root, lane); break;
        case 5: pass_r<T, 5, G>(a, b, n, cnt, Ls, s, root, lane); break;
        case 7: pass_r<T, 7, G>(a, b, n, cnt, Ls, s, root, lane); break;
        default: pass_direct<T, G>(a, b, n, cnt, r, Ls, root, lane); break;
        }
        gsync<G>();
        Ls *= r;
        cv<T> *t = a;
        a = b;
        b = t;
    }
    return a;
}

template <typename T, int G> __device__ __forceinline__ T group_max(T v, T *red) {
    if constexpr (G == 32) {
#pragma unroll
        for (int o = 16; o; o >>= 1) v = fmax(v, __shfl_xor_sync(0xffffffffu, v, o));
        return v;
    } else {
        return block_max<G>(v, red);
    }
}

}  // namespace anyk

// smem layout: [twN: N][twL: L][Q~: N M M if qsm][Bluestein tables N, L] then per group
// [b0: bl][b1: bl][A: RP MN | t0: bM, t1: bM].
// Real output: a group takes RP = 2 rows at a time -- their 2M real channels share M complex
// forward FFTs and one inverse FFT gives f(row 0) + i f(row 1) (both spectra are Hermitian).
// Analytic output (z = f + i Hf is complex): one row at a time.
template <typename T, int G, int GPB>
__global__ void __launch_bounds__(G * GPB) mci_anylen_kernel(const AnyArgs<T> a) {
    using V = cv<T>;
    using namespace anyk;
    extern __shared__ __align__(16) unsigned char smem_raw[];
    const int M = a.M, N = a.N, L = a.L, MN = a.MN, K1 = a.K1, Kmax = a.Kmax;
    const int RP = (a.analytic || a.offgrid || a.cplx || a.resid) ? 1 : 2;
    const int bl = max((a.cplx ? M : (RP * M + 1) / 2) * N, L);
    V *twN = reinterpret_cast<V *>(smem_raw);
    V *twL = twN + N;
    V *Qs = twL + L;
    const int qn = a.qsm ? N * M * M : 0;
    V *btab = Qs + qn;
    Blue<T> blN, blL;
    const AnyRadix *rr[2] = {&a.rn, &a.rl};
    Blue<T> *bb[2] = {&blN, &blL};
    for (int t = 0; t < 2; ++t) {  // stage the Bluestein tables in shared memory
        Blue<T> &q = *bb[t];
        q.p = rr[t]->bp;
        q.M = rr[t]->bM;
        if (!q.p) continue;
        const int Mp = q.M + q.M / 16 + 1;  // padded root tables (see pass_r)
        V *c = btab, *H = c + q.p, *wm = H + q.M, *wp = wm + Mp;
        for (int i = threadIdx.x; i < q.p; i += G * GPB) c[i] = ((const V *)rr[t]->bc)[i];
        for (int i = threadIdx.x; i < q.M; i += G * GPB) {
            H[i] = ((const V *)rr[t]->bH)[i];
            wm[i + (i >> 4)] = ((const V *)rr[t]->bwm)[i];
            wp[i + (i >> 4)] = ((const V *)rr[t]->bwp)[i];
        }
        q.c = c; q.H = H; q.wm = wm; q.wp = wp;
        btab = wp + Mp;
    }
    const int bmx = max(blN.M, blL.M);
    const int grp = threadIdx.x / G, lane = threadIdx.x % G;
    V *b0 = btab + (size_t)grp * (2 * bl + max(RP * MN, 2 * bmx));
    V *b1 = b0 + bl;
    V *A = b1 + bl;  // a(k) of row rl at A[rl MN + k - K1], k = K1 .. K1 + MN - 1
    // Bluestein buffers alias A: A is written after the forward FFT and dead before the inverse
    blN.t0 = blL.t0 = A;
    blN.t1 = blL.t1 = A + bmx;
    for (int i = threadIdx.x; i < N; i += G * GPB) twN[i] = a.twN[i];
    for (int i = threadIdx.x; i < L; i += G * GPB) twL[i] = a.twL[i];
    for (int i = threadIdx.x; i < qn; i += G * GPB) Qs[i] = a.Q[i];
    const V *Qt = a.qsm ? Qs : a.Q;
    __shared__ T red[(G > 32 ? G : 32) / 32];
    __shared__ int escale_s[GPB][16];
    int *escale = escale_s[grp];
    __syncthreads();
    const int64_t nunits = (a.rows + RP - 1) / RP;
    for (int64_t u = (int64_t)blockIdx.x * GPB + grp; u < nunits; u += (int64_t)gridDim.x * GPB) {
        const RowAddr &ra = a.ra;
        const int64_t row0 = u * RP;
        const int nr = (int)min((int64_t)RP, a.rows - row0);  // rows in this unit
        const int nvc = nr * M, npv = a.cplx ? M : (nvc + 1) / 2;  // real channels, complex FFTs
        auto chan = [&](int vc) {  // address of virtual channel vc = rl M + m
            const int64_t row = row0 + vc / M;
            return a.g + (row / (ra.D0 * ra.D1)) * ra.s2 + ((row / ra.D0) % ra.D1) * ra.s1 + (row % ra.D0) * ra.s0 +
                   (int64_t)(vc % M) * ra.cs;
        };
        // ---- load channel pairs z_c = g_{2c} + i g_{2c+1} (complex mode: z_m = g_m), per-channel
        //      exact power-of-two scaling
        if (a.cplx) {
            const V *gc = reinterpret_cast<const V *>(a.g);
            const int64_t rb = (row0 / (ra.D0 * ra.D1)) * ra.s2 + ((row0 / ra.D0) % ra.D1) * ra.s1 + (row0 % ra.D0) * ra.s0;
            for (int c = 0; c < M; ++c) {
                T mx = 0;
                for (int n = lane; n < N; n += G) {
                    const V v = gc[rb + (int64_t)c * ra.cs + (int64_t)n * ra.ss];
                    b0[c * N + n] = v;
                    mx = fmax(mx, fmax(fabs(v.x), fabs(v.y)));
                }
                mx = group_max<T, G>(mx, red);
                if (lane == 0) {
                    int e0 = 0;
                    if (mx > 0) frexp(mx, &e0);
                    escale[2 * c] = escale[2 * c + 1] = e0;
                }
            }
        }
        for (int c = 0; c < (a.cplx ? 0 : npv); ++c) {
            T m0 = 0, m1 = 0;
            const T *p0 = chan(2 * c), *p1 = (2 * c + 1 < nvc) ? chan(2 * c + 1) : nullptr;
            for (int n = lane; n < N; n += G) {
                const T re = __ldg(p0 + (int64_t)n * ra.ss);
                const T im = p1 ? __ldg(p1 + (int64_t)n * ra.ss) : T(0);
                b0[c * N + n] = V{re, im};
                m0 = fmax(m0, fabs(re));
                m1 = fmax(m1, fabs(im));
            }
            m0 = group_max<T, G>(m0, red);
            m1 = group_max<T, G>(m1, red);
            if (lane == 0) {
                int e0 = 0, e1 = 0;
                if (m0 > 0) frexp(m0, &e0);
                if (m1 > 0) frexp(m1, &e1);
                escale[2 * c] = e0;
                escale[2 * c + 1] = e1;
            }
        }
        gsync<G>();
        for (int c = 0; c < npv; ++c) {
            const int s0 = -escale[2 * c], s1 = -escale[2 * c + 1];
            for (int n = lane; n < N; n += G) {
                const V z = b0[c * N + n];
                b0[c * N + n] = V{ldexp(z.x, s0), ldexp(z.y, s1)};
            }
        }
        gsync<G>();
        // ---- forward DFTs G_c[q] = sum_n z_c[n] e^{-2 pi i q n / N}
        V *Z = fft_any<T, G>(b0, b1, N, npv, a.rn, -1, twN, blN, lane);
        // ---- per-class solve for every class q: a(j_q + l N), j_q = K1 + ((q - K1) mod N)
        const int q0 = (int)((((int64_t)-K1) % N + N) % N);  // (q - K1) mod N = (q + q0) mod N
        for (int rl = 0; rl < nr; ++rl)
        for (int q = lane; q < N; q += G) {
            const int qm = q == 0 ? 0 : N - q;
            int t = q + q0;
            if (t >= N) t -= N;
            const int jq = K1 + t;
            V v[8];
#pragma unroll
            for (int l = 0; l < 8; ++l) v[l] = V{0, 0};
            for (int m = 0; m < M; ++m) {
                const int vc = rl * M + m;
                V gm;
                if (a.cplx) {  // own FFT per channel: G_m = Z_m
                    const V zc = Z[m * N + q];
                    gm = V{ldexp(zc.x, escale[2 * m]), ldexp(zc.y, escale[2 * m])};
                } else {
                    const V zc = Z[(vc >> 1) * N + q], zm = cconj(Z[(vc >> 1) * N + qm]);
                    gm = (vc & 1) ? V{(T)0.5 * (zc.y - zm.y), (T)-0.5 * (zc.x - zm.x)}  // (zc - zm) / (2i)
                                  : V{(T)0.5 * (zc.x + zm.x), (T)0.5 * (zc.y + zm.y)};  // (zc + zm) / 2
                    gm = V{ldexp(gm.x, escale[vc]), ldexp(gm.y, escale[vc])};
                }
                const V *qrow = Qt + ((int64_t)q * M + m) * M;
#pragma unroll
                for (int l = 0; l < 8; ++l)
                    if (l < M) v[l] = cadd(v[l], cmul(gm, qrow[l]));
            }
#pragma unroll
            for (int l = 0; l < 8; ++l)
                if (l < M) A[rl * MN + jq + l * N - K1] = v[l];
        }
        gsync<G>();
        // ---- inverse input: bin i of the length-L transform
        //      real:     sum over k = i (mod L), |k| <= Kmax, of Xf(k) = (a(k) + conj a(-k)) / 2
        //      analytic: Xf(0) at i = 0, 2 Xf(i) for 0 < i <= Kmax
        auto af = [&](int rl, int k) { return (k >= K1 && k < K1 + MN) ? A[rl * MN + k - K1] : V{0, 0}; };
        auto xf = [&](int rl, int k) {
            const V p = af(rl, k), m = cconj(af(rl, -k));
            return V{(T)0.5 * (p.x + m.x), (T)0.5 * (p.y + m.y)};
        };
        if (a.resid) {
            // ---- consistency residual (Theorem consistency): for every channel m,
            //      F_m(q) = sum_l a(j_q + lN) b_m(j_q + lN) (a^ b_m folded mod N); the inverse DFT
            //      y_m(n) = sum_q F_m(q) e^{2 pi i q n / N} (conj trick through the forward plan) is
            //      (T_N f * h_m)(t_n); out[row] = max_{m,n} |y_m(n) - g_m[n]|.  All M channels are
            //      folded first (A is overwritten by the transform's Bluestein buffers).
            const int q0r = (int)((((int64_t)-K1) % N + N) % N);
            for (int m = 0; m < M; ++m)
                for (int q = lane; q < N; q += G) {
                    int t = q + q0r;
                    if (t >= N) t -= N;
                    const int jq = K1 + t;
                    double fr = 0.0, fi = 0.0;
                    for (int l = 0; l < M; ++l) {
                        const V x = A[jq + l * N - K1];
                        const double2 b = bmul(a.sys[m], (int64_t)jq + (int64_t)l * N);
                        fr += (double)x.x * b.x - (double)x.y * b.y;
                        fi += (double)x.x * b.y + (double)x.y * b.x;
                    }
                    b0[m * N + q] = V{(T)fr, (T)-fi};  // conj
                }
            gsync<G>();
            V *Y = fft_any<T, G>(b0, b1, N, M, a.rn, -1, twN, blN, lane);
            T best = 0;
            for (int m = 0; m < M; ++m) {
                const T *gm = chan(m);
                for (int n = lane; n < N; n += G) {
                    const V y = Y[m * N + n];
                    const T gv = gm[(int64_t)n * ra.ss];
                    best = fmax(best, sqrt((y.x - gv) * (y.x - gv) + y.y * y.y));  // y = conj(Y)
                }
            }
            best = group_max<T, G>(best, red);
            if (lane == 0) a.f[row0] = best;
            gsync<G>();
            continue;
        }
        if (a.offgrid) {
            // ---- off-grid evaluation (Eq. drictexpression / Lemma 2):
            //      f(t) = Xf(0) + 2 sum_{k=1}^{Kmax} Re(Xf(k) e^{ikt}),  Hf(t) = 2 sum_k Im(Xf(k) e^{ikt});
            //      Horner's scheme in fp64 on z = e^{it}: p = sum_{k>=1} Xf(k) z^k (4 DFMA per term,
            //      error ~ 2 Kmax eps), then f = Xf(0) + 2 Re p, Hf = 2 Im p
            for (int k = lane; k <= Kmax; k += G) b0[k] = xf(0, k);
            gsync<G>();
            T *frow = a.f + row0 * (int64_t)a.npts;
            T *hrow = a.analytic ? a.hf + row0 * (int64_t)a.npts : nullptr;
            constexpr int PP = 4;  // points per thread: independent Horner chains (ILP)
            for (int j0 = lane; j0 < a.npts; j0 += G * PP) {
                double zr[PP], zi[PP], qr[PP], qi[PP];
#pragma unroll
                for (int u = 0; u < PP; ++u) {
                    const int j = j0 + u * G;
                    sincos(j < a.npts ? (double)a.tp[j] : 0.0, &zi[u], &zr[u]);
                    qr[u] = qi[u] = 0.0;
                }
                for (int k = Kmax; k >= 1; --k) {  // q <- (q + X_k) z
                    const V x = b0[k];
#pragma unroll
                    for (int u = 0; u < PP; ++u) {
                        const double ar = qr[u] + (double)x.x, ai = qi[u] + (double)x.y;
                        qr[u] = fma(ar, zr[u], -ai * zi[u]);
                        qi[u] = fma(ar, zi[u], ai * zr[u]);
                    }
                }
#pragma unroll
                for (int u = 0; u < PP; ++u) {
                    const int j = j0 + u * G;
                    if (j < a.npts) {
                        frow[j] = (T)((double)b0[0].x + 2.0 * qr[u]);
                        if (hrow) hrow[j] = (T)(2.0 * qi[u]);
                    }
                }
            }
            gsync<G>();
            continue;
        }
        for (int i = lane; i < L; i += G) {
            V z = V{0, 0};
            if (a.cplx) {  // T_N f: a(k) at bin k mod L (M N <= L: at most one k per bin)
                if (i >= K1 && i < K1 + MN) z = A[i - K1];
                else if (i - L >= K1 && i - L < K1 + MN) z = A[i - L - K1];
            } else if (!a.analytic) {  // Z0(i) + i Z1(i), Zr = row r's folded Hermitian spectrum
                for (int rl = 0; rl < nr; ++rl) {
                    V zr = V{0, 0};
                    if (i <= Kmax) zr = xf(rl, i);
                    if (i > 0 && L - i <= Kmax) zr = cadd(zr, xf(rl, i - L));
                    z = rl ? cadd(z, crot(zr, 1)) : zr;
                }
            } else {
                if (i == 0) z = xf(0, 0);
                else if (i <= Kmax) z = cscale(xf(0, i), (T)2);
            }
            b0[i] = z;
        }
        gsync<G>();
        V *out = fft_any<T, G>(b0, b1, L, 1, a.rl, +1, twL, blL, lane);
        if (a.cplx) {
            V *fo = reinterpret_cast<V *>(a.f) + row0 * (int64_t)L;
            for (int p = lane; p < L; p += G) fo[p] = out[p];
            gsync<G>();
            continue;
        }
        T *frow = a.f + row0 * (int64_t)L;
        T *hrow = a.analytic ? a.hf + row0 * (int64_t)L : (nr > 1 ? frow + L : nullptr);  // Hf, or row 1's f
        for (int p = lane; p < L; p += G) {
            const V z = out[p];
            frow[p] = z.x;
            if (hrow) hrow[p] = z.y;
        }
        gsync<G>();
    }
}

// shared memory: root tables + Q~ (if small) + per row group [2 bl + MN] complex values
static size_t group_elems(const Axis1D &ax) {
    const int64_t rp = (ax.analytic || ax.cplx) ? 1 : 2;  // rows per unit (real output pairs rows)
    const int64_t nfft = ax.cplx ? ax.M : (rp * ax.M + 1) / 2;
    return (size_t)(2 * std::max<int64_t>(nfft * ax.N, ax.L) +
                    std::max<int64_t>(rp * ax.M * ax.N, 2 * std::max(ax.radN.bM, ax.radL.bM)));
}
static size_t blue_elems(const AnyRadix &r) { return r.bp ? (size_t)(r.bp + 3 * r.bM + 2 * (r.bM / 16 + 1)) : 0; }
static bool q_in_smem(const Axis1D &ax) { return ax.N * ax.M * ax.M <= 4096; }
static size_t smem_for(const Axis1D &ax, int groups) {
    const size_t vs = ax.dtype == MCI_F64 ? 16 : 8;
    return (size_t)(ax.N + ax.L + (q_in_smem(ax) ? ax.N * ax.M * ax.M : 0) + blue_elems(ax.radN) + blue_elems(ax.radL) +
                    groups * group_elems(ax)) * vs;
}
// warp per row when a row's working set is small: the most rows per CTA (8, 4 or 2) that still
// lets two CTAs share an SM; else one 256-thread CTA per row
static int warp_groups(const Axis1D &ax) {
    for (int gp : {8, 4, 2})
        if (smem_for(ax, gp) <= 110 * 1024) return gp;
    return smem_for(ax, 8) <= 200 * 1024 ? 8 : 0;
}

size_t anylen_smem_bytes(const Axis1D &ax) {
    const int gp = warp_groups(ax);
    return gp ? smem_for(ax, gp) : smem_for(ax, 1);
}

bool anylen_supported(const Axis1D &ax) {
    return ax.M <= 8 && ax.N <= 65536 && ax.L <= (1 << 22) && anylen_smem_bytes(ax) <= 200 * 1024;
}

template <typename T, int G, int GPB>
static cudaError_t anylen_launch_t(const Axis1D &ax, const RowAddr &ra, int64_t rows, const void *g, void *f, void *hf,
                                   cudaStream_t st, const void *tp = nullptr, int64_t npts = 0) {
    AnyArgs<T> a;
    a.offgrid = tp != nullptr && npts > 0;
    a.resid = tp != nullptr && npts < 0;
    a.cplx = ax.cplx;
    for (int m = 0; m < 8; ++m) a.sys[m] = ax.sys[m];
    a.tp = (const T *)tp;
    a.npts = (int)npts;
    a.M = ax.M; a.N = (int)ax.N; a.L = (int)ax.L; a.MN = (int)(ax.M * ax.N);
    a.K1 = (int)ax.K1; a.Kmax = (int)(-ax.K1); a.analytic = ax.analytic;
    a.rn = ax.radN; a.rl = ax.radL;
    a.rows = rows; a.ra = ra;
    a.g = (const T *)g; a.f = (T *)f; a.hf = (T *)hf;
    a.Q = (const cv<T> *)ax.Qt;
    a.twN = (const cv<T> *)ax.twF;
    a.twL = (const cv<T> *)ax.twLhi;
    a.qsm = q_in_smem(ax) ? 1 : 0;
    const size_t smem = smem_for(ax, GPB);
    auto kern = mci_anylen_kernel<T, G, GPB>;
    cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    if (e != cudaSuccess) return e;
    int dev = 0, nsm = 148, occ = 1;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, dev);
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, kern, G * GPB, smem);
    int64_t grid = (int64_t)nsm * (occ < 1 ? 1 : occ);
    const int64_t need = (rows + GPB - 1) / GPB;
    if (grid > need) grid = need;
    kern<<<(unsigned)grid, G * GPB, smem, st>>>(a);
    return cudaGetLastError();
}

static cudaError_t anylen_dispatch(const Axis1D &ax, const RowAddr &ra, int64_t rows, const void *g, void *f, void *hf,
                                   cudaStream_t st, const void *tp, int64_t npts) {
    const bool d = ax.dtype == MCI_F64;
    switch (warp_groups(ax)) {
    case 8: return d ? anylen_launch_t<double, 32, 8>(ax, ra, rows, g, f, hf, st, tp, npts)
                     : anylen_launch_t<float, 32, 8>(ax, ra, rows, g, f, hf, st, tp, npts);
    case 4: return d ? anylen_launch_t<double, 32, 4>(ax, ra, rows, g, f, hf, st, tp, npts)
                     : anylen_launch_t<float, 32, 4>(ax, ra, rows, g, f, hf, st, tp, npts);
    case 2: return d ? anylen_launch_t<double, 32, 2>(ax, ra, rows, g, f, hf, st, tp, npts)
                     : anylen_launch_t<float, 32, 2>(ax, ra, rows, g, f, hf, st, tp, npts);
    default: return d ? anylen_launch_t<double, 256, 1>(ax, ra, rows, g, f, hf, st, tp, npts)
                      : anylen_launch_t<float, 256, 1>(ax, ra, rows, g, f, hf, st, tp, npts);
    }
}

cudaError_t launch_anylen(const Axis1D &ax, const RowAddr &ra, int64_t rows, const void *g, void *f, void *hf,
                          cudaStream_t st, int *n_launches) {
    if (rows <= 0) return cudaSuccess;
    if (n_launches) *n_launches += 1;
    return anylen_dispatch(ax, ra, rows, g, f, hf, st, nullptr, 0);
}

cudaError_t launch_anylen_residual(const Axis1D &ax, const RowAddr &ra, int64_t rows, const void *g, void *out,
                                   cudaStream_t st) {
    if (rows <= 0) return cudaSuccess;
    static const int marker = 0;  // residual mode: tp set, npts < 0
    return anylen_dispatch(ax, ra, rows, g, out, nullptr, st, &marker, -1);
}

// eps(f, N) of a batch of spectra (Theorem error, Eq. averageerror / errorestimate).
// The weight of a band-external coefficient n,
// Averaged error eps(f, N) (Eq. averageerror) with its bound (Eq.
// errorestimate, reading R12) and the out-of-band energy, per spectrum a(k_lo .. k_lo + nf - 1).
// The weight of an out-of-band coefficient, 1 + sum_l |sum_m r_m(n + (l-k)N) b_m(n)|^2, and
// sum_m |b_m(n)|^2 depend on n only.  Execute never allocates (include/mci.h), so the weights
// live in shared memory: persistent CTAs (one per SM) compute the table for the whole
// frequency range once (weights in the plan's precision: 8 B per frequency in fp32, 16 B in
// fp64; up to AE_CAP frequencies), then stream their spectra through it, one warp per spectrum,
// the in-band run [K1, K1 + MN) skipped whole (those coefficients carry no error).  Longer
// frequency ranges are walked in chunks of AE_CAP, the chunk's weights recomputed per group of
// a CTA's spectra (partial sums in shared memory).  Sums are fp64 in a fixed order:
// deterministic.  The spectra stream from HBM exactly once.
constexpr int AE_THREADS = 1024;
constexpr int AE_SMEM = 200 * 1024;           // weight table bytes per CTA
constexpr int AE_GROUP = 256;                 // spectra per partial-sum group (chunked mode)

__device__ __forceinline__ double2 avg_error_weight(int64_t n, int M, int N, int64_t K1, const void *Qv, bool q64,
                                                    const AnyErrSys &sy) {
    using namespace anyk;
    const int64_t d = n - K1;
    const int64_t kb = (d >= 0 ? d / N : -((-d + N - 1) / N)) + 1;  // block index of n
    if (kb >= 1 && kb <= M) return make_double2(-1.0, 0.0);
    const int64_t j = n - (kb - 1) * N;  // the class element of I_1
    const int q = (int)(((j % N) + N) % N);
    double2 b[8];
    double bsum = 0;
    for (int m = 0; m < M; ++m) {
        b[m] = bmul(sy.s[m], n);
        bsum += b[m].x * b[m].x + b[m].y * b[m].y;
    }
    double w = 0;
    for (int l = 0; l < M; ++l) {  // S_l = sum_m r_m(j + lN) b_m(n), r_m(j + lN) = N Q~_q[m][l]
        double sr = 0, si = 0;
        for (int m = 0; m < M; ++m) {
            const int64_t e = ((int64_t)q * M + m) * M + l;
            double rr, ri;
            if (q64) {
                const double2 r = static_cast<const double2 *>(Qv)[e];
                rr = r.x * N, ri = r.y * N;
            } else {
                const float2 r = static_cast<const float2 *>(Qv)[e];
                rr = (double)r.x * N, ri = (double)r.y * N;
            }
            sr += rr * b[m].x - ri * b[m].y;
            si += rr * b[m].y + ri * b[m].x;
        }
        w += sr * sr + si * si;
    }
    return make_double2(1.0 + w, bsum);
}

// weight entry in the table's precision
template <typename T> struct AEW { using type = float2; };
template <> struct AEW<double> { using type = double2; };

template <typename T>
__global__ void __launch_bounds__(AE_THREADS, 1) mci_avg_error_kernel(const cv<T> *__restrict__ spec, int nf,
                                                                       int64_t batch, int64_t k_lo, int M, int N,
                                                                       int64_t K1, const void *Qv, bool q64,
                                                                       AnyErrSys sy, double omega_sum,
                                                                       T *__restrict__ out) {
    using W = typename AEW<T>::type;
    constexpr int CAP = AE_SMEM / sizeof(W);
    extern __shared__ __align__(16) unsigned char ae_smem[];
    W *wt = reinterpret_cast<W *>(ae_smem);
    __shared__ double acc[AE_GROUP][3];  // chunked mode: (e2, oob, cs) per spectrum of the group
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    constexpr int NW = AE_THREADS / 32;
    const int64_t MN = (int64_t)M * N;
    const bool one = nf <= CAP;  // whole range resident: weights once, then stream
    // spectra of this CTA: s = blockIdx.x + i gridDim.x; groups of AE_GROUP in chunked mode
    const int64_t mine = batch > blockIdx.x ? (batch - 1 - blockIdx.x) / gridDim.x + 1 : 0;
    const int64_t gsz = one ? mine : AE_GROUP;
    for (int64_t g0 = 0; g0 < mine; g0 += gsz) {
        const int64_t ng = mine - g0 < gsz ? mine - g0 : gsz;
        if (!one) {
            __syncthreads();  // previous group's sums written out
            for (int i = threadIdx.x; i < AE_GROUP * 3; i += AE_THREADS) (&acc[0][0])[i] = 0.0;
        }
        for (int c0 = 0; c0 < nf; c0 += CAP) {
            const int nc = min(CAP, nf - c0);
            if (!one || g0 == 0) {
                __syncthreads();  // previous chunk's weights consumed
                for (int i = threadIdx.x; i < nc; i += AE_THREADS) {
                    const double2 w = avg_error_weight(k_lo + c0 + i, M, N, K1, Qv, q64, sy);
                    wt[i] = W{(decltype(W::x))w.x, (decltype(W::x))w.y};
                }
                __syncthreads();
            }
            // in-band run of this chunk, [ib0, ib1) (chunk-relative), skipped whole
            const int64_t lo = K1 - (k_lo + c0), hi = lo + MN;
            auto clampc = [&](int64_t x) { return (int)(x < 0 ? 0 : x > nc ? nc : x); };
            const int ib0 = clampc(lo), ib1 = clampc(hi);
            for (int64_t si = warp; si < ng; si += NW) {  // one warp per spectrum
                const int64_t sp = blockIdx.x + (g0 + si) * gridDim.x;
                const cv<T> *a = spec + sp * (int64_t)nf + c0;
                double e2 = 0, oob = 0, cs = 0;
                auto run = [&](int b0, int b1) {
                    int i = b0 + lane;
                    for (; i + 96 < b1; i += 128) {  // four independent loads in flight per lane
                        cv<T> av[4];
#pragma unroll
                        for (int u = 0; u < 4; ++u) av[u] = a[i + 32 * u];
#pragma unroll
                        for (int u = 0; u < 4; ++u) {
                            const W w = wt[i + 32 * u];
                            const double a2 = (double)av[u].x * av[u].x + (double)av[u].y * av[u].y;
                            e2 += a2 * (double)w.x;
                            oob += a2;
                            cs += a2 * (double)w.y;
                        }
                    }
                    for (; i < b1; i += 32) {
                        const cv<T> an = a[i];
                        const W w = wt[i];
                        const double a2 = (double)an.x * an.x + (double)an.y * an.y;
                        e2 += a2 * (double)w.x;
                        oob += a2;
                        cs += a2 * (double)w.y;
                    }
                };
                run(0, ib0);
                run(ib1, nc);
#pragma unroll
                for (int o = 16; o; o >>= 1) {
                    e2 += __shfl_xor_sync(0xffffffffu, e2, o);
                    oob += __shfl_xor_sync(0xffffffffu, oob, o);
                    cs += __shfl_xor_sync(0xffffffffu, cs, o);
                }
                if (one) {
                    if (lane == 0) {
                        T *o = out + sp * 3;
                        o[0] = (T)sqrt(e2);
                        o[1] = (T)sqrt(oob + M * omega_sum * cs);
                        o[2] = (T)oob;
                    }
                } else if (lane == 0) {
                    acc[si][0] += e2;
                    acc[si][1] += oob;
                    acc[si][2] += cs;
                }
            }
        }
        if (!one) {
            __syncthreads();
            for (int si = threadIdx.x; si < ng; si += AE_THREADS) {
                const double e2 = acc[si][0], oob = acc[si][1], cs = acc[si][2];
                T *o = out + (blockIdx.x + (g0 + si) * gridDim.x) * 3;
                o[0] = (T)sqrt(e2);
                o[1] = (T)sqrt(oob + M * omega_sum * cs);
                o[2] = (T)oob;
            }
        }
    }
}

cudaError_t launch_averaged_error(const Axis1D &ax, int64_t batch, const void *spec, int64_t k_lo, int64_t n_freq,
                                  void *out, cudaStream_t st) {
    if (batch <= 0) return cudaSuccess;
    AnyErrSys sy;
    for (int m = 0; m < 8; ++m) sy.s[m] = ax.sys[m];
    int dev = 0, nsm = 148;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, dev);
    int64_t grid = std::min<int64_t>(nsm, batch);  // persistent: one CTA per SM
    if (const char *e = getenv("MCI_AE_GRID")) grid = std::max<int64_t>(1, std::min<int64_t>(atoi(e), batch));  // tests
    if (ax.dtype == MCI_F64) {
        auto k = mci_avg_error_kernel<double>;
        if (cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, AE_SMEM) != cudaSuccess)
            return cudaErrorInvalidValue;
        k<<<(unsigned)grid, AE_THREADS, AE_SMEM, st>>>((const cv<double> *)spec, (int)n_freq, batch, k_lo, ax.M,
                                                       (int)ax.N, ax.K1, ax.Qt, true, sy, ax.omega_sum, (double *)out);
    } else {
        auto k = mci_avg_error_kernel<float>;
        if (cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, AE_SMEM) != cudaSuccess)
            return cudaErrorInvalidValue;
        k<<<(unsigned)grid, AE_THREADS, AE_SMEM, st>>>((const cv<float> *)spec, (int)n_freq, batch, k_lo, ax.M,
                                                       (int)ax.N, ax.K1, ax.Qt, false, sy, ax.omega_sum, (float *)out);
    }
    return cudaGetLastError();
}

cudaError_t launch_anylen_offgrid(const Axis1D &ax, const RowAddr &ra, int64_t rows, const void *g, int64_t n_pts,
                                  const void *t, void *f, void *hf, cudaStream_t st) {
    if (rows <= 0 || n_pts <= 0) return cudaSuccess;
    return anylen_dispatch(ax, ra, rows, g, f, hf, st, t, n_pts);
}

}  // namespace mci
