/*
 * mci_oracle.c -- plain, slow, obviously-correct fp64 CPU oracle for MCI.
 *
 * TEST INFRASTRUCTURE ONLY.  Only tests/, __graft_entry__.smoke() and the
 * cpu_baseline / --impl reference legs of bench.py may load this library.
 * It shares no code, header, table or constant generator with the CUDA path
 * (paper_1802_10291_b200/csrc) and never calls it.
 *
 * What it computes is the paper's definition (arXiv 1802.10291, PAPER.md):
 *
 *   T_N f(t) = (1/L_p) sum_{m=1}^{M} sum_{p=0}^{L_p-1} g_m(t_p) y_m(t - t_p)
 *       Theorem 1 Eq. (drictexpression) PAPER.md:307-314 and the
 *       approximation operator Eq. (appxi operator) PAPER.md:542-545,
 *   y_m(t) = sum_{n in I^N} r_m(n) e^{i n t}                Eq. (ym) PAPER.md:256-259,
 *   r_m(n) = q_{mk}(n + L_p - k L_p) for n in I_k           Eq. (defrm) PAPER.md:250-255,
 *   q_{mk}(n) = (H_n^{-1})_{mk},  (H_n)_{jk} = b_k(n + jL_p - L_p)  Eq. (defH) PAPER.md:236-249,
 *
 * where the paper's L_p (samples per channel) is this code's N, the band is
 * I^N = {K1 .. K1 + M N - 1}, samples are at t_n = 2 pi n/N and outputs at
 * t_p = 2 pi p/L (SURVEY.md §0 notation map).  The returned output is the
 * real part Re T_N f (SURVEY.md §8(c) reading 3) and the Hilbert output is
 * Re H T_N f with multiplier -i sgn(n) (Example 6 PAPER.md:522-531).
 * Singular H_n: pivot < 1e-12 * largest initial row max-norm (SPEC.md:184
 * reading); Remark 1 null bins are zero-filled.
 *
 * Nothing here is blocked, fused or reordered beyond the formulas: the kernel
 * table is the literal sum of Eq. (ym) at grid points (exact integer phase
 * reduction (k s) mod L, fp64 cos/sin), and evaluation is the literal double
 * sum of Eq. (drictexpression).
 */
#include <complex.h>
#include <math.h>
#include <stdint.h>
#include <stdlib.h>
#include <string.h>
#ifdef _OPENMP
#include <omp.h>
#endif

enum { ORA_IDENTITY = 0, ORA_DERIVATIVE = 1, ORA_HILBERT = 2, ORA_DELAY = 3, ORA_TABLE = 4 };

static const double ORA_PI = 3.14159265358979323846264338327950288;

static void set_threads(int threads) {
#ifdef _OPENMP
    if (threads > 0) omp_set_num_threads(threads);
#else
    (void)threads;
#endif
}

/* b_m(n): the channel's Fourier multiplier, Eq. (sysfunction) PAPER.md:139-145.
 * derivative: (i n)^order (Example 2); hilbert: -i sgn(n)
 * (PAPER.md:110); delay: e^{i n tau}; table: caller-supplied b(n) on the band. */
static double complex multiplier(int kind, int order, double tau, const double *table,
                                 int64_t K1, int64_t n) {
    switch (kind) {
    case ORA_IDENTITY:
        return 1.0;
    case ORA_DERIVATIVE: {
        double complex v = 1.0;
        for (int i = 0; i < order; ++i) v *= I * (double)n;
        return v;
    }
    case ORA_HILBERT:
        return n > 0 ? -I : (n < 0 ? I : 0.0);
    case ORA_DELAY:
        return cexp(I * (double)n * tau);
    case ORA_TABLE: {
        int64_t idx = n - K1;
        return table[2 * idx] + I * table[2 * idx + 1];
    }
    }
    return 0.0;
}

/* Multiplier of one channel at band frequency n (exposed for tests). */
void ora_multiplier(int kind, int order, double tau, const double *table, int64_t K1,
                    int64_t n, double *re, double *im) {
    double complex v = multiplier(kind, order, tau, table, K1, n);
    *re = creal(v);
    *im = cimag(v);
}

/* Gauss-Jordan inversion with partial pivoting of an M x M complex matrix.
 * A is destroyed.  Returns 0, or 1 if a pivot falls below thresh. */
static int gauss_jordan_inverse(int M, double complex *A, double complex *Ainv, double thresh) {
    for (int i = 0; i < M; ++i)
        for (int j = 0; j < M; ++j) Ainv[i * M + j] = (i == j) ? 1.0 : 0.0;
    for (int c = 0; c < M; ++c) {
        int piv = c;
        double best = cabs(A[c * M + c]);
        for (int r = c + 1; r < M; ++r)
            if (cabs(A[r * M + c]) > best) { best = cabs(A[r * M + c]); piv = r; }
        if (!(best >= thresh) || best == 0.0) return 1;
        if (piv != c)
            for (int j = 0; j < M; ++j) {
                double complex t = A[c * M + j]; A[c * M + j] = A[piv * M + j]; A[piv * M + j] = t;
                t = Ainv[c * M + j]; Ainv[c * M + j] = Ainv[piv * M + j]; Ainv[piv * M + j] = t;
            }
        double complex inv = 1.0 / A[c * M + c];
        for (int j = 0; j < M; ++j) { A[c * M + j] *= inv; Ainv[c * M + j] *= inv; }
        for (int r = 0; r < M; ++r) {
            if (r == c) continue;
            double complex f = A[r * M + c];
            if (f == 0.0) continue;
            for (int j = 0; j < M; ++j) {
                A[r * M + j] -= f * A[c * M + j];
                Ainv[r * M + j] -= f * Ainv[c * M + j];
            }
        }
    }
    return 0;
}

/* For every n in I_1 = {K1 .. K1+N-1} build H_n (Eq. defH: row l = shift, column
 * m = channel, entry b_m(n + l N)) and invert it.  Output Q[(n-K1)][m][l] =
 * q_{m,l}(n) (re, im interleaved).  Null bins get Q = 0 (Remark 1).
 * Returns 0 on success, 1 + (n - K1) of the first singular non-null bin,
 * or -1 on bad arguments.  *cond_max receives max ||H||_1 ||H^{-1}||_1. */
int ora_inverse(int M, int64_t N, int64_t K1, const int *kind, const int *order,
                const double *tau, const double *const *tables, const int64_t *null_bins,
                int n_null, double *Q, double *cond_max) {
    if (M < 1 || M > 16 || N < 1) return -1;
    double complex H[256], A[256], Hinv[256];
    double cmax = 0.0;
    for (int64_t jj = 0; jj < N; ++jj) {
        int64_t n = K1 + jj;
        int is_null = 0;
        for (int z = 0; z < n_null; ++z)
            if (null_bins[z] == n) is_null = 1;
        double *q = Q + (size_t)jj * M * M * 2;
        if (is_null) {
            memset(q, 0, sizeof(double) * 2 * M * M);
            continue;
        }
        double rowmax = 0.0;
        for (int l = 0; l < M; ++l) {
            double rmax = 0.0;
            for (int m = 0; m < M; ++m) {
                H[l * M + m] = multiplier(kind[m], order[m], tau[m], tables ? tables[m] : NULL, K1,
                                          n + (int64_t)l * N);
                A[l * M + m] = H[l * M + m];
                if (cabs(H[l * M + m]) > rmax) rmax = cabs(H[l * M + m]);
            }
            if (rmax > rowmax) rowmax = rmax;
        }
        if (gauss_jordan_inverse(M, A, Hinv, 1e-12 * rowmax)) return (int)(1 + jj);
        /* 1-norm condition number (max column sum) */
        double n1 = 0.0, n2 = 0.0;
        for (int c = 0; c < M; ++c) {
            double s1 = 0.0, s2 = 0.0;
            for (int r = 0; r < M; ++r) { s1 += cabs(H[r * M + c]); s2 += cabs(Hinv[r * M + c]); }
            if (s1 > n1) n1 = s1;
            if (s2 > n2) n2 = s2;
        }
        if (n1 * n2 > cmax) cmax = n1 * n2;
        /* Hinv[m][l] = q_{m,l}(n) */
        for (int m = 0; m < M; ++m)
            for (int l = 0; l < M; ++l) {
                q[2 * (m * M + l)] = creal(Hinv[m * M + l]);
                q[2 * (m * M + l) + 1] = cimag(Hinv[m * M + l]);
            }
    }
    if (cond_max) *cond_max = cmax;
    return 0;
}

/* r_m(k) for k in the band, Eq. (defrm): k = n + l N with n in I_1 gives
 * r_m(k) = q_{m,l}(n).  r[m][k-K1] (re, im). */
void ora_r_from_q(int M, int64_t N, int64_t K1, const double *Q, double *r) {
    int64_t MN = (int64_t)M * N;
    for (int m = 0; m < M; ++m)
        for (int64_t kk = 0; kk < MN; ++kk) {
            int64_t jj = kk % N, l = kk / N; /* k = K1 + kk = (K1 + jj) + l N */
            const double *q = Q + (size_t)jj * M * M * 2;
            r[2 * ((size_t)m * MN + kk)] = q[2 * (m * M + l)];
            r[2 * ((size_t)m * MN + kk) + 1] = q[2 * (m * M + l) + 1];
        }
}

static int64_t mod64(int64_t a, int64_t b) {
    int64_t r = a % b;
    return r < 0 ? r + b : r;
}

/* Kernel table on the output grid, Eq. (ym) at t = 2 pi s / L:
 *   Y[m][s] = Re sum_{k in band} w(k) r_m(k) e^{2 pi i ((k s) mod L)/L},
 * w(k) = 1 (f) or -i sgn(k) (Hf: Hilbert transform of y_m, Example 6). */
int ora_kernel_table(int M, int64_t MN, int64_t K1, int64_t L, const double *r, int hilbert,
                     double *Y, int threads) {
    if (L < 1) return -1;
    set_threads(threads);
    double *cs = (double *)malloc(sizeof(double) * 2 * L);
    if (!cs) return -2;
    for (int64_t u = 0; u < L; ++u) {
        cs[2 * u] = cos(2.0 * ORA_PI * (double)u / (double)L);
        cs[2 * u + 1] = sin(2.0 * ORA_PI * (double)u / (double)L);
    }
    for (int m = 0; m < M; ++m) {
        const double *rm = r + 2 * (size_t)m * MN;
#pragma omp parallel for schedule(static)
        for (int64_t s = 0; s < L; ++s) {
            double acc = 0.0;
            for (int64_t kk = 0; kk < MN; ++kk) {
                int64_t k = K1 + kk;
                double complex rk = rm[2 * kk] + I * rm[2 * kk + 1];
                if (hilbert) rk *= (k > 0 ? -I : (k < 0 ? I : 0.0));
                int64_t u = mod64(mod64(k, L) * s, L);
                acc += creal(rk) * cs[2 * u] - cimag(rk) * cs[2 * u + 1];
            }
            Y[(size_t)m * L + s] = acc;
        }
    }
    free(cs);
    return 0;
}

/* Eq. (drictexpression) on the output grid (requires L % N == 0):
 *   f[p] = (1/N) sum_m sum_n g_m[n] Y_m[(p - n L/N) mod L],  p = 0..L-1,
 * for `rows` independent rows g[row][m][n]. */
int ora_eval_grid(int M, int64_t N, int64_t L, const double *Y, int64_t rows, const double *g,
                  double *f, int threads) {
    if (L % N != 0) return -1;
    set_threads(threads);
    int64_t step = L / N;
#pragma omp parallel for collapse(2) schedule(static)
    for (int64_t row = 0; row < rows; ++row)
        for (int64_t p = 0; p < L; ++p) {
            const double *gr = g + (size_t)row * M * N;
            double acc = 0.0;
            for (int m = 0; m < M; ++m)
                for (int64_t n = 0; n < N; ++n)
                    acc += gr[(size_t)m * N + n] * Y[(size_t)m * L + mod64(p - n * step, L)];
            f[(size_t)row * L + p] = acc / (double)N;
        }
    return 0;
}

/* Same formula at a list of output indices p[i] for one row g[m][n]. */
int ora_eval_grid_points(int M, int64_t N, int64_t L, const double *Y, const double *g,
                         int64_t np, const int64_t *p, double *out, int threads) {
    if (L % N != 0) return -1;
    set_threads(threads);
    int64_t step = L / N;
#pragma omp parallel for schedule(static)
    for (int64_t i = 0; i < np; ++i) {
        double acc = 0.0;
        for (int m = 0; m < M; ++m)
            for (int64_t n = 0; n < N; ++n)
                acc += g[(size_t)m * N + n] * Y[(size_t)m * L + mod64(p[i] - n * step, L)];
        out[i] = acc / (double)N;
    }
    return 0;
}

/* Off-grid evaluation straight from the definitions (any t, any N):
 *   out(t) = (1/N) sum_m sum_n g_m[n] Re sum_k w(k) r_m(k) e^{i k (t - 2 pi n/N)}.
 * O(M N MN) per point: tiny sizes only (paper's Table approximatedtable). */
int ora_eval_offgrid(int M, int64_t N, int64_t K1, const double *r, int hilbert, const double *g,
                     int64_t nt, const double *t, double *out, int threads) {
    set_threads(threads);
    int64_t MN = (int64_t)M * N;
#pragma omp parallel for schedule(static)
    for (int64_t i = 0; i < nt; ++i) {
        double acc = 0.0;
        for (int m = 0; m < M; ++m)
            for (int64_t n = 0; n < N; ++n) {
                double tau = t[i] - 2.0 * ORA_PI * (double)n / (double)N;
                double y = 0.0;
                for (int64_t kk = 0; kk < MN; ++kk) {
                    int64_t k = K1 + kk;
                    double complex rk = r[2 * ((size_t)m * MN + kk)] + I * r[2 * ((size_t)m * MN + kk) + 1];
                    if (hilbert) rk *= (k > 0 ? -I : (k < 0 ? I : 0.0));
                    y += creal(rk * cexp(I * (double)k * tau));
                }
                acc += g[(size_t)m * N + n] * y;
            }
        out[i] = acc / (double)N;
    }
    return 0;
}

/* Delay bank b_m(k) = e^{i k tau_m}, tau_m = 2 pi m/(M N), band {-K..K-1}, K = MN/2.
 * Its inverse is closed-form: H_n = W diag(e^{i n tau_m}) with W[l][m] =
 * e^{2 pi i l m/M}, so r_m(k) = e^{-i k tau_m}/M and
 *   Re y_m(t) = (1/M) cos(u/2) sin(K u)/sin(u/2),  u = t - tau_m  (2K/M at u = 0 mod 2 pi).
 * With t = 2 pi p/L, t_n = 2 pi n/N and L % (M N) == 0 every shift is
 * u = 2 pi s'/L, s' = p - n L/N - m L/(MN), reduced exactly mod L. */
static double delay_kernel_re(int M, int64_t K, int64_t L, int64_t s) {
    s = mod64(s, L);
    if (s == 0) return 2.0 * (double)K / (double)M;
    double half = ORA_PI * (double)s / (double)L;               /* u/2 */
    double sinKu = sin(2.0 * ORA_PI * (double)mod64(K * s, L) / (double)L);
    return cos(half) * sinKu / (sin(half) * (double)M);
}

int ora_delay_kernel_table(int M, int64_t N, int64_t L, double *Y) {
    int64_t MN = (int64_t)M * N;
    if (L % MN != 0 || MN % 2 != 0) return -1;
    int64_t K = MN / 2, sub = L / MN;
    for (int m = 0; m < M; ++m)
        for (int64_t s = 0; s < L; ++s) Y[(size_t)m * L + s] = delay_kernel_re(M, K, L, s - m * sub);
    return 0;
}

int ora_eval_delay_points(int M, int64_t N, int64_t L, const double *g, int64_t np,
                          const int64_t *p, double *out, int threads) {
    int64_t MN = (int64_t)M * N;
    if (L % MN != 0 || MN % 2 != 0) return -1;
    set_threads(threads);
    int64_t K = MN / 2, step = L / N, sub = L / MN;
#pragma omp parallel for schedule(static)
    for (int64_t i = 0; i < np; ++i) {
        double acc = 0.0;
        for (int m = 0; m < M; ++m)
            for (int64_t n = 0; n < N; ++n)
                acc += g[(size_t)m * N + n] * delay_kernel_re(M, K, L, p[i] - n * step - m * sub);
        out[i] = acc / (double)N;
    }
    return 0;
}
