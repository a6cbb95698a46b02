/*
 * mci.h -- C ABI of the B200-native multichannel-interpolation (MCI) library.
 *
 * Method: arXiv 1802.10291, "fast multichannel interpolation".
 * A real 2*pi-periodic signal f whose spectrum lies in the band
 * I^N = {K1 .. K1+M*N-1}, K1 = -floor(M*N/2) (odd M*N: the symmetric band of
 * Examples 1-2), is reconstructed from N uniform
 * samples g_m(t_n), t_n = 2*pi*n/N, of each of M channel responses
 * g_m = h_m * f (Eq. sysfunction).  The output is
 *   f(t_p) = Re T_N f(t_p),  t_p = 2*pi*p/L,  p = 0..L-1,
 * with T_N the operator of Eq. (appxi operator) PAPER.md:542-545, computed by
 * the FFT form Eq. (DFTexpression) PAPER.md:316-323:
 *   forward DFT of each channel (Lemma 1),
 *   per-bin M x M solve A_n = D_n H_n^{-1} (Eq. matrixeqn1),
 *   Hermitian-part assembly and zero-padding to L, inverse real FFT.
 * Optional Hilbert twin Hf = H(Re T_N f), multiplier -i*sgn(k)
 * (Example 6 PAPER.md:522-531), via one analytic inverse
 * transform (Example 4).
 * Notation: this header's N is the paper's L (samples per channel) and this
 * header's L is the paper's N_out.
 *
 * Conventions (all entry points):
 *  - Status codes, never exceptions.  On create failure *out is set to NULL.
 *  - Device pointers are CUDA device pointers (e.g. torch data_ptr()); the
 *    caller owns them and the stream.  mci_execute_* never allocate, never
 *    synchronise the device, and only enqueue work on `cuda_stream`
 *    (a cudaStream_t; NULL = legacy default stream).
 *  - The plan owns its device tables (inverse matrices, twiddles) and any
 *    workspace; it is immutable after create and may be used concurrently
 *    from several streams and host threads.  Plans with a workspace (four-step,
 *    2D and SISR paths) order their executions on the GPU: each waits (a
 *    cudaStreamWaitEvent on the caller's stream) for the previous execution's
 *    workspace use, whatever stream it ran on, so concurrent calls on one such
 *    plan run one after the other (use one plan per stream for overlap).  The
 *    host-buffer entry points serialise per plan (internal staging buffers).
 *  - Results are deterministic for a given plan and batch (no atomics).
 *  - Arithmetic type is the plan dtype (MCI_F32: float, MCI_F64: double);
 *    host-side plan construction is always fp64.
 */
#ifndef MCI_H
#define MCI_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

typedef struct mci_plan_s *mci_plan; /* opaque */

typedef enum {
    MCI_OK = 0,
    MCI_E_ARG = 1,         /* NULL pointer, non-positive size, bad enum            */
    MCI_E_BAND = 2,        /* band invalid (M*N < 2)                                */
    MCI_E_ALIAS = 3,       /* L < M*N or L not a multiple of N        */
    MCI_E_SINGULAR = 4,    /* some H_n singular (see mci_last_singular_bin)         */
    MCI_E_SIZE = 5,        /* sizes not supported (N < 2, or too large for a path)  */
    MCI_E_CUDA = 6,        /* a CUDA runtime call or kernel launch failed           */
    MCI_E_UNSUPPORTED = 7  /* valid request this build does not implement           */
} mci_status;

typedef enum { MCI_F32 = 0, MCI_F64 = 1 } mci_dtype;

/* Channel system h_m given by its Fourier multiplier b_m(k) (Eq. sysfunction). */
typedef enum {
    MCI_SYS_IDENTITY = 0,   /* b(k) = 1                                  */
    MCI_SYS_DERIVATIVE = 1, /* b(k) = (i k)^order   (Example 2)          */
    MCI_SYS_HILBERT = 2,    /* b(k) = -i sgn(k)     (Examples 3, 5)      */
    MCI_SYS_DELAY = 3,      /* b(k) = exp(i k tau)  (interlaced sampling) */
    MCI_SYS_TABLE = 4       /* b(k) = table[2(k-K1)] + i table[2(k-K1)+1], k in band */
} mci_sys_kind;

typedef struct {
    int kind;            /* mci_sys_kind                                    */
    int order;           /* derivative order (MCI_SYS_DERIVATIVE)           */
    double tau;          /* delay in radians (MCI_SYS_DELAY)                */
    const double *table; /* host, 2*M*N doubles (MCI_SYS_TABLE); copied     */
} mci_system;

enum {
    MCI_OUT_HILBERT = 1u, /* plan also produces Hf                                            */
    MCI_OFFGRID = 2u,     /* plan also evaluates at arbitrary points (mci_execute_offgrid); it is
                             built on the arbitrary-length path                                */
    MCI_COMPLEX = 4u,     /* complex-valued f: complex channel samples
                             in, T_N f itself out (no real part, no Hermitian assembly); any bank
                             (Hermitian or not) and any band K1 (mci_plan_create_band), e.g.
                             Example 5.  Not combinable with MCI_OUT_HILBERT or
                             MCI_OFFGRID in this build (MCI_E_UNSUPPORTED).                      */
    MCI_ANALYSIS = 8u     /* plan also supports mci_consistency_residual and mci_averaged_error
                             (built-in system kinds only: MCI_SYS_TABLE is MCI_E_UNSUPPORTED)     */
};

/* ---- plans ------------------------------------------------------------------------ */

/* 1D plan: M channels (1..8), N samples per channel, L output points.
 * Requirements: N >= 2, L >= M*N, L % N == 0, Hermitian bank (b_m(-k) =
 * conj b_m(k), true for every built-in kind).  N and L powers of two with M*N
 * even use the specialised paths (fused per-row kernels, four-step for long
 * signals); any other sizes (e.g. the paper's SISR widths 107..170, L = 3N, odd
 * M*N) use the arbitrary-length path (mixed-radix FFTs, one CTA per row; it
 * needs 2 max(ceil(M/2) N, L) + M N complex values of shared memory <= 200 KB,
 * else MCI_E_SIZE).
 * H_n (entry (l,m) = b_m(n + l N), Eq. defH) must be
 * invertible for every n in I_1 except the listed Remark-1 null bins
 * (PAPER.md:325-327), whose inverse is set to zero.  Singular: some pivot
 * < 1e-12 * max row norm (SPEC.md:184 reading).  Host arrays are copied. */
mci_status mci_plan_create(mci_plan *out, int M, int64_t N, int64_t L, const mci_system *sys,
                           const int64_t *null_bins, int n_null, mci_dtype dtype, unsigned flags);

/* As mci_plan_create with an explicit band {K1 .. K1+M*N-1} (any integer K1; the real-output
 * paths need the Hermitian reading of the band, see mci_plan_create, so K1 is only free with
 * MCI_COMPLEX or when K1 = -floor(M*N/2)).  With MCI_COMPLEX, mci_execute_1d takes g as
 * [batch][M][N] complex (interleaved re, im in the plan dtype) and writes f as [batch][L]
 * complex; hf must be NULL. */
mci_status mci_plan_create_band(mci_plan *out, int M, int64_t N, int64_t L, int64_t K1, const mci_system *sys,
                                const int64_t *null_bins, int n_null, mci_dtype dtype, unsigned flags);

/* 2D separable plan: tensor bank {sx} x {sy}; channel images
 * g[n][My][Mx][Ny][Nx]; output [n][scale*Ny][scale*Nx].  Re is taken after
 * each 1D pass.  flags must be 0. */
mci_status mci_plan_create_2d(mci_plan *out, int Mx, int64_t Nx, const mci_system *sx, int My,
                              int64_t Ny, const mci_system *sy, int scale, mci_dtype dtype,
                              unsigned flags);

/* Single-image super-resolution by MCI: the
 * paper's scheme on a periodic H x W low-resolution image, scale s >= 3 per axis.  Rows
 * first: channels f, f', f'' along x by three-point centred differences on the grid
 * t = 2 pi x / W (f' = (f[x+1] - f[x-1]) / (2d), f'' = (f[x+1] - 2 f[x] + f[x-1]) / d^2,
 * d = 2 pi / W), then MCI with the Example-2 bank (1, ik, -k^2) to
 * s W points; then the same along y on the row-interpolated image.  Any H, W >= 2
 * (the paper's 107..170 included).  The plan owns a workspace for a chunk of images. */
mci_status mci_plan_create_sisr(mci_plan *out, int64_t H, int64_t W, int scale, mci_dtype dtype);

/* lr: device [n_images][H][W]; hr: device [n_images][s H][s W] (plan dtype). */
mci_status mci_execute_sisr(mci_plan p, int64_t n_images, const void *lr, void *hr, void *cuda_stream);

void mci_plan_destroy(mci_plan p);

/* ---- execution (device buffers) ---------------------------------------------------- */

/* g:  device, [batch][M][N] row-major, plan dtype.
 * f:  device, [batch][L]; hf: device [batch][L] (required iff MCI_OUT_HILBERT, else NULL).
 * Input and output must not overlap.  Asynchronous on cuda_stream. */
mci_status mci_execute_1d(mci_plan p, int64_t batch, const void *g, void *f, void *hf,
                          void *cuda_stream);

/* Off-grid evaluation (Eq. drictexpression / Lemma 2):
 *   f[b][j] = Re T_N f_b(t_j) = sum_k Xf(k) e^{i k t_j},  Xf(k) = (a(k) + conj a(-k)) / 2,
 *   hf[b][j] = H(Re T_N f_b)(t_j)  (only with MCI_OUT_HILBERT; else pass NULL),
 * for arbitrary t_j in radians (any real value).  Plan created with MCI_OFFGRID.
 * g: device [batch][M][N]; t: device [n_pts] (plan dtype), shared by all rows;
 * f, hf: device [batch][n_pts].  Per row the spectrum is computed once, then every point
 * is a direct sum over the band in fp64 (cost O(n_pts M N) per row). */
mci_status mci_execute_offgrid(mci_plan p, int64_t batch, const void *g, int64_t n_pts, const void *t, void *f,
                               void *hf, void *cuda_stream);

/* ---- error analysis, plans created with MCI_ANALYSIS ----------------
 * Consistency residual (Theorem consistency): per row,
 *   out[b] = max_{m,n} |(T_N f * h_m)(t_n) - g_m[n]|,
 * T_N f the complex reconstruction (a^ on the band), resampled through each channel's multiplier.
 * g: device [batch][M][N]; out: device [batch] (plan dtype). */
mci_status mci_consistency_residual(mci_plan p, int64_t batch, const void *g, void *out, void *cuda_stream);

/* Averaged error eps(f, N) (Theorem error, Eq. averageerror) of batches of true
 * spectra a(n), n = k_lo .. k_lo + n_freq - 1 (zero elsewhere), I_k = {K1+(k-1)N .. K1+kN-1}:
 *   eps^2 = sum_{n not in I^N} |a(n)|^2
 *         + sum_{k not in 1..M} sum_{n in I_k} |a(n)|^2 sum_{l=1}^M |sum_m r_m(n+(l-k)N) b_m(n)|^2,
 *   bound^2 = sum_{n not in I^N} |a|^2 + M (sum_m Omega_m) sum_{n not in I^N} sum_m |a(n) b_m(n)|^2,
 *   Omega_m = sup_{i in I^N} |r_m(i)|^2 (Eq. errorestimate, Cauchy-Schwarz reading).
 * spec: device [batch][n_freq] complex (plan dtype, interleaved); out: device [batch][3] =
 * (eps, bound, out-of-band energy), plan dtype; sums accumulated in fp64. */
mci_status mci_averaged_error(mci_plan p, int64_t batch, const void *spec, int64_t k_lo, int64_t n_freq,
                              void *out, void *cuda_stream);

/* g: device [n_images][My][Mx][Ny][Nx]; out: device [n_images][Ly][Lx]. */
mci_status mci_execute_2d(mci_plan p, int64_t n_images, const void *g, void *out,
                          void *cuda_stream);

/* ---- execution (host buffers) -------------------------------------------------------
 * Same layouts, but g/f/hf/out are HOST pointers (page-locked for full speed).
 * The library streams the batch through plan-owned device staging buffers in
 * chunks, overlapping host->device copy, compute and device->host copy on
 * internal streams; returns after the results are in host memory. */
mci_status mci_execute_1d_host(mci_plan p, int64_t batch, const void *g, void *f, void *hf);
mci_status mci_execute_2d_host(mci_plan p, int64_t n_images, const void *g, void *out);

/* ---- introspection ------------------------------------------------------------------- */
double mci_plan_cond_max(mci_plan p);          /* max ||H_n||_1 ||H_n^{-1}||_1 */
int64_t mci_last_singular_bin(void);           /* n of the last MCI_E_SINGULAR (this thread) */
size_t mci_plan_workspace_bytes(mci_plan p);   /* device bytes owned by the plan            */
int mci_plan_path(mci_plan p);                 /* 0 fused 1D, 1 four-step 1D, 2 separable 2D, 3 SISR */
int64_t mci_plan_launches(mci_plan p, int64_t batch); /* kernels one execute enqueues       */
const char *mci_status_str(mci_status s);
const char *mci_version(void);

#ifdef __cplusplus
}
#endif
#endif /* MCI_H */
