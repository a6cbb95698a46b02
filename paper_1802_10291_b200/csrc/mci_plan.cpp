// Plan builder and C-ABI entry points (include/mci.h).
//
// Host side, fp64: for every class q = 0..N/2 (j_q in I_1 = {-K .. -K+N-1},
// j_q = q mod N) build H_{j_q}[l][m] = b_m(j_q + l N) (Eq. defH),
// invert it by LU with partial pivoting, and pack Qt_q = H_{j_q}^{-1} / N
// (the 1/N of d_m = G_m/N, Lemma 1, is folded in).  Classes
// N/2+1..N-1 are never needed: for a Hermitian bank they are the conjugate
// mirrors of classes N-q.  Remark 1 null bins get Qt = 0.
// Twiddle tables are rounded from fp64.  Nothing here runs per execute.
#include <cuda_runtime.h>

#include <algorithm>
#include <cmath>
#include <complex>
#include <cstdio>
#include <cstring>
#include <cstdlib>
#include <mutex>
#include <new>
#include <type_traits>
#include <vector>

#include "mci_internal.h"

using cd = std::complex<double>;

namespace {

thread_local int64_t g_last_singular = 0;
const double PI = 3.14159265358979323846264338327950288;

bool is_pow2(int64_t x) { return x > 0 && (x & (x - 1)) == 0; }
int64_t next_pow2(int64_t x) {
    int64_t p = 1;
    while (p < x) p <<= 1;
    return p;
}

cd sys_multiplier(const mci_system &s, int64_t K1, int64_t k) {
    switch (s.kind) {
    case MCI_SYS_IDENTITY: return 1.0;
    case MCI_SYS_DERIVATIVE: {
        cd v = 1.0;
        for (int i = 0; i < s.order; ++i) v *= cd(0.0, (double)k);
        return v;
    }
    case MCI_SYS_HILBERT: return k > 0 ? cd(0, -1) : (k < 0 ? cd(0, 1) : cd(0, 0));
    case MCI_SYS_DELAY: {
        double ang = std::fmod((double)k * s.tau, 2 * PI);
        return cd(std::cos(ang), std::sin(ang));
    }
    case MCI_SYS_TABLE: return cd(s.table[2 * (k - K1)], s.table[2 * (k - K1) + 1]);
    }
    return 0.0;
}

// LU with partial pivoting; returns false if a pivot < thresh.  inv = A^{-1}.
bool lu_inverse(int M, std::vector<cd> A, std::vector<cd> &inv, double thresh) {
    std::vector<int> piv(M);
    for (int i = 0; i < M; ++i) piv[i] = i;
    for (int c = 0; c < M; ++c) {
        int p = c;
        for (int r = c + 1; r < M; ++r)
            if (std::abs(A[r * M + c]) > std::abs(A[p * M + c])) p = r;
        if (!(std::abs(A[p * M + c]) >= thresh) || std::abs(A[p * M + c]) == 0.0) return false;
        if (p != c) {
            for (int j = 0; j < M; ++j) std::swap(A[c * M + j], A[p * M + j]);
            std::swap(piv[c], piv[p]);
        }
        for (int r = c + 1; r < M; ++r) {
            cd f = A[r * M + c] / A[c * M + c];
            A[r * M + c] = f;
            for (int j = c + 1; j < M; ++j) A[r * M + j] -= f * A[c * M + j];
        }
    }
    inv.assign(M * M, 0.0);
    for (int col = 0; col < M; ++col) {
        std::vector<cd> y(M);
        for (int i = 0; i < M; ++i) {  // forward substitution on P e_col
            cd s = (piv[i] == col) ? 1.0 : 0.0;
            for (int j = 0; j < i; ++j) s -= A[i * M + j] * y[j];
            y[i] = s;
        }
        for (int i = M - 1; i >= 0; --i) {
            cd s = y[i];
            for (int j = i + 1; j < M; ++j) s -= A[i * M + j] * inv[j * M + col];
            inv[i * M + col] = s / A[i * M + i];
        }
    }
    return true;
}

template <typename T> void push_c(std::vector<T> &v, cd z) {
    v.push_back((T)z.real());
    v.push_back((T)z.imag());
}

// e^{sign 2 pi i m / P} for m in [0, count) at stride `stride` (exact integer reduction)
template <typename T> void push_roots(std::vector<T> &v, int64_t P, int64_t count, int64_t stride, int sign) {
    for (int64_t i = 0; i < count; ++i) {
        int64_t m = (i * stride) % P;
        double a = 2.0 * PI * (double)m / (double)P;
        push_c(v, cd(std::cos(a), sign * std::sin(a)));
    }
}

}  // namespace

struct mci_plan_s {
    int path = mci::PATH_FUSED;
    int dtype = MCI_F32;
    unsigned flags = 0;
    mci::Axis1D ax;          // 1D plan, or the x axis (row pass) of a 2D plan
    mci::Axis1D ay;          // y axis (column pass) of a 2D plan
    int Mx = 0, My = 0;
    int64_t Nx = 0, Ny = 0, Lx = 0, Ly = 0;
    void *tables = nullptr;  // one device block for every table
    void *ws = nullptr;      // workspace (four-step / 2D intermediate)
    size_t ws_bytes = 0;
    int64_t ws_units = 0;    // signals (four-step) or images (2D) per workspace fill
    double cond_max = 0.0;
    // host-buffer execution (allocated on first use)
    void *stage[4] = {nullptr, nullptr, nullptr, nullptr};
    size_t stage_bytes[2] = {0, 0};
    int64_t stage_rows = 0;
    cudaStream_t hs[2] = {nullptr, nullptr};
    // 2D with two workspace halves: odd chunks on a second stream (MCI_2D_STREAMS=2)
    int ws_halves = 1;
    cudaStream_t s2 = nullptr;
    cudaEvent_t ev[2] = {nullptr, nullptr};
    // plans with a workspace (four-step, 2D, SISR) or host staging are shared state: executions
    // are ordered on the GPU by an event (each waits for the previous one's workspace use, on
    // whatever stream it ran) and on the host by a mutex around the enqueue
    std::mutex mu;
    cudaEvent_t ws_ev = nullptr;
    bool ws_ev_recorded = false;
};

// Enqueue f(stream) for a plan with a workspace: after every earlier execution of the plan (their
// workspace use, on any stream), and before every later one.  Plans without one run directly.
template <typename F> mci_status with_workspace(mci_plan p, cudaStream_t st, F &&f) {
    if (!p->ws) return f(st);
    std::lock_guard<std::mutex> lock(p->mu);
    if (!p->ws_ev && cudaEventCreateWithFlags(&p->ws_ev, cudaEventDisableTiming) != cudaSuccess) return MCI_E_CUDA;
    if (p->ws_ev_recorded && cudaStreamWaitEvent(st, p->ws_ev, 0) != cudaSuccess) return MCI_E_CUDA;
    const mci_status s = f(st);
    if (cudaEventRecord(p->ws_ev, st) != cudaSuccess) return MCI_E_CUDA;
    p->ws_ev_recorded = true;
    return s;
}


namespace {

size_t esize(int dtype) { return dtype == MCI_F64 ? 8 : 4; }

// Build one axis: validation, inverse tables, twiddles (host vectors, scalar type T).
template <typename T>
mci_status build_axis(mci::Axis1D &ax, int M, int64_t N, int64_t L, const mci_system *sys, const int64_t *null_bins,
                      int n_null, bool analytic, bool fourstep, std::vector<T> &blob, std::vector<size_t> &offs,
                      double &cond_max) {
    if (M < 1 || M > 8 || !sys) return MCI_E_ARG;
    if (!is_pow2(N) || N < 2) return MCI_E_SIZE;
    if ((M * N) % 2) return MCI_E_BAND;
    if (!is_pow2(L) || L < M * N || L % N) return MCI_E_ALIAS;
    const int64_t K = (int64_t)M * N / 2, K1 = -K;
    for (int m = 0; m < M; ++m) {
        const mci_system &s = sys[m];
        if (s.kind < MCI_SYS_IDENTITY || s.kind > MCI_SYS_TABLE) return MCI_E_ARG;
        if (s.kind == MCI_SYS_DERIVATIVE && s.order < 0) return MCI_E_ARG;
        if (s.kind == MCI_SYS_TABLE) {
            if (!s.table) return MCI_E_ARG;
            for (int64_t k = 1; k < K; ++k) {  // Hermitian requirement of the real-output path
                cd a = sys_multiplier(s, K1, k), b = sys_multiplier(s, K1, -k);
                if (std::abs(a - std::conj(b)) > 1e-12 * (1 + std::abs(a))) return MCI_E_UNSUPPORTED;
            }
        }
    }
    ax.M = M; ax.N = N; ax.L = L; ax.K = K; ax.analytic = analytic ? 1 : 0;
    ax.S = analytic ? next_pow2(K) : next_pow2(2 * K);
    if (ax.S < 16) ax.S = std::min<int64_t>(16, L);
    ax.R = L / ax.S;
    // ---- inverse tables per class q = 0..N/2
    offs.push_back(blob.size());  // Qt
    std::vector<cd> H(M * M), inv;
    cond_max = 0.0;
    for (int64_t q = 0; q <= N / 2; ++q) {
        const int64_t jq = -K + (((q + K) % N) + N) % N;
        bool is_null = false;
        for (int z = 0; z < n_null; ++z)
            if (null_bins[z] == jq) is_null = true;
        double rowmax = 0.0;
        for (int l = 0; l < M; ++l) {
            double rm = 0.0;
            for (int m = 0; m < M; ++m) {
                H[l * M + m] = sys_multiplier(sys[m], K1, jq + (int64_t)l * N);
                rm = std::max(rm, std::abs(H[l * M + m]));
            }
            rowmax = std::max(rowmax, rm);
        }
        if (is_null) {
            inv.assign(M * M, 0.0);
        } else {
            if (!lu_inverse(M, H, inv, 1e-12 * rowmax)) {
                g_last_singular = jq;
                return MCI_E_SINGULAR;
            }
            double n1 = 0, n2 = 0;
            for (int c = 0; c < M; ++c) {
                double s1 = 0, s2 = 0;
                for (int r = 0; r < M; ++r) { s1 += std::abs(H[r * M + c]); s2 += std::abs(inv[r * M + c]); }
                n1 = std::max(n1, s1);
                n2 = std::max(n2, s2);
            }
            cond_max = std::max(cond_max, n1 * n2);
        }
        for (int m = 0; m < M; ++m)
            for (int l = 0; l < M; ++l) push_c(blob, inv[m * M + l] / (double)N);
    }
    // uniform interleaved delay bank: H_j = W diag(e^{i j tau_m}),
    // W[l][m] = e^{2 pi i l m / M}, so H_j^{-1} = diag(e^{-i j tau_m}) W^H / M
    {
        bool du = M == 4 && n_null == 0 && L % ((int64_t)M * N) == 0 && !getenv("MCI_ROW_QTAB");
        for (int m = 0; du && m < M; ++m)
            du = sys[m].kind == MCI_SYS_DELAY &&
                 std::abs(sys[m].tau - 2 * PI * m / ((double)M * N)) <= 1e-12 * (1 + 2 * PI * m / ((double)M * N));
        ax.bank_delay_uniform = du ? 1 : 0;
        bool um = !getenv("MCI_FS_CHANNEL_MAX");
        for (int m = 0; um && m < M; ++m) um = sys[m].kind == MCI_SYS_IDENTITY || sys[m].kind == MCI_SYS_DELAY;
        ax.bank_unimodular = um ? 1 : 0;
    }
    // ---- forward-sign root table e^{-2 pi i m/TW}
    if (fourstep) ax.TW = std::max<int64_t>({1024, N / 1024, ax.S / 1024});
    else ax.TW = std::max<int64_t>({N, ax.S, 1024});
    offs.push_back(blob.size());
    push_roots(blob, ax.TW, ax.TW, 1, -1);
    // ---- two-level tables: [L/LO hi][LO lo] of e^{+2 pi i m/L} (+ N (forward), S (inverse) for four-step)
    ax.LO = std::min<int64_t>(L, 1024);
    offs.push_back(blob.size());
    push_roots(blob, L, L / ax.LO, ax.LO, +1);
    push_roots(blob, L, ax.LO, 1, +1);
    if (!fourstep && !getenv("MCI_DISABLE_ROW") && std::is_same<T, float>::value) {
        ax.dtype = MCI_F32;
        if (mci::row_supported(ax) || mci::rowg_supported(ax)) {
            // Example 2 bank (f, f', f'') with no null bins: the row kernel evaluates the
            // paper's closed-form H^{-1} instead of reading the table
            ax.bank_deriv012 = (M == 3 && n_null == 0 && sys[0].kind == MCI_SYS_IDENTITY &&
                                sys[1].kind == MCI_SYS_DERIVATIVE && sys[1].order == 1 &&
                                sys[2].kind == MCI_SYS_DERIVATIVE && sys[2].order == 2 && !getenv("MCI_ROW_QTAB"))
                                   ? 1 : 0;
            // derivative bank (ik)^m, m < M (the row-kernel family's Vandermonde closed form)
            bool dm = n_null == 0 && !getenv("MCI_ROW_QTAB") && sys[0].kind == MCI_SYS_IDENTITY;
            for (int m = 1; dm && m < M; ++m) dm = sys[m].kind == MCI_SYS_DERIVATIVE && sys[m].order == m;
            ax.bank_derivM = dm ? 1 : 0;
            // time-interleaved sampling: tau_m = 2 pi m / (M N), M in {2, 4, 8}
            bool ti = n_null == 0 && !getenv("MCI_ROW_QTAB") && (M == 2 || M == 4 || M == 8);
            for (int m = 0; ti && m < M; ++m) {
                const double tau = 2 * PI * m / ((double)M * N);
                ti = (sys[m].kind == MCI_SYS_DELAY && std::abs(sys[m].tau - tau) <= 1e-12 * (1 + tau)) ||
                     (m == 0 && sys[m].kind == MCI_SYS_IDENTITY);
            }
            ax.bank_delay_ti = ti ? 1 : 0;
            // the config-2 shape runs the tuned kernel (mci_row.cu); the other shapes run the
            // family kernel (mci_rowg.cu).  A/B: MCI_ROWG=1 runs the family kernel on the config-2
            // shape too, MCI_ROWG=2 in addition with the generic derivative-bank solve
            const int fam = getenv("MCI_ROWG") ? atoi(getenv("MCI_ROWG")) : 0;
            ax.rowg = !mci::row_supported(ax) || fam >= 1;
            if (fam == 2 && ax.bank_derivM) ax.bank_deriv012 = 0;
            // row kernel tables: [wp: K+1][fw2: 32x32][itw: 64x64][fw3: 16x64][fw8: 8x8]
            // + family: [tw256: 16x16][tw2k: 2048][ainv: M x M reals, padded to an even count]
            offs.push_back(blob.size());
            push_roots(blob, L, K + 1, 1, +1);
            for (int j = 0; j < 32; ++j) push_roots(blob, 1024, 32, j, -1);
            for (int j = 0; j < 64; ++j) push_roots(blob, 4096, 64, j, +1);
            for (int j = 0; j < 16; ++j) push_roots(blob, 1024, 64, j, -1);
            for (int j = 0; j < 8; ++j) push_roots(blob, 64, 8, j, -1);
            for (int j = 0; j < 16; ++j) push_roots(blob, 256, 16, j, -1);
            push_roots(blob, 2048, 2048, 1, -1);
            {  // W[r][l] = (l N)^r; v = W^{-1} f, stored as ainv[l M + r] = (W^{-1})[l][r] / N
                std::vector<cd> W(M * M), Wi;
                for (int r = 0; r < M; ++r)
                    for (int l = 0; l < M; ++l) W[r * M + l] = std::pow((double)l * (double)N, (double)r);
                if (!lu_inverse(M, W, Wi, 0.0)) return MCI_E_ARG;
                for (int l = 0; l < M; ++l)
                    for (int r = 0; r < M; ++r) blob.push_back((T)(Wi[l * M + r].real() / (double)N));
                if ((M * M) & 1) blob.push_back((T)0);
            }
            push_roots(blob, 512, 512, 1, -1);  // family, N = 512: e^{-2 pi i m / 512}
            ax.row_variant = getenv("MCI_ROW_VARIANT") ? atoi(getenv("MCI_ROW_VARIANT")) : 0;
            ax.special = 1;
        } else if (mci::line_supported(ax)) {
            // (1, ik) bank with no null bins: closed-form inverse instead of the Q~ table
            ax.bank_deriv01 = (M == 2 && n_null == 0 && sys[0].kind == MCI_SYS_IDENTITY &&
                               sys[1].kind == MCI_SYS_DERIVATIVE && sys[1].order == 1 && !getenv("MCI_ROW_QTAB"))
                                  ? 1 : 0;
            // line kernel tables: [wp: K+1][fwt: 32x16][iw: 32x32]
            offs.push_back(blob.size());
            push_roots(blob, L, K + 1, 1, +1);
            for (int j = 0; j < 32; ++j) push_roots(blob, 512, 16, j, -1);
            for (int j = 0; j < 32; ++j) push_roots(blob, 1024, 32, j, +1);
            ax.special = 2;
        } else if (mci::hilbert_supported(ax)) {
            // Hilbert kernel tables: [whi: 256][wlo: 256][itw: 32 x 65 (row stride 65; col 64 unused)]
            ax.bank_deriv01 = (M == 2 && n_null == 0 && sys[0].kind == MCI_SYS_IDENTITY &&
                               sys[1].kind == MCI_SYS_DERIVATIVE && sys[1].order == 1 && !getenv("MCI_ROW_QTAB"))
                                  ? 1 : 0;
            offs.push_back(blob.size());
            push_roots(blob, L, 256, 256, +1);
            push_roots(blob, L, 256, 1, +1);
            for (int j = 0; j < 32; ++j) push_roots(blob, 2048, 65, j, +1);
            ax.special = 3;
        }
    }
    if (fourstep) {
        push_roots(blob, N, N / ax.LO, ax.LO, -1);
        push_roots(blob, N, ax.LO, 1, -1);
        push_roots(blob, ax.S, ax.S / ax.LO, ax.LO, +1);
        push_roots(blob, ax.S, ax.LO, 1, +1);
        // packed four-step kernels' shared-memory tables, laid out as they are copied (one bulk
        // copy per CTA instead of per-entry gathers from twF): [tw16: 256][tw32: 1024][tw128: 96]
        // tw16[q] = e^{-2 pi i 4 (q >> 4)(q & 15) / 1024}, tw32[q] = e^{-2 pi i (q >> 5)(q & 31) / 1024},
        // tw128[q] = e^{+2 pi i 8 ((q >> 5) + 1)(q & 31) / 1024}  (the same roots as twF with TW = 1024)
        offs.push_back(blob.size());
        auto root1024 = [&](int64_t m, int sign) {
            m %= 1024;
            const double a = 2.0 * PI * (double)m / 1024.0;
            push_c(blob, cd(std::cos(a), sign * std::sin(a)));
        };
        for (int q = 0; q < 256; ++q) root1024(4 * (q >> 4) * (q & 15), -1);
        for (int q = 0; q < 1024; ++q) root1024((q >> 5) * (q & 31), -1);
        for (int q = 0; q < 96; ++q) root1024(8 * ((q >> 5) + 1) * (q & 31), +1);
    }
    return MCI_OK;
}

// Arbitrary-length axis (mci_anylen.cu): any N >= 2, L % N == 0,
// L >= MN, band K1 = -floor(MN/2).  Q~ for every class q in [0, N), full root tables.
bool use_anylen(int M, int64_t N, int64_t L) {
    return !(is_pow2(N) && is_pow2(L) && ((int64_t)M * N) % 2 == 0) || getenv("MCI_FORCE_ANYLEN");
}

mci::AnyRadix radix_plan(int64_t n) {
    mci::AnyRadix p;
    auto push = [&](int r) { p.r[p.n++] = r; };
    while (n % 4 == 0 && p.n < 23) { push(4); n /= 4; }
    if (n % 2 == 0) { push(2); n /= 2; }
    for (int r : {3, 5, 7})
        while (n % r == 0 && p.n < 23) { push(r); n /= r; }
    for (int64_t d = 11; d * d <= n && p.n < 23; d += 2)
        while (n % d == 0) { push((int)d); n /= d; }
    if (n > 1) push((int)n);
    // Bluestein (chirp-z) for the largest prime radix > 40 whose convolution fits M <= 4096.  Its
    // butterflies run one at a time (two M-point FFTs each), so below ~40 the direct pass, which
    // is parallel over all n outputs, is cheaper (measured: radix 17 in 170 / 510, config 8)
    for (int i = 0; i < p.n; ++i)
        if (p.r[i] > 40 && p.r[i] > p.bp && next_pow2(2 * (int64_t)p.r[i] - 1) <= 4096) p.bp = p.r[i];
    if (p.bp) p.bM = (int)next_pow2(2 * (int64_t)p.bp - 1);
    return p;
}

// Bluestein tables for a radix-p pass of sign s (fp64): chirp, H^ = FFT_-(h)/M with
// h_n = conj c_n (n < p), h_{M-n} = conj c_n (0 < n < p), and the M-point roots.
// X_m = sum_j x_j e^{s 2 pi i j m / p} = c_m sum_j (x_j c_j) conj c_{m-j}  (jm = (j^2 + m^2 - (m-j)^2)/2).
template <typename T> void push_bluestein(std::vector<T> &blob, int p, int M, int s, size_t off[4]) {
    std::vector<cd> c(p), h(M, 0.0), H(M);
    for (int j = 0; j < p; ++j) {
        const int64_t e = ((int64_t)j * j) % (2 * p);
        c[j] = std::polar(1.0, s * PI * (double)e / p);
    }
    for (int n = 0; n < p; ++n) {
        h[n] = std::conj(c[n]);
        if (n) h[M - n] = std::conj(c[n]);
    }
    for (int k = 0; k < M; ++k) {
        cd acc = 0.0;
        for (int n = 0; n < M; ++n) acc += h[n] * std::polar(1.0, -2 * PI * (double)(((int64_t)n * k) % M) / M);
        H[k] = acc / (double)M;
    }
    off[0] = blob.size();
    for (int j = 0; j < p; ++j) push_c(blob, c[j]);
    off[1] = blob.size();
    for (int k = 0; k < M; ++k) push_c(blob, H[k]);
    off[2] = blob.size();
    push_roots(blob, M, M, 1, -1);
    off[3] = blob.size();
    push_roots(blob, M, M, 1, +1);
}

constexpr int64_t K1_DEFAULT = INT64_MIN;

template <typename T>
mci_status build_axis_any(mci::Axis1D &ax, int M, int64_t N, int64_t L, const mci_system *sys,
                          const int64_t *null_bins, int n_null, bool analytic, std::vector<T> &blob,
                          std::vector<size_t> &offs, double &cond_max, int64_t K1_in = K1_DEFAULT,
                          bool cplx = false) {
    if (M < 1 || M > 8 || !sys) return MCI_E_ARG;
    if (N < 2) return MCI_E_SIZE;
    const int64_t MN = (int64_t)M * N;
    if (MN < 2) return MCI_E_BAND;
    if (L < MN || L % N) return MCI_E_ALIAS;
    const int64_t K1 = K1_in == K1_DEFAULT ? -(MN / 2) : K1_in;
    for (int m = 0; m < M; ++m) {
        const mci_system &s = sys[m];
        if (s.kind < MCI_SYS_IDENTITY || s.kind > MCI_SYS_TABLE) return MCI_E_ARG;
        if (s.kind == MCI_SYS_DERIVATIVE && s.order < 0) return MCI_E_ARG;
        if (s.kind == MCI_SYS_TABLE) {
            if (!s.table) return MCI_E_ARG;
            for (int64_t k = 1; !cplx && -k >= K1 && k < K1 + MN; ++k) {  // Hermitian requirement (real output)
                cd a = sys_multiplier(s, K1, k), b = sys_multiplier(s, K1, -k);
                if (std::abs(a - std::conj(b)) > 1e-12 * (1 + std::abs(a))) return MCI_E_UNSUPPORTED;
            }
        }
    }
    ax.M = M; ax.N = N; ax.L = L; ax.K = -K1; ax.K1 = K1; ax.analytic = analytic ? 1 : 0;
    ax.cplx = cplx ? 1 : 0;
    for (int m = 0; m < M; ++m) {
        ax.sys[m].kind = sys[m].kind;
        ax.sys[m].order = sys[m].order;
        ax.sys[m].tau = sys[m].tau;
    }
    std::vector<double> omega(M, 0.0);
    ax.S = L; ax.R = 1;
    ax.radN = radix_plan(N);
    ax.radL = radix_plan(L);
    if (ax.radN.n > 23 || ax.radL.n > 23) return MCI_E_SIZE;
    offs.push_back(blob.size());  // Qt: every class
    std::vector<cd> H(M * M), inv;
    cond_max = 0.0;
    for (int64_t q = 0; q < N; ++q) {
        const int64_t jq = K1 + (((q - K1) % N) + N) % N;
        bool is_null = false;
        for (int z = 0; z < n_null; ++z)
            if (null_bins[z] == jq) is_null = true;
        double rowmax = 0.0;
        for (int l = 0; l < M; ++l)
            for (int m = 0; m < M; ++m) {
                H[l * M + m] = sys_multiplier(sys[m], K1, jq + (int64_t)l * N);
                rowmax = std::max(rowmax, std::abs(H[l * M + m]));
            }
        if (is_null) {
            inv.assign(M * M, 0.0);
        } else {
            if (!lu_inverse(M, H, inv, 1e-12 * rowmax)) {
                g_last_singular = jq;
                return MCI_E_SINGULAR;
            }
            double n1 = 0, n2 = 0;
            for (int c = 0; c < M; ++c) {
                double s1 = 0, s2 = 0;
                for (int r = 0; r < M; ++r) { s1 += std::abs(H[r * M + c]); s2 += std::abs(inv[r * M + c]); }
                n1 = std::max(n1, s1);
                n2 = std::max(n2, s2);
            }
            cond_max = std::max(cond_max, n1 * n2);
        }
        for (int m = 0; m < M; ++m)
            for (int l = 0; l < M; ++l) {
                push_c(blob, inv[m * M + l] / (double)N);
                omega[m] = std::max(omega[m], std::norm(inv[m * M + l]));  // |r_m(j_q + l N)|^2
            }
    }
    ax.omega_sum = 0;
    for (double o : omega) ax.omega_sum += o;
    offs.push_back(blob.size());  // twF = e^{-2 pi i m / N}
    push_roots(blob, N, N, 1, -1);
    offs.push_back(blob.size());  // twLhi = e^{+2 pi i m / L}
    push_roots(blob, L, L, 1, +1);
    ax.LO = L;  // (twLlo unused on this path)
    // Bluestein tables (offsets 3..6: forward N, 7..10: inverse L), resolved in set_ptrs_any
    size_t ob[4];
    if (ax.radN.bp) {
        push_bluestein(blob, ax.radN.bp, ax.radN.bM, -1, ob);
        for (size_t o : ob) offs.push_back(o);
    } else {
        for (int i = 0; i < 4; ++i) offs.push_back(0);
    }
    if (ax.radL.bp) {
        push_bluestein(blob, ax.radL.bp, ax.radL.bM, +1, ob);
        for (size_t o : ob) offs.push_back(o);
    } else {
        for (int i = 0; i < 4; ++i) offs.push_back(0);
    }
    ax.special = 4;
    return MCI_OK;
}

template <typename T>
mci_status upload(mci_plan p, std::vector<T> &blob) {
    void *d = nullptr;
    if (cudaMalloc(&d, blob.size() * sizeof(T)) != cudaSuccess) return MCI_E_CUDA;
    if (cudaMemcpy(d, blob.data(), blob.size() * sizeof(T), cudaMemcpyHostToDevice) != cudaSuccess) {
        cudaFree(d);
        return MCI_E_CUDA;
    }
    p->tables = d;
    return MCI_OK;
}

void set_ptrs(mci::Axis1D &ax, void *base, const std::vector<size_t> &offs, size_t elem) {
    char *b = (char *)base;
    ax.Qt = b + offs[0] * elem;
    ax.twF = b + offs[1] * elem;
    ax.twLhi = b + offs[2] * elem;
    ax.twLlo = b + (offs[2] + 2 * (ax.L / ax.LO)) * elem;
    if (ax.special == 4) {  // arbitrary-length path: Bluestein tables
        mci::AnyRadix *rp[2] = {&ax.radN, &ax.radL};
        for (int t = 0; t < 2; ++t) {
            if (!rp[t]->bp) continue;
            rp[t]->bc = b + offs[3 + 4 * t] * elem;
            rp[t]->bH = b + offs[4 + 4 * t] * elem;
            rp[t]->bwm = b + offs[5 + 4 * t] * elem;
            rp[t]->bwp = b + offs[6 + 4 * t] * elem;
        }
        ax.rowtab = nullptr;
        return;
    }
    ax.rowtab = offs.size() > 3 ? (const void *)(b + offs[3] * elem) : nullptr;
}

template <typename T>
mci_status create_1d(mci_plan p, int M, int64_t N, int64_t L, const mci_system *sys, const int64_t *null_bins,
                     int n_null, unsigned flags, int64_t K1 = K1_DEFAULT) {
    std::vector<T> blob;
    std::vector<size_t> offs;
    const bool analytic = flags & MCI_OUT_HILBERT;
    mci::Axis1D ax;
    ax.dtype = p->dtype;
    mci_status s;
    const bool cplx = flags & MCI_COMPLEX;
    if (cplx || use_anylen(M, N, L)) {  // arbitrary lengths / odd band / complex output
        s = build_axis_any<T>(ax, M, N, L, sys, null_bins, n_null, analytic, blob, offs, p->cond_max, K1, cplx);
        if (s != MCI_OK) return s;
        if (!mci::anylen_supported(ax)) return MCI_E_SIZE;
        p->path = mci::PATH_FUSED;
    } else {
        s = build_axis<T>(ax, M, N, L, sys, null_bins, n_null, analytic, false, blob, offs, p->cond_max);
        if (s != MCI_OK) return s;
        if (!mci::fused_supported(ax)) {
            blob.clear();
            offs.clear();
            s = build_axis<T>(ax, M, N, L, sys, null_bins, n_null, analytic, true, blob, offs, p->cond_max);
            if (s != MCI_OK) return s;
            if (!mci::fourstep_supported(ax)) return MCI_E_UNSUPPORTED;
            p->path = mci::PATH_FOURSTEP;
        }
    }
    // off-grid evaluator (NEXT-3): an arbitrary-length axis on the minimal grid L' = M N in the
    // plan's second axis slot (its inverse is never run; only the forward + solve tables are used)
    std::vector<T> blob2;
    std::vector<size_t> offs2;
    mci::Axis1D ay;
    ay.dtype = p->dtype;
    if (flags & (MCI_OFFGRID | MCI_ANALYSIS)) {
        if (flags & MCI_ANALYSIS)
            for (int m = 0; m < M; ++m)
                if (sys[m].kind == MCI_SYS_TABLE) return MCI_E_UNSUPPORTED;
        double c2 = 0;
        s = build_axis_any<T>(ay, M, N, (int64_t)M * N, sys, null_bins, n_null, analytic, blob2, offs2, c2);
        if (s != MCI_OK) return s;
        if (!mci::anylen_supported(ay)) return MCI_E_SIZE;
    }
    const size_t n1 = blob.size();
    blob.insert(blob.end(), blob2.begin(), blob2.end());
    if ((s = upload<T>(p, blob)) != MCI_OK) return s;
    set_ptrs(ax, p->tables, offs, sizeof(T));
    p->ax = ax;
    if (flags & (MCI_OFFGRID | MCI_ANALYSIS)) {
        set_ptrs(ay, (char *)p->tables + n1 * sizeof(T), offs2, sizeof(T));
        p->ay = ay;
    }
    if (p->path == mci::PATH_FOURSTEP) {
        // workspace for a chunk of signals.  Measured on B200 (config 4, 16 signals of
        // 20 MB intermediates): fewer, fuller launches beat L2 residency (96 MB: 0.491 ms,
        // 192 MB: 0.464 ms, 384 MB: 0.427 ms); 384 MB default (MCI_FS_WS_MB overrides)
        const size_t per = mci::fourstep_ws_bytes_per_signal(ax);
        const size_t ws_mb = getenv("MCI_FS_WS_MB") ? (size_t)atoi(getenv("MCI_FS_WS_MB")) : 384;
        int64_t units = std::max<int64_t>(1, (int64_t)((ws_mb << 20) / per));
        p->ws_units = units;
        p->ws_bytes = per * units;
        if (cudaMalloc(&p->ws, p->ws_bytes) != cudaSuccess) return MCI_E_CUDA;
        // unimodular bank: the channel-magnitude words stay 0 (no scaling), written once here
        if (ax.bank_unimodular && cudaMemset(p->ws, 0, p->ws_bytes) != cudaSuccess) return MCI_E_CUDA;
    }
    return MCI_OK;
}

template <typename T>
mci_status create_2d(mci_plan p, int Mx, int64_t Nx, const mci_system *sx, int My, int64_t Ny,
                     const mci_system *sy, int scale) {
    std::vector<T> bx, by;
    std::vector<size_t> ox, oy;
    double cx = 0, cy = 0;
    mci::Axis1D ax, ay;
    ax.dtype = ay.dtype = p->dtype;
    auto axis = [&](mci::Axis1D &a, int M, int64_t N, const mci_system *sy_, std::vector<T> &b, std::vector<size_t> &o,
                    double &c) -> mci_status {
        const int64_t L = (int64_t)scale * N;
        if (use_anylen(M, N, L)) {
            mci_status st = build_axis_any<T>(a, M, N, L, sy_, nullptr, 0, false, b, o, c);
            if (st == MCI_OK && !mci::anylen_supported(a)) st = MCI_E_SIZE;
            return st;
        }
        mci_status st = build_axis<T>(a, M, N, L, sy_, nullptr, 0, false, false, b, o, c);
        if (st == MCI_OK && !mci::fused_supported(a)) st = MCI_E_UNSUPPORTED;
        return st;
    };
    mci_status s = axis(ax, Mx, Nx, sx, bx, ox, cx);
    if (s != MCI_OK) return s;
    s = axis(ay, My, Ny, sy, by, oy, cy);
    if (s != MCI_OK) return s;
    p->cond_max = std::max(cx, cy);
    const size_t nx = bx.size();
    bx.insert(bx.end(), by.begin(), by.end());
    if ((s = upload<T>(p, bx)) != MCI_OK) return s;
    set_ptrs(ax, p->tables, ox, sizeof(T));
    set_ptrs(ay, (char *)p->tables + nx * sizeof(T), oy, sizeof(T));
    p->ax = ax;
    p->ay = ay;
    p->Mx = Mx; p->My = My; p->Nx = Nx; p->Ny = Ny; p->Lx = ax.L; p->Ly = ay.L;
    p->path = mci::PATH_2D;
    // intermediate per image: column-first Mx Nx Ly, row-first (line kernels) My Ny Lx
    const size_t per = (size_t)std::max<int64_t>((int64_t)Mx * Nx * ay.L, (int64_t)My * Ny * ax.L) * sizeof(T);
    // images per chunk: measured on B200 (config 5), fewer and fuller launches beat L2
    // residency of the intermediate (first kernels: 32 MB 1.35 ms, 256 MB 1.12 ms, 512 MB
    // 1.10 ms per 64 images; current kernels: 32 MB 1.05 ms, 128 MB 0.79 ms, 256 MB 0.735 ms,
    // 512 MB 0.706 ms); 512 MB is the default footprint (MCI_2D_WS_MB overrides)
    const size_t ws_mb = getenv("MCI_2D_WS_MB") ? (size_t)atoi(getenv("MCI_2D_WS_MB")) : 512;
    int64_t units = std::max<int64_t>(1, (int64_t)((ws_mb << 20) / per));
    p->ws_units = units;
    p->ws_halves = (getenv("MCI_2D_STREAMS") && atoi(getenv("MCI_2D_STREAMS")) == 2) ? 2 : 1;
    p->ws_bytes = per * units * p->ws_halves;
    if (cudaMalloc(&p->ws, p->ws_bytes) != cudaSuccess) return MCI_E_CUDA;
    return MCI_OK;
}

mci_status from_cuda(cudaError_t e) {
    if (e != cudaSuccess && getenv("MCI_DEBUG")) fprintf(stderr, "mci: CUDA error: %s\n", cudaGetErrorString(e));
    return e == cudaSuccess ? MCI_OK : MCI_E_CUDA;
}

mci_status exec_1d(mci_plan p, int64_t batch, const void *g, void *f, void *hf, cudaStream_t st, int *nl) {
    if (p->path == mci::PATH_FUSED) {
        mci::RowAddr ra;
        ra.s2 = (int64_t)p->ax.M * p->ax.N;
        ra.cs = p->ax.N;
        ra.ss = 1;
        return from_cuda(mci::launch_axis(p->ax, ra, batch, g, f, hf, st, nl));
    }
    return from_cuda(mci::launch_fourstep(p->ax, batch, g, f, p->ws, p->ws_units, st, nl));
}

mci_status exec_2d(mci_plan p, int64_t n, const void *g, void *out, cudaStream_t st, int *nl) {
    const size_t es = esize(p->dtype);
    const int64_t Mx = p->Mx, My = p->My, Nx = p->Nx, Ny = p->Ny, Lx = p->Lx, Ly = p->Ly;
    const int64_t in_img = My * Mx * Ny * Nx, out_img = Ly * Lx;
    // two workspace halves: chunk c runs on stream c & 1 (the caller's stream or s2), so one
    // chunk's row pass overlaps the next chunk's column pass; s2 joins the caller's stream
    const bool two = p->ws_halves == 2 && n > p->ws_units;
    cudaStream_t st0 = st;
    if (two) {
        if (!p->s2 && cudaStreamCreateWithFlags(&p->s2, cudaStreamNonBlocking) != cudaSuccess) return MCI_E_CUDA;
        for (int k = 0; k < 2; ++k)
            if (!p->ev[k] && cudaEventCreateWithFlags(&p->ev[k], cudaEventDisableTiming) != cudaSuccess)
                return MCI_E_CUDA;
        if (cudaEventRecord(p->ev[0], st0) != cudaSuccess || cudaStreamWaitEvent(p->s2, p->ev[0], 0) != cudaSuccess)
            return MCI_E_CUDA;
    }
    const size_t half_bytes = p->ws_bytes / p->ws_halves;
    int64_t chunk_id = 0;
    for (int64_t i0 = 0; i0 < n; i0 += p->ws_units) {
        const int64_t ni = std::min<int64_t>(p->ws_units, n - i0);
        cudaStream_t sc = (two && (chunk_id & 1)) ? p->s2 : st0;
        void *wsc = (char *)p->ws + (two ? (size_t)(chunk_id & 1) * half_bytes : 0);
        ++chunk_id;
        const char *gi = (const char *)g + i0 * in_img * es;
        char *oi = (char *)out + i0 * out_img * es;
        if (p->ay.special == 2 && p->ax.special == 2) {
            // Line kernels on both axes: row pass first, on contiguous input lines (img, my, ny),
            // storing ws[img][my][px][ny] transposed; the column pass then reads contiguous
            // lines (img, px) and stores out[img][py][px] transposed.  Both passes prefetch
            // whole lines (16-byte cp.async) instead of gathering strided samples.  The
            // separable result is order-independent (Re after each pass).
            mci::RowAddr ra1;  // row pass on g: channels mx, samples nx
            ra1.D0 = Ny; ra1.D1 = My; ra1.s0 = Nx; ra1.s1 = Mx * Ny * Nx; ra1.s2 = My * Mx * Ny * Nx;
            ra1.cs = Ny * Nx; ra1.ss = 1;
            mci::RowAddr ra2;  // column pass on ws: channels my, samples ny
            ra2.D0 = Lx; ra2.D1 = 1; ra2.s0 = Ny; ra2.s1 = 0; ra2.s2 = My * Lx * Ny;
            ra2.cs = Lx * Ny; ra2.ss = 1;
            // opt-in (MCI_2D_ORDER=1): measured slower than column-first on config 5 (0.99 vs
            // 0.81 ms per 64 images): the untiled transposed-store passes issue at ~31 %
            const bool order_rows = getenv("MCI_2D_ORDER") && atoi(getenv("MCI_2D_ORDER")) == 1 &&
                                    mci::line_tstore_ok(p->ax, ra1, ni * My * Ny, gi, wsc) &&
                                    mci::line_tstore_ok(p->ay, ra2, ni * Lx, wsc, oi);
            if (order_rows) {
                if (mci::launch_line(p->ax, ra1, ni * My * Ny, gi, wsc, sc, nl, true) != cudaSuccess ||
                    mci::launch_line(p->ay, ra2, ni * Lx, wsc, oi, sc, nl, true) != cudaSuccess)
                    return MCI_E_CUDA;
                continue;
            }
        }
        // column pass (along y, channels my) on the input -> ws[img][mx][nx][Ly]
        mci::RowAddr rc;
        rc.D0 = Nx; rc.D1 = Mx; rc.s0 = 1; rc.s1 = Ny * Nx; rc.s2 = My * Mx * Ny * Nx;
        rc.cs = Mx * Ny * Nx; rc.ss = Nx;
        // line kernels on both axes: the column pass stores ws transposed, ws[img][mx][py][nx],
        // so the row pass reads contiguous lines (measured: 0.33 -> 0.25 ms per 65,536 lines)
        const bool tws = p->ay.special == 2 && p->ax.special == 2 &&
                         mci::line_tstore_ok(p->ay, rc, ni * Mx * Nx, gi, wsc);
        cudaError_t e = tws ? mci::launch_line(p->ay, rc, ni * Mx * Nx, gi, wsc, sc, nl, true)
                            : mci::launch_axis(p->ay, rc, ni * Mx * Nx, gi, wsc, nullptr, sc, nl);
        if (e != cudaSuccess) return MCI_E_CUDA;
        // row pass (along x, channels mx) on ws -> out[img][py][Lx]
        mci::RowAddr rr;
        if (tws) {  // ws[img][mx][py][nx]: line py, channel stride Ly Nx, samples contiguous
            rr.D0 = Ly; rr.D1 = 1; rr.s0 = Nx; rr.s1 = 0; rr.s2 = Mx * Ly * Nx;
            rr.cs = Ly * Nx; rr.ss = 1;
        } else {  // ws[img][mx][nx][py]: samples strided by Ly
            rr.D0 = Ly; rr.D1 = 1; rr.s0 = 1; rr.s1 = 0; rr.s2 = Mx * Nx * Ly;
            rr.cs = Nx * Ly; rr.ss = Ly;
        }
        e = mci::launch_axis(p->ax, rr, ni * Ly, wsc, oi, nullptr, sc, nl);
        if (e != cudaSuccess) return MCI_E_CUDA;
    }
    if (two && (cudaEventRecord(p->ev[1], p->s2) != cudaSuccess || cudaStreamWaitEvent(st0, p->ev[1], 0) != cudaSuccess))
        return MCI_E_CUDA;
    return MCI_OK;
}

}  // namespace

namespace mci {
cudaError_t launch_axis(const Axis1D &ax, const RowAddr &ra, int64_t rows, const void *g, void *f, void *hf,
                        cudaStream_t st, int *nl) {
    if (ax.special == 4) return launch_anylen(ax, ra, rows, g, f, hf, st, nl);
    const bool dense = ra.D0 == 1 && ra.D1 == 1 && ra.ss == 1 && ra.cs == ax.N && ra.s2 == ax.M * ax.N;
    const bool al = aligned16(g) && aligned16(f) && (!hf || aligned16(hf));
    if (ax.special == 1 && dense && al)
        return ax.rowg ? launch_rowg(ax, rows, g, f, st, nl) : launch_row(ax, ax.rowtab, rows, g, f, st, nl);
    if (ax.special == 2) return launch_line(ax, ra, rows, g, f, st, nl);  // checks its own alignment
    if (ax.special == 3 && dense && al) return launch_hilbert(ax, rows, g, f, hf, st, nl);
    return launch_fused(ax, ra, rows, g, f, hf, st, nl);
}
}  // namespace mci

namespace {
// SISR plan (NEXT-2): two Example-2 axes (f, f', f'') on the W and H grids, scale s.
template <typename T>
mci_status create_sisr(mci_plan p, int64_t H, int64_t W, int s) {
    static const mci_system bank[3] = {{MCI_SYS_IDENTITY, 0, 0.0, nullptr},
                                       {MCI_SYS_DERIVATIVE, 1, 0.0, nullptr},
                                       {MCI_SYS_DERIVATIVE, 2, 0.0, nullptr}};
    std::vector<T> bx, by;
    std::vector<size_t> ox, oy;
    double cx = 0, cy = 0;
    mci::Axis1D ax, ay;
    ax.dtype = ay.dtype = p->dtype;
    auto axis = [&](mci::Axis1D &a, int64_t N, std::vector<T> &b, std::vector<size_t> &o, double &c) -> mci_status {
        const int64_t L = (int64_t)s * N;
        if (use_anylen(3, N, L)) {
            mci_status st = build_axis_any<T>(a, 3, N, L, bank, nullptr, 0, false, b, o, c);
            if (st == MCI_OK && !mci::anylen_supported(a)) st = MCI_E_SIZE;
            return st;
        }
        mci_status st = build_axis<T>(a, 3, N, L, bank, nullptr, 0, false, false, b, o, c);
        if (st == MCI_OK && !mci::fused_supported(a)) st = MCI_E_UNSUPPORTED;
        return st;
    };
    mci_status st = axis(ax, W, bx, ox, cx);
    if (st != MCI_OK) return st;
    st = axis(ay, H, by, oy, cy);
    if (st != MCI_OK) return st;
    p->cond_max = std::max(cx, cy);
    const size_t nx = bx.size();
    bx.insert(bx.end(), by.begin(), by.end());
    if ((st = upload<T>(p, bx)) != MCI_OK) return st;
    set_ptrs(ax, p->tables, ox, sizeof(T));
    set_ptrs(ay, (char *)p->tables + nx * sizeof(T), oy, sizeof(T));
    p->ax = ax;
    p->ay = ay;
    p->Mx = p->My = 3;
    p->Nx = W; p->Ny = H; p->Lx = s * W; p->Ly = s * H;
    p->path = mci::PATH_SISR;
    const size_t per = mci::sisr_ws_per_image((int)H, (int)W, s, p->dtype);
    const size_t ws_mb = getenv("MCI_2D_WS_MB") ? (size_t)atoi(getenv("MCI_2D_WS_MB")) : 256;
    p->ws_units = std::max<int64_t>(1, (int64_t)((ws_mb << 20) / per));
    p->ws_bytes = per * p->ws_units;
    if (cudaMalloc(&p->ws, p->ws_bytes) != cudaSuccess) return MCI_E_CUDA;
    return MCI_OK;
}

}  // namespace

extern "C" {

mci_status mci_plan_create_band(mci_plan *out, int M, int64_t N, int64_t L, int64_t K1, const mci_system *sys,
                                const int64_t *null_bins, int n_null, mci_dtype dtype, unsigned flags) {
    if (!out) return MCI_E_ARG;
    *out = nullptr;
    if ((dtype != MCI_F32 && dtype != MCI_F64) || (flags & ~(MCI_OUT_HILBERT | MCI_OFFGRID | MCI_COMPLEX | MCI_ANALYSIS)) ||
        n_null < 0 || (n_null > 0 && !null_bins))
        return MCI_E_ARG;
    if ((flags & MCI_COMPLEX) && (flags & (MCI_OUT_HILBERT | MCI_OFFGRID | MCI_ANALYSIS))) return MCI_E_UNSUPPORTED;
    // real output: the Hermitian assembly of the paths needs the default band
    if (!(flags & MCI_COMPLEX) && K1 != K1_DEFAULT && K1 != -(((int64_t)M * N) / 2)) return MCI_E_UNSUPPORTED;
    mci_plan p = new (std::nothrow) mci_plan_s();
    if (!p) return MCI_E_ARG;
    p->dtype = dtype;
    p->flags = flags;
    mci_status s = dtype == MCI_F64 ? create_1d<double>(p, M, N, L, sys, null_bins, n_null, flags, K1)
                                    : create_1d<float>(p, M, N, L, sys, null_bins, n_null, flags, K1);
    if (s != MCI_OK) {
        mci_plan_destroy(p);
        return s;
    }
    *out = p;
    return MCI_OK;
}

mci_status mci_plan_create(mci_plan *out, int M, int64_t N, int64_t L, const mci_system *sys,
                           const int64_t *null_bins, int n_null, mci_dtype dtype, unsigned flags) {
    if (!out) return MCI_E_ARG;
    *out = nullptr;
    if ((dtype != MCI_F32 && dtype != MCI_F64) || (flags & ~(MCI_OUT_HILBERT | MCI_OFFGRID | MCI_COMPLEX | MCI_ANALYSIS)) ||
        n_null < 0 || (n_null > 0 && !null_bins))
        return MCI_E_ARG;
    if ((flags & MCI_COMPLEX) && (flags & (MCI_OUT_HILBERT | MCI_OFFGRID | MCI_ANALYSIS))) return MCI_E_UNSUPPORTED;
    mci_plan p = new (std::nothrow) mci_plan_s();
    if (!p) return MCI_E_ARG;
    p->dtype = dtype;
    p->flags = flags;
    mci_status s = dtype == MCI_F64 ? create_1d<double>(p, M, N, L, sys, null_bins, n_null, flags)
                                    : create_1d<float>(p, M, N, L, sys, null_bins, n_null, flags);
    if (s != MCI_OK) {
        mci_plan_destroy(p);
        return s;
    }
    *out = p;
    return MCI_OK;
}

mci_status mci_plan_create_sisr(mci_plan *out, int64_t H, int64_t W, int scale, mci_dtype dtype) {
    if (!out) return MCI_E_ARG;
    *out = nullptr;
    if ((dtype != MCI_F32 && dtype != MCI_F64) || scale < 3 || H < 2 || W < 2 || H > (1 << 20) || W > (1 << 20))
        return MCI_E_ARG;
    mci_plan p = new (std::nothrow) mci_plan_s();
    if (!p) return MCI_E_ARG;
    p->dtype = dtype;
    mci_status s = dtype == MCI_F64 ? create_sisr<double>(p, H, W, scale) : create_sisr<float>(p, H, W, scale);
    if (s != MCI_OK) {
        mci_plan_destroy(p);
        return s;
    }
    *out = p;
    return MCI_OK;
}

mci_status mci_execute_sisr(mci_plan p, int64_t n_images, const void *lr, void *hr, void *stream) {
    if (!p || p->path != mci::PATH_SISR || n_images < 0) return MCI_E_ARG;
    if (n_images == 0) return MCI_OK;
    if (!lr || !hr) return MCI_E_ARG;
    const size_t es = esize(p->dtype);
    const int H = (int)p->Ny, W = (int)p->Nx, s = (int)(p->Lx / p->Nx);
    return with_workspace(p, (cudaStream_t)stream, [&](cudaStream_t st) {
        for (int64_t i0 = 0; i0 < n_images; i0 += p->ws_units) {
            const int64_t ni = std::min<int64_t>(p->ws_units, n_images - i0);
            cudaError_t e = mci::launch_sisr_chunk(p->ax, p->ay, ni, H, W, s,
                                                   (const char *)lr + i0 * (int64_t)H * W * es,
                                                   (char *)hr + i0 * (int64_t)s * H * s * W * es, p->ws, st, nullptr);
            if (e != cudaSuccess) return MCI_E_CUDA;
        }
        return MCI_OK;
    });
}

mci_status mci_plan_create_2d(mci_plan *out, int Mx, int64_t Nx, const mci_system *sx, int My, int64_t Ny,
                              const mci_system *sy, int scale, mci_dtype dtype, unsigned flags) {
    if (!out) return MCI_E_ARG;
    *out = nullptr;
    if ((dtype != MCI_F32 && dtype != MCI_F64) || flags != 0 || scale < 1) return MCI_E_ARG;
    mci_plan p = new (std::nothrow) mci_plan_s();
    if (!p) return MCI_E_ARG;
    p->dtype = dtype;
    mci_status s = dtype == MCI_F64 ? create_2d<double>(p, Mx, Nx, sx, My, Ny, sy, scale)
                                    : create_2d<float>(p, Mx, Nx, sx, My, Ny, sy, scale);
    if (s != MCI_OK) {
        mci_plan_destroy(p);
        return s;
    }
    *out = p;
    return MCI_OK;
}

void mci_plan_destroy(mci_plan p) {
    if (!p) return;
    if (p->ws_ev) cudaEventDestroy(p->ws_ev);
    for (int i = 0; i < 2; ++i)
        if (p->hs[i]) cudaStreamDestroy(p->hs[i]);
    if (p->s2) cudaStreamDestroy(p->s2);
    for (int i = 0; i < 2; ++i)
        if (p->ev[i]) cudaEventDestroy(p->ev[i]);
    for (int i = 0; i < 4; ++i)
        if (p->stage[i]) cudaFree(p->stage[i]);
    if (p->ws) cudaFree(p->ws);
    if (p->tables) cudaFree(p->tables);
    delete p;
}

// the 1D entry points serve 1D plans only: a 2D or SISR plan has neither the 1D axis nor the
// workspace layout exec_1d would launch on
static bool is_1d(mci_plan p) { return p && (p->path == mci::PATH_FUSED || p->path == mci::PATH_FOURSTEP); }

mci_status mci_execute_1d(mci_plan p, int64_t batch, const void *g, void *f, void *hf, void *stream) {
    if (!is_1d(p) || batch < 0) return MCI_E_ARG;
    if (batch == 0) return MCI_OK;
    if (!g || !f) return MCI_E_ARG;
    if ((p->flags & MCI_OUT_HILBERT) ? !hf : (hf != nullptr)) return MCI_E_ARG;
    return with_workspace(p, (cudaStream_t)stream,
                          [&](cudaStream_t st) { return exec_1d(p, batch, g, f, hf, st, nullptr); });
}

mci_status mci_execute_offgrid(mci_plan p, int64_t batch, const void *g, int64_t n_pts, const void *t, void *f,
                               void *hf, void *stream) {
    if (!is_1d(p) || !(p->flags & MCI_OFFGRID) || p->ay.special != 4 || batch < 0 ||
        n_pts < 0 || n_pts > INT32_MAX)
        return MCI_E_ARG;
    if (batch == 0 || n_pts == 0) return MCI_OK;
    if (!g || !t || !f) return MCI_E_ARG;
    if ((p->flags & MCI_OUT_HILBERT) ? !hf : (hf != nullptr)) return MCI_E_ARG;
    mci::RowAddr ra;
    ra.s2 = (int64_t)p->ax.M * p->ax.N;
    ra.cs = p->ax.N;
    ra.ss = 1;
    return from_cuda(mci::launch_anylen_offgrid(p->ay, ra, batch, g, n_pts, t, f, hf, (cudaStream_t)stream));
}

mci_status mci_consistency_residual(mci_plan p, int64_t batch, const void *g, void *out, void *stream) {
    if (!is_1d(p) || !(p->flags & MCI_ANALYSIS) ||
        p->ay.special != 4 || batch < 0)
        return MCI_E_ARG;
    if (batch == 0) return MCI_OK;
    if (!g || !out) return MCI_E_ARG;
    mci::RowAddr ra;
    ra.s2 = (int64_t)p->ay.M * p->ay.N;
    ra.cs = p->ay.N;
    ra.ss = 1;
    return from_cuda(mci::launch_anylen_residual(p->ay, ra, batch, g, out, (cudaStream_t)stream));
}

mci_status mci_averaged_error(mci_plan p, int64_t batch, const void *spec, int64_t k_lo, int64_t n_freq, void *out,
                              void *stream) {
    if (!is_1d(p) || !(p->flags & MCI_ANALYSIS) ||
        p->ay.special != 4 || batch < 0 || n_freq < 0 || n_freq > INT32_MAX)
        return MCI_E_ARG;
    if (batch == 0) return MCI_OK;
    if (!spec || !out) return MCI_E_ARG;
    return from_cuda(mci::launch_averaged_error(p->ay, batch, spec, k_lo, n_freq, out, (cudaStream_t)stream));
}

mci_status mci_execute_2d(mci_plan p, int64_t n_images, const void *g, void *out, void *stream) {
    if (!p || p->path != mci::PATH_2D || n_images < 0) return MCI_E_ARG;
    if (n_images == 0) return MCI_OK;
    if (!g || !out) return MCI_E_ARG;
    return with_workspace(p, (cudaStream_t)stream,
                          [&](cudaStream_t st) { return exec_2d(p, n_images, g, out, st, nullptr); });
}

// Host-buffer execution: two streams ping-pong over chunks (H2D, compute, D2H).
static mci_status exec_host(mci_plan p, int64_t units, const void *g, void *f, void *hf) {
    const size_t es = esize(p->dtype);
    size_t in_u, out_u;
    int nout = 1;
    if (p->path == mci::PATH_2D) {
        in_u = (size_t)p->My * p->Mx * p->Ny * p->Nx * es;
        out_u = (size_t)p->Ly * p->Lx * es;
    } else {
        const size_t cf = (p->flags & MCI_COMPLEX) ? 2 : 1;  // complex: two scalars per value
        in_u = (size_t)p->ax.M * p->ax.N * es * cf;
        out_u = (size_t)p->ax.L * es * cf;
        nout = (p->flags & MCI_OUT_HILBERT) ? 2 : 1;
    }
    int64_t chunk = std::max<int64_t>(1, (int64_t)((64u << 20) / (out_u * nout)));
    // 2D: 256 MB of output per chunk (16 config-5 images), so the copies of neighbouring
    // chunks overlap (exec_2d splits a chunk by the workspace size itself)
    if (p->path == mci::PATH_2D)
        chunk = std::min<int64_t>(p->ws_units, std::max<int64_t>(1, (int64_t)((256u << 20) / (out_u * nout))));
    if (p->path == mci::PATH_FOURSTEP) chunk = std::max<int64_t>(chunk, p->ws_units);
    chunk = std::min(chunk, units);
    if (p->stage_rows < chunk) {
        for (int i = 0; i < 4; ++i)
            if (p->stage[i]) { cudaFree(p->stage[i]); p->stage[i] = nullptr; }
        for (int b = 0; b < 2; ++b) {
            if (cudaMalloc(&p->stage[2 * b], in_u * chunk) != cudaSuccess) return MCI_E_CUDA;
            if (cudaMalloc(&p->stage[2 * b + 1], out_u * nout * chunk) != cudaSuccess) return MCI_E_CUDA;
        }
        p->stage_rows = chunk;
    }
    for (int b = 0; b < 2; ++b)
        if (!p->hs[b] && cudaStreamCreateWithFlags(&p->hs[b], cudaStreamNonBlocking) != cudaSuccess) return MCI_E_CUDA;
    // Chunk i on stream i&1: H2D_i, [wait compute_{i-1} if the plan has a
    // shared workspace], compute_i, record, D2H_i.  Copies of one chunk overlap
    // compute of the neighbouring chunk.
    cudaEvent_t done[2];
    for (int b = 0; b < 2; ++b)
        if (cudaEventCreateWithFlags(&done[b], cudaEventDisableTiming) != cudaSuccess) return MCI_E_CUDA;
    mci_status s = MCI_OK;
    int it = 0;
    for (int64_t u0 = 0; u0 < units && s == MCI_OK; u0 += chunk, ++it) {
        const int64_t n = std::min(chunk, units - u0);
        const int b = it & 1;
        cudaStream_t st = p->hs[b];
        char *din = (char *)p->stage[2 * b], *dout = (char *)p->stage[2 * b + 1];
        if (cudaMemcpyAsync(din, (const char *)g + u0 * in_u, n * in_u, cudaMemcpyHostToDevice, st) != cudaSuccess) {
            s = MCI_E_CUDA;
            break;
        }
        if (p->ws && it > 0) cudaStreamWaitEvent(st, done[b ^ 1], 0);
        // the first chunk also waits for the workspace use of earlier device-buffer executions
        if (p->ws && it == 0 && p->ws_ev_recorded) cudaStreamWaitEvent(st, p->ws_ev, 0);
        if (p->path == mci::PATH_2D) s = exec_2d(p, n, din, dout, st, nullptr);
        else s = exec_1d(p, n, din, dout, nout == 2 ? dout + n * out_u : nullptr, st, nullptr);
        if (s != MCI_OK) break;
        cudaEventRecord(done[b], st);
        if (cudaMemcpyAsync((char *)f + u0 * out_u, dout, n * out_u, cudaMemcpyDeviceToHost, st) != cudaSuccess)
            s = MCI_E_CUDA;
        else if (nout == 2 && cudaMemcpyAsync((char *)hf + u0 * out_u, dout + n * out_u, n * out_u,
                                               cudaMemcpyDeviceToHost, st) != cudaSuccess)
            s = MCI_E_CUDA;
    }
    for (int b = 0; b < 2; ++b)
        if (cudaStreamSynchronize(p->hs[b]) != cudaSuccess) s = MCI_E_CUDA;
    for (int b = 0; b < 2; ++b) cudaEventDestroy(done[b]);
    return s;
}

mci_status mci_execute_1d_host(mci_plan p, int64_t batch, const void *g, void *f, void *hf) {
    if (!is_1d(p) || batch < 0) return MCI_E_ARG;
    if (batch == 0) return MCI_OK;
    if (!g || !f) return MCI_E_ARG;
    if ((p->flags & MCI_OUT_HILBERT) ? !hf : (hf != nullptr)) return MCI_E_ARG;
    std::lock_guard<std::mutex> lock(p->mu);  // staging buffers and streams of the plan
    return exec_host(p, batch, g, f, hf);
}

mci_status mci_execute_2d_host(mci_plan p, int64_t n_images, const void *g, void *out) {
    if (!p || p->path != mci::PATH_2D || n_images < 0) return MCI_E_ARG;
    if (n_images == 0) return MCI_OK;
    if (!g || !out) return MCI_E_ARG;
    std::lock_guard<std::mutex> lock(p->mu);  // staging buffers and streams of the plan
    return exec_host(p, n_images, g, out, nullptr);
}

double mci_plan_cond_max(mci_plan p) { return p ? p->cond_max : 0.0; }
int64_t mci_last_singular_bin(void) { return g_last_singular; }
size_t mci_plan_workspace_bytes(mci_plan p) { return p ? p->ws_bytes : 0; }
int mci_plan_path(mci_plan p) { return p ? p->path : -1; }

int64_t mci_plan_launches(mci_plan p, int64_t batch) {
    if (!p || batch <= 0) return 0;
    if (p->path == mci::PATH_FUSED) return 1;
    const int64_t chunks = (batch + p->ws_units - 1) / p->ws_units;
    if (p->path == mci::PATH_SISR) return 5 * chunks;  // fd rows, MCI x, fd cols, MCI y, transpose
    return p->path == mci::PATH_FOURSTEP ? (p->ax.bank_unimodular ? 3 : 4) * chunks : 2 * chunks;
}

const char *mci_status_str(mci_status s) {
    switch (s) {
    case MCI_OK: return "ok";
    case MCI_E_ARG: return "invalid argument";
    case MCI_E_BAND: return "invalid band (M*N < 2)";
    case MCI_E_ALIAS: return "L must be >= M*N and a multiple of N";
    case MCI_E_SINGULAR: return "system matrix H_n singular (see mci_last_singular_bin)";
    case MCI_E_SIZE: return "unsupported size (N < 2, or too large for the arbitrary-length path)";
    case MCI_E_CUDA: return "CUDA error";
    case MCI_E_UNSUPPORTED: return "unsupported configuration";
    }
    return "unknown status";
}

const char *mci_version(void) { return "mci-b200 0.1 (sm_100a)"; }

}  // extern "C"
