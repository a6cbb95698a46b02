// Four-step MCI path for lengths beyond one CTA's shared memory (config 4:
// N = 262144, L = 4194304).  Same mathematics as the fused kernel
// (Lemma 1 forward DFT, per-class solve Eq. matrixeqn1, Hermitian-part
// assembly, pruned inverse of Eq. DFTexpression), split into three kernels
// around HBM/L2-resident intermediates:
//
//   FA  forward step 1: length-N1 DFTs over n1 (input stride N2) for every
//       residue n2, twiddle e^{-2 pi i n2 q1/N}            -> T[c][q1][n2]
//   FB  forward step 2 for the residue pair {q1, N1-q1}: length-N2 DFTs give
//       G[q1 + N1 q2]; per-class solve; assembly X[p], p = +-q1 mod N1;
//       pre-twiddle e^{2 pi i k p1/L}; inverse step 1: length-S2 DFTs over
//       k1 of Zin[k2 + N1 k1] (k2 in the pair), twiddle e^{2 pi i k2 u/S}
//                                                            -> U[ip][k2][u]
//   IC  inverse step 2: length-N1 DFTs over k2 for a tile of u, giving
//       y[u + S2 v] = f[R p2 + p1] for p2 = u + S2 v       -> f (coalesced runs)
//
// Residues mod N1 line up because N1 divides N and S: class q = k mod N and
// FFT index k' = k mod S share k mod N1, so one FB CTA owns everything a
// residue pair needs (including the mirror classes for real-signal unpacking).
#include <algorithm>
#include <cstdlib>
#include <type_traits>

#include "mci_fourstep.cuh"

namespace mci {

// ---- channel magnitude pre-pass (exact power-of-two scaling before channel packing) ----------
static constexpr int MX_NT = 256, MX_BLK = 16;

template <typename T>
__global__ void __launch_bounds__(MX_NT) mci_fs_max(const FSArgs<T> a) {
    const int blk = blockIdx.x % MX_BLK;
    const int m = (blockIdx.x / MX_BLK) % a.M;
    const int64_t sl = blockIdx.x / ((int64_t)MX_BLK * a.M);
    const T *g0 = a.g + ((a.sig0 + sl) * a.M + m) * a.N;
    T v = 0;
    for (int64_t n = (int64_t)blk * MX_NT + threadIdx.x; n < a.N; n += (int64_t)MX_BLK * MX_NT) v = fmax(v, fabs(__ldg(g0 + n)));
    __shared__ T red[MX_NT / 32];
    v = block_max<MX_NT>(v, red);
    if (threadIdx.x == 0) {
        if constexpr (sizeof(T) == 4) atomicMax(a.cmax + sl * a.M + m, __float_as_uint(v));
        else atomicMax(a.cmax + sl * a.M + m, (unsigned long long)__double_as_longlong(v));
    }
}

// ---- FA ------------------------------------------------------------------------------------
static constexpr int FA_TN2 = 8, FA_NT = 256;

template <typename T, int TN2>
__global__ void __launch_bounds__(FA_NT) mci_fs_fa(const FSArgs<T> a) {
    using V = cv<T>;
    extern __shared__ __align__(16) unsigned char smem_raw[];
    V *buf = reinterpret_cast<V *>(smem_raw);  // [FA_TN2][N1]
    const int ntiles = (int)(a.N2 / TN2);
    const int tile = blockIdx.x % ntiles;
    const int c = (blockIdx.x / ntiles) % a.npair;
    const int64_t sl = blockIdx.x / ((int64_t)ntiles * a.npair);  // signal within chunk
    const T *g0 = a.g + (a.sig0 + sl) * (int64_t)a.M * a.N;
    const int e0 = chan_exp(a, sl, 2 * c), e1 = chan_exp(a, sl, 2 * c + 1);
    for (int idx = threadIdx.x; idx < TN2 * N1; idx += FA_NT) {
        const int n1 = idx / TN2, t = idx % TN2;
        const int64_t n = (int64_t)n1 * a.N2 + tile * TN2 + t;
        T re = __ldg(g0 + (int64_t)(2 * c) * a.N + n);
        T im = (2 * c + 1 < a.M) ? __ldg(g0 + (int64_t)(2 * c + 1) * a.N + n) : T(0);
        buf[t * N1 + n1] = V{ldexp(re, -e0), ldexp(im, -e1)};
    }
    __syncthreads();
    block_fft_ct<T, N1, 1, -1, FA_NT, TN2>(buf, N1, a.twF, a.TW);
    V *out = a.Tw + (sl * a.npair + c) * (int64_t)N1 * a.N2;
    for (int idx = threadIdx.x; idx < TN2 * N1; idx += FA_NT) {
        const int q1 = idx / TN2, t = idx % TN2;
        const int64_t n2 = (int64_t)tile * TN2 + t;
        out[(int64_t)q1 * a.N2 + n2] = cmul(buf[t * N1 + q1], a.twN(n2 * q1));
    }
}

// ---- FB ------------------------------------------------------------------------------------
static constexpr int FB_NT = 256;

template <typename T>
__global__ void __launch_bounds__(FB_NT) mci_fs_fb(const FSArgs<T> a) {
    using V = cv<T>;
    extern __shared__ __align__(16) unsigned char smem_raw[];
    const int q1 = blockIdx.x % (N1 / 2 + 1);
    const int64_t sl = blockIdx.x / (N1 / 2 + 1);
    const int nres = (q1 == 0 || q1 == N1 / 2) ? 1 : 2;
    const int res[2] = {q1, N1 - q1};
    const int64_t N2 = a.N2, S2 = a.S2, N = a.N, K = a.K;
    const int M = a.M, npair = a.npair, npi = a.npi;
    const int64_t xl = K / N1 + 2;
    V *FA = reinterpret_cast<V *>(smem_raw);      // [nres][npair][N2]
    V *FB = FA + 2 * npair * N2;                  // ping-pong
    V *Xl = FB + 2 * npair * N2;                  // [2][xl]
    V *UA = Xl + 2 * xl;                          // [nres][npi][S2]
    V *UB = UA + 2 * npi * S2;
    // 1. load T rows for both residues
    for (int64_t idx = threadIdx.x; idx < (int64_t)nres * npair * N2; idx += FB_NT) {
        const int r = (int)(idx / (npair * N2));
        const int c = (int)((idx / N2) % npair);
        const int64_t n2 = idx % N2;
        FA[idx] = a.Tw[((sl * npair + c) * N1 + res[r]) * N2 + n2];
    }
    __syncthreads();
    // 2. length-N2 forward DFTs: G_c[res_r + N1 q2] at Z[(r*npair + c)*N2 + q2]
    V *Z = block_fft_rt<T, -1>(FA, FB, (int)N2, nres * npair, (int)N2, a.twF, a.TW);
    // 3. solve classes q = res_r + N1 q2 <= N/2 and assemble X at p = +-res mod N1
    for (int64_t idx = threadIdx.x; idx < (int64_t)nres * N2; idx += FB_NT) {
        const int r = (int)(idx / N2);
        const int64_t q2 = idx % N2;
        const int64_t q = res[r] + (int64_t)N1 * q2;
        if (q > N / 2) continue;
        // mirror index (N - q) mod N = res_r' + N1 q2'
        const int rm = (nres == 1) ? 0 : 1 - r;
        const int64_t q2m = (res[r] == 0) ? ((N2 - q2) % N2) : (N2 - 1 - q2);
        const int64_t jq = -K + (((q + K) % N) + N) % N;
        V v[8];
#pragma unroll
        for (int l = 0; l < 8; ++l) v[l] = V{0, 0};
        for (int m = 0; m < M; ++m) {
            const int c = m >> 1;
            V zc = Z[((int64_t)r * npair + c) * N2 + q2], zm = cconj(Z[((int64_t)rm * npair + c) * N2 + q2m]);
            V gm = (m & 1) ? V{(T)0.5 * (zc.y - zm.y), (T)-0.5 * (zc.x - zm.x)}
                           : V{(T)0.5 * (zc.x + zm.x), (T)0.5 * (zc.y + zm.y)};
            const int em = chan_exp(a, sl, m);
            gm = V{ldexp(gm.x, em), ldexp(gm.y, em)};
            const V *qrow = a.Qt + (q * M + m) * M;
            for (int l = 0; l < M && l < 8; ++l) v[l] = cadd(v[l], cmul(gm, __ldg(qrow + l)));
        }
        const bool selfm = (q == 0) || (2 * q == N);
        for (int l = 0; l < M; ++l) {
            const int64_t k = jq + (int64_t)l * N;
            int64_t p = -1;
            V val;
            if (!selfm) {
                p = k > 0 ? k : -k;
                val = k > 0 ? v[l] : cconj(v[l]);
            } else {
                const int64_t lm = -k - jq;
                const bool neg_in = (lm >= 0) && (lm % N == 0) && (lm / N < M);
                if (k >= 0 || !neg_in) {
                    p = k >= 0 ? k : -k;
                    V ap = V{0, 0}, an = V{0, 0};
                    const int64_t lp = p - jq, ln = -p - jq;
                    if (lp >= 0 && lp % N == 0 && lp / N < M) ap = v[lp / N];
                    if (ln >= 0 && ln % N == 0 && ln / N < M) an = v[ln / N];
                    val = V{(T)0.5 * (ap.x + an.x), (T)0.5 * (ap.y - an.y)};
                }
            }
            if (p >= 0) {
                const int pr = (int)(p % N1);
                const int slot = (pr == res[0]) ? 0 : 1;
                Xl[slot * xl + p / N1] = val;
            }
        }
    }
    __syncthreads();
    // 4. pre-twiddle + inverse step 1 inputs: Zin[k2 + N1 k1], k2 = res_r
    for (int64_t idx = threadIdx.x; idx < (int64_t)nres * npi * S2; idx += FB_NT) {
        const int r = (int)(idx / (npi * S2));
        const int ip = (int)((idx / S2) % npi);
        const int64_t k1 = idx % S2;
        const int64_t kp = res[r] + (int64_t)N1 * k1;
        const int pa = 2 * ip, pb = 2 * ip + 1;
        V acc = V{0, 0};
#pragma unroll
        for (int w = 0; w < 2; ++w) {
            const int64_t k = w == 0 ? kp : kp - a.S;
            if (k > K || k < -K) continue;
            const int64_t ak = k >= 0 ? k : -k;
            const int slot = ((int)(ak % N1) == res[0]) ? 0 : 1;
            V y = Xl[slot * xl + ak / N1];
            V ta = a.twL(ak * pa), tb = a.twL(ak * pb);
            if (k < 0) { y = cconj(y); ta = cconj(ta); tb = cconj(tb); }
            V wa = cmul(y, ta);
            V wb = (pb < a.R) ? cmul(y, tb) : V{0, 0};
            acc = cadd(acc, V{wa.x - wb.y, wa.y + wb.x});
        }
        UA[idx] = acc;
    }
    __syncthreads();
    V *U = block_fft_rt<T, 1>(UA, UB, (int)S2, nres * npi, (int)S2, a.twF, a.TW);
    // 5. twiddle e^{2 pi i k2 u / S} and store U[ip][k2][u]
    for (int64_t idx = threadIdx.x; idx < (int64_t)nres * npi * S2; idx += FB_NT) {
        const int r = (int)(idx / (npi * S2));
        const int ip = (int)((idx / S2) % npi);
        const int64_t u = idx % S2;
        V val = cmul(U[idx], a.twS((int64_t)res[r] * u));
        a.Uw[((sl * npi + ip) * N1 + res[r]) * S2 + u] = val;
    }
}

// ---- IC ------------------------------------------------------------------------------------
static constexpr int IC_TU = 8, IC_NT = 512;

template <typename T>
__global__ void __launch_bounds__(IC_NT) mci_fs_ic(const FSArgs<T> a) {
    using V = cv<T>;
    extern __shared__ __align__(16) unsigned char smem_raw[];
    V *buf = reinterpret_cast<V *>(smem_raw);  // [npi*IC_TU][N1]
    const int64_t ntiles = a.S2 / IC_TU;
    const int64_t tile = blockIdx.x % ntiles;
    const int64_t sl = blockIdx.x / ntiles;
    const int npi = a.npi;
    const int64_t u0 = tile * IC_TU;
    for (int64_t idx = threadIdx.x; idx < (int64_t)npi * N1 * IC_TU; idx += IC_NT) {
        const int t = (int)(idx % IC_TU);
        const int k2 = (int)((idx / IC_TU) % N1);
        const int ip = (int)(idx / (IC_TU * N1));
        buf[(ip * IC_TU + t) * N1 + k2] = a.Uw[((sl * npi + ip) * N1 + k2) * a.S2 + u0 + t];
    }
    __syncthreads();
    if (npi == 2) block_fft_ct<T, N1, 1, 1, IC_NT, 2 * IC_TU>(buf, N1, a.twF, a.TW);
    else block_fft_ct<T, N1, 1, 1, IC_NT, IC_TU>(buf, N1, a.twF, a.TW);
    // f[R (u + S2 v) + p1]: for fixed v a run of IC_TU*R floats
    T *frow = a.f + (a.sig0 + sl) * a.L;
    const int R = (int)a.R;
    for (int64_t idx = threadIdx.x; idx < (int64_t)N1 * IC_TU; idx += IC_NT) {
        const int t = (int)(idx % IC_TU);
        const int v = (int)(idx / IC_TU);
        T vals[16];
        for (int ip = 0; ip < npi; ++ip) {
            V z = buf[(ip * IC_TU + t) * N1 + v];
            vals[2 * ip] = z.x;
            vals[2 * ip + 1] = z.y;
        }
        T *dst = frow + (int64_t)R * (u0 + t + a.S2 * v);
        if constexpr (sizeof(T) == 4) {
            if (R == 4 && aligned16(dst)) {
                *reinterpret_cast<float4 *>(dst) = make_float4(vals[0], vals[1], vals[2], vals[3]);
                continue;
            }
        }
        for (int j = 0; j < R; ++j) dst[j] = vals[j];
    }
}

// ---------------------------------------------------------------------------------------------
static size_t vsize(const Axis1D &ax) { return ax.dtype == MCI_F64 ? 16 : 8; }

size_t fourstep_ws_bytes_per_signal(const Axis1D &ax) {
    const int64_t npair = (ax.M + 1) / 2, npi = ax.R / 2;
    return (size_t)(npair * ax.N + npi * ax.S) * vsize(ax) + 8 * (size_t)ax.M;
}

static size_t fb_smem(const Axis1D &ax) {
    const int64_t npair = (ax.M + 1) / 2, npi = ax.R / 2;
    const int64_t N2 = ax.N / N1, S2 = ax.S / N1, xl = ax.K / N1 + 2;
    return (size_t)(4 * npair * N2 + 2 * xl + 4 * npi * S2) * vsize(ax);
}

bool fourstep_supported(const Axis1D &ax) {
    if (ax.analytic || ax.M > 8) return false;
    if (ax.N < 2 * N1 || ax.S < 2 * N1 || ax.N % N1 || ax.S % N1) return false;
    if (ax.R != 2 && ax.R != 4) return false;      // npi in {1,2}
    if ((ax.S / N1) % IC_TU) return false;
    return fb_smem(ax) <= 200 * 1024;
}

template <typename T>
static cudaError_t fs_launch_t(const Axis1D &ax, int64_t batch, const void *g, void *f, void *ws, int64_t ws_sig,
                               cudaStream_t st, int *nl) {
    FSArgs<T> a;
    a.M = ax.M; a.npair = (ax.M + 1) / 2; a.npi = (int)(ax.R / 2);
    a.N = ax.N; a.N2 = ax.N / N1; a.S = ax.S; a.S2 = ax.S / N1; a.L = ax.L; a.K = ax.K; a.R = ax.R;
    a.g = (const T *)g; a.f = (T *)f;
    a.Tw = (cv<T> *)ws;
    a.Uw = a.Tw + ws_sig * a.npair * ax.N;
    a.cmax = (decltype(a.cmax))(a.Uw + ws_sig * a.npi * ax.S);
    a.Qt = (const cv<T> *)ax.Qt; a.twF = (const cv<T> *)ax.twF; a.TW = ax.TW;
    a.fbt = ax.TW == 1024 ? (const cv<T> *)ax.rowtab : nullptr;
    a.Kmod = ax.K % ax.N;
    a.delay_uniform = ax.bank_delay_uniform;
    a.lmn = ax.bank_delay_uniform ? ax.L / ((int64_t)ax.M * ax.N) : 0;
    const cv<T> *const *ext = (const cv<T> *const *)nullptr;
    (void)ext;
    // two-level tables live right after twLlo in the plan's table block (see mci_plan.cpp)
    const cv<T> *blk = (const cv<T> *)ax.twLhi;
    const int64_t LO = ax.LO;
    const int lob = ilog2c(LO);
    // layout: [L/LO hi_L][LO lo_L][N/LO hi_N][LO lo_N][S/LO hi_S][LO lo_S]
    a.twL = Tw2<T>{blk, blk + ax.L / LO, lob, ax.L - 1};
    const cv<T> *nb = blk + ax.L / LO + LO;
    a.twN = Tw2<T>{nb, nb + ax.N / LO, lob, ax.N - 1};
    const cv<T> *sb = nb + ax.N / LO + LO;
    a.twS = Tw2<T>{sb, sb + ax.S / LO, lob, ax.S - 1};

    const size_t vs = vsize(ax);
    const int tn2 = (int)std::min<int64_t>(FA_TN2, a.N2);
    const size_t fa_sm = (size_t)tn2 * N1 * vs;
    auto fa = tn2 == 8 ? mci_fs_fa<T, 8> : (tn2 == 4 ? mci_fs_fa<T, 4> : mci_fs_fa<T, 2>);
    const size_t fb_sm = fb_smem(ax);
    const size_t ic_sm = (size_t)a.npi * IC_TU * N1 * vs;
    cudaError_t e;
    if ((e = cudaFuncSetAttribute(fa, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)fa_sm))) return e;
    if ((e = cudaFuncSetAttribute(mci_fs_fb<T>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)fb_sm))) return e;
    if ((e = cudaFuncSetAttribute(mci_fs_ic<T>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)ic_sm))) return e;
    const bool fast = fourstep_fast_ok(ax) && aligned16(g) && aligned16(f) && !getenv("MCI_FOURSTEP_GENERIC");
    for (int64_t s0 = 0; s0 < batch; s0 += ws_sig) {
        const int64_t ns = (batch - s0 < ws_sig) ? batch - s0 : ws_sig;
        a.sig0 = s0;
        // channel maxima for the exact power-of-two scaling before channel packing (R10); a
        // unimodular bank (|b_m(k)| = 1) gives channels of equal energy: no pre-pass, the
        // words stay 0 (zeroed at plan creation), i.e. no scaling (reading R14)
        const int pre = ax.bank_unimodular ? 0 : 1;
        if (pre) {
            if ((e = cudaMemsetAsync(a.cmax, 0, sizeof(*a.cmax) * ns * a.M, st))) return e;
            mci_fs_max<T><<<(unsigned)(ns * a.M * MX_BLK), MX_NT, 0, st>>>(a);
        }
        if constexpr (std::is_same<T, float>::value) {
            if (fast) {
                if ((e = fourstep_fast_chunk(a, ns, st))) return e;
                if (nl) *nl += 3 + pre;
                continue;
            }
        }
        fa<<<(unsigned)(ns * a.npair * (a.N2 / tn2)), FA_NT, fa_sm, st>>>(a);
        mci_fs_fb<T><<<(unsigned)(ns * (N1 / 2 + 1)), FB_NT, fb_sm, st>>>(a);
        mci_fs_ic<T><<<(unsigned)(ns * (a.S2 / IC_TU)), IC_NT, ic_sm, st>>>(a);
        if (nl) *nl += 3 + pre;
        if ((e = cudaGetLastError())) return e;
    }
    return cudaSuccess;
}

cudaError_t launch_fourstep(const Axis1D &ax, int64_t batch, const void *g, void *f, void *ws, int64_t ws_sig,
                            cudaStream_t st, int *nl) {
    if (batch <= 0) return cudaSuccess;
    if (ax.dtype == MCI_F64) return fs_launch_t<double>(ax, batch, g, f, ws, ws_sig, st, nl);
    return fs_launch_t<float>(ax, batch, g, f, ws, ws_sig, st, nl);
}

}  // namespace mci
