// Shared definitions of the four-step path (mci_fourstep.cu, mci_fourstep_fast.cu).
#pragma once

#include <type_traits>

#include "mci_fft.cuh"
#include "mci_internal.h"

namespace mci {

static constexpr int N1 = 1024;  // shared residue modulus / step-1 length

template <typename T> struct Tw2 {
    const cv<T> *hi, *lo;
    int lob;
    int64_t mask;  // size - 1
    __device__ __forceinline__ cv<T> operator()(int64_t m) const {
        m &= mask;
        return cmul(__ldg(hi + (m >> lob)), __ldg(lo + (m & ((1 << lob) - 1))));
    }
    // the same lookup with 32-bit index arithmetic (tables of at most 2^31 entries, |m| < 2^31)
    __device__ __forceinline__ cv<T> at32(int m) const {
        const unsigned mm = (unsigned)m & (unsigned)mask;
        return cmul(__ldg(hi + (mm >> lob)), __ldg(lo + (mm & ((1u << lob) - 1u))));
    }
};

template <typename T> struct FSArgs {
    int M, npair, npi;
    int64_t N, N2, S, S2, L, K, R;
    const T *g;
    T *f;
    cv<T> *Tw;  // workspace T   [sig][npair][N1][N2]
    cv<T> *Uw;  // workspace U   [sig][npi][N1][S2]
    const cv<T> *Qt;
    const cv<T> *twF;  // e^{-2 pi i m/TW} (TW >= max(N1, N2, S2))
    int64_t TW;
    Tw2<T> twN;  // e^{-2 pi i m/N}
    Tw2<T> twS;  // e^{+2 pi i m/S}
    Tw2<T> twL;  // e^{+2 pi i m/L}
    int64_t sig0;  // first signal of this chunk (input/output offset)
    int64_t Kmod;  // K mod N (class index j_q = -K + (q + Kmod) mod N without a division)
    int delay_uniform;  // closed-form solve for the uniform delay bank (Axis1D::bank_delay_uniform)
    int64_t lmn;        // L / (M N): e^{-i j tau_m} = conj(w_L^{j m lmn})
    typename std::conditional<sizeof(T) == 4, unsigned, unsigned long long>::type *cmax;  // [sig][M] |g| max bits
    const cv<T> *fbt = nullptr;  // packed kernels' tables [tw16 256][tw32 1024][tw128 96] (plan block)
};

// exponent e with max|g_m| = f 2^e, f in [0.5, 1) (0 for an all-zero channel)
template <typename T> __device__ __forceinline__ int chan_exp(const FSArgs<T> &a, int64_t sl, int m) {
    if (m >= a.M) return 0;
    T mx;
    if constexpr (sizeof(T) == 4) mx = __uint_as_float(a.cmax[sl * a.M + m]);
    else mx = __longlong_as_double((long long)a.cmax[sl * a.M + m]);
    int e = 0;
    if (mx > 0) frexp(mx, &e);
    return e;
}

bool fourstep_fast_ok(const Axis1D &ax);
cudaError_t fourstep_fast_chunk(const FSArgs<float> &a, int64_t ns, cudaStream_t st);

}  // namespace mci
