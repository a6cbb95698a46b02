// Device FFT building blocks for the MCI kernels (sm_100a).
//
// Complex values are float2/double2.  Radix-2/4/8/16 codelets run in
// registers; block FFTs are Stockham autosort passes through shared memory
// (natural order in, natural order out).  DIR = -1: forward e^{-2 pi i/n}
// (Lemma 1's omega); DIR = +1: inverse (unnormalised).
// Twiddles come from fp64-derived tables (no __sinf / fast math): SURVEY.md
// §8(c) item 15.
#pragma once

#include <cuda_runtime.h>
#include <type_traits>

namespace mci {

template <typename T> struct cvec;
template <> struct cvec<float> { using type = float2; };
template <> struct cvec<double> { using type = double2; };
template <typename T> using cv = typename cvec<T>::type;

template <typename V> __device__ __forceinline__ V cadd(V a, V b) { return V{a.x + b.x, a.y + b.y}; }
template <typename V> __device__ __forceinline__ V csub(V a, V b) { return V{a.x - b.x, a.y - b.y}; }
template <typename V> __device__ __forceinline__ V cmul(V a, V b) {
    return V{a.x * b.x - a.y * b.y, a.x * b.y + a.y * b.x};
}
template <typename V> __device__ __forceinline__ V cconj(V a) { return V{a.x, -a.y}; }
template <typename V, typename S> __device__ __forceinline__ V cscale(V a, S s) { return V{a.x * s, a.y * s}; }
// multiply by DIR*i : DIR=-1 -> -i v ; DIR=+1 -> +i v
template <int DIR, typename V> __device__ __forceinline__ V rot(V v) {
    if constexpr (DIR < 0) return V{v.y, -v.x};
    else return V{-v.y, v.x};
}

// multiply by e^{DIR 2 pi i E / 16}, E compile-time in [0,16)
template <int E, int DIR, typename V> __device__ __forceinline__ V tw16(V v) {
    using S = decltype(v.x);
    constexpr int e = E & 15;
    const S c1 = (S)0.92387953251128675613, s1 = (S)0.38268343236508977173;
    const S h = (S)0.70710678118654752440;
    if constexpr (e == 0) return v;
    else if constexpr (e == 4) return rot<DIR>(v);
    else if constexpr (e == 8) return V{-v.x, -v.y};
    else if constexpr (e == 12) return rot<-DIR>(v);
    else if constexpr (e == 2 || e == 6 || e == 10 || e == 14) {
        // (cos, DIR sin) of pi e/8 = multiples of 45 deg
        constexpr int q = e / 2;  // 1,3,5,7 -> angle q*45
        const S cr = (q == 1 || q == 7) ? h : -h;
        const S si = (q == 1 || q == 3) ? h : -h;
        const S sd = DIR < 0 ? -si : si;
        return V{v.x * cr - v.y * sd, v.x * sd + v.y * cr};
    } else {
        // odd e: angle e*22.5 deg
        constexpr int o = e;  // 1,3,5,7,9,11,13,15
        S c, s;
        if constexpr (o == 1) { c = c1; s = s1; }
        else if constexpr (o == 3) { c = s1; s = c1; }
        else if constexpr (o == 5) { c = -s1; s = c1; }
        else if constexpr (o == 7) { c = -c1; s = s1; }
        else if constexpr (o == 9) { c = -c1; s = -s1; }
        else if constexpr (o == 11) { c = -s1; s = -c1; }
        else if constexpr (o == 13) { c = s1; s = -c1; }
        else { c = c1; s = -s1; }
        const S sd = DIR < 0 ? -s : s;
        return V{v.x * c - v.y * sd, v.x * sd + v.y * c};
    }
}

template <int DIR, typename V> __device__ __forceinline__ void dft2(V &a, V &b) {
    V t = a;
    a = cadd(t, b);
    b = csub(t, b);
}

template <int DIR, typename V> __device__ __forceinline__ void dft4(V &x0, V &x1, V &x2, V &x3) {
    V t0 = cadd(x0, x2), t1 = csub(x0, x2), t2 = cadd(x1, x3), t3 = rot<DIR>(csub(x1, x3));
    x0 = cadd(t0, t2);
    x2 = csub(t0, t2);
    x1 = cadd(t1, t3);
    x3 = csub(t1, t3);
}

// In-register DFT of size R on x[0..R) (natural order in and out).
template <int R, int DIR, typename V> __device__ __forceinline__ void dft(V *x) {
    if constexpr (R == 1) {
    } else if constexpr (R == 2) {
        dft2<DIR>(x[0], x[1]);
    } else if constexpr (R == 4) {
        dft4<DIR>(x[0], x[1], x[2], x[3]);
    } else if constexpr (R == 8) {
        // x[n1 + 2 n2]: DFT4 over n2 for n1 = 0,1; twiddle w8^{n1 k2}; DFT2 over n1.
        dft4<DIR>(x[0], x[2], x[4], x[6]);
        dft4<DIR>(x[1], x[3], x[5], x[7]);
        x[3] = tw16<2, DIR>(x[3]);
        x[5] = tw16<4, DIR>(x[5]);
        x[7] = tw16<6, DIR>(x[7]);
        V y[8];
#pragma unroll
        for (int k2 = 0; k2 < 4; ++k2) {
            V a = x[2 * k2], b = x[2 * k2 + 1];
            y[k2] = cadd(a, b);
            y[k2 + 4] = csub(a, b);
        }
#pragma unroll
        for (int i = 0; i < 8; ++i) x[i] = y[i];
    } else if constexpr (R == 16) {
        // x[n1 + 4 n2]: DFT4 over n2 (k2), twiddle w16^{n1 k2}, DFT4 over n1 (k1); out y[k2 + 4 k1]
#pragma unroll
        for (int n1 = 0; n1 < 4; ++n1) dft4<DIR>(x[n1], x[n1 + 4], x[n1 + 8], x[n1 + 12]);
        // now x[n1 + 4 k2]
        x[5] = tw16<1, DIR>(x[5]);
        x[9] = tw16<2, DIR>(x[9]);
        x[13] = tw16<3, DIR>(x[13]);
        x[6] = tw16<2, DIR>(x[6]);
        x[10] = tw16<4, DIR>(x[10]);
        x[14] = tw16<6, DIR>(x[14]);
        x[7] = tw16<3, DIR>(x[7]);
        x[11] = tw16<6, DIR>(x[11]);
        x[15] = tw16<9, DIR>(x[15]);
        V y[16];
#pragma unroll
        for (int k2 = 0; k2 < 4; ++k2) {
            V a = x[4 * k2], b = x[4 * k2 + 1], c = x[4 * k2 + 2], d = x[4 * k2 + 3];
            dft4<DIR>(a, b, c, d);
            y[k2] = a;
            y[k2 + 4] = b;
            y[k2 + 8] = c;
            y[k2 + 12] = d;
        }
#pragma unroll
        for (int i = 0; i < 16; ++i) x[i] = y[i];
    } else {
        static_assert(R <= 16, "radix");
    }
}

// Twiddle e^{DIR 2 pi i m / TW} from the forward table tw[m] = e^{-2 pi i m/TW}.
template <int DIR, typename V> __device__ __forceinline__ V twid(const V *__restrict__ tw, int64_t m) {
    V w = __ldg(tw + m);
    if constexpr (DIR > 0) w.y = -w.y;
    return w;
}

// Block-wide max (NT threads, red = NT/32 scratch slots).  All threads get the result.
template <int NT, typename T> __device__ __forceinline__ T block_max(T v, T *red) {
#pragma unroll
    for (int o = 16; o; o >>= 1) v = fmax(v, __shfl_xor_sync(0xffffffffu, v, o));
    if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = v;
    __syncthreads();
    T r = red[0];
#pragma unroll
    for (int w = 1; w < NT / 32; ++w) r = fmax(r, red[w]);
    __syncthreads();
    return r;
}

__host__ __device__ constexpr int ilog2c(int64_t n) { return n <= 1 ? 0 : 1 + ilog2c(n / 2); }
// radix of the next pass for an n-point FFT after `done` points combined
__host__ __device__ constexpr int next_radix(int64_t n, int64_t done) {
    int rem = ilog2c(n / done);
    int passes = (rem + 3) / 4;
    int bits = passes ? (rem + passes - 1) / passes : 0;
    return 1 << bits;
}

// One Stockham pass, compile-time sizes, in place: every thread first loads
// all its butterflies, the block synchronises, then results are stored.
// `batch` sequences of length S at buf + b*bstride.
template <typename T, int S, int R, int LS, int DIR, int NT, int BATCH>
__device__ __forceinline__ void stockham_pass_ct(cv<T> *buf, int bstride, const cv<T> *__restrict__ tw,
                                                 int64_t TW) {
    using V = cv<T>;
    constexpr int NB = S / R;
    constexpr int TOT = NB * BATCH;
    constexpr int PER = (TOT + NT - 1) / NT;
    V x[PER][R];
#pragma unroll
    for (int u = 0; u < PER; ++u) {
        int id = threadIdx.x + u * NT;
        if (TOT % NT == 0 || id < TOT) {
            int b = id / NB, i = id % NB;
#pragma unroll
            for (int j = 0; j < R; ++j) x[u][j] = buf[b * bstride + i + j * NB];
        }
    }
    __syncthreads();
#pragma unroll
    for (int u = 0; u < PER; ++u) {
        int id = threadIdx.x + u * NT;
        if (TOT % NT == 0 || id < TOT) {
            int b = id / NB, i = id % NB;
            int k = i & (LS - 1);
            if constexpr (LS > 1) {
                const int64_t step = TW / (LS * R);
#pragma unroll
                for (int j = 1; j < R; ++j) x[u][j] = cmul(x[u][j], twid<DIR>(tw, (int64_t)(j * k) * step));
            }
            dft<R, DIR>(x[u]);
            int base = (i - k) * R + k;
#pragma unroll
            for (int j = 0; j < R; ++j) buf[b * bstride + base + j * LS] = x[u][j];
        }
    }
    __syncthreads();
}

template <typename T, int S, int LS, int DIR, int NT, int BATCH>
__device__ __forceinline__ void block_fft_ct(cv<T> *buf, int bstride, const cv<T> *__restrict__ tw, int64_t TW) {
    if constexpr (LS < S) {
        constexpr int R = next_radix(S, LS);
        stockham_pass_ct<T, S, R, LS, DIR, NT, BATCH>(buf, bstride, tw, TW);
        block_fft_ct<T, S, LS * R, DIR, NT, BATCH>(buf, bstride, tw, TW);
    }
}

// Runtime-size Stockham pass (out of place, src -> dst), radix R compile-time.
template <typename T, int R, int DIR>
__device__ __forceinline__ void stockham_pass_rt(const cv<T> *src, cv<T> *dst, int n, int ls, int batch,
                                                 int bstride, const cv<T> *__restrict__ tw, int64_t TW) {
    using V = cv<T>;
    const int nb = n / R;
    const int tot = nb * batch;
    const int64_t step = TW / ((int64_t)ls * R);
    for (int id = threadIdx.x; id < tot; id += blockDim.x) {
        int b = id / nb, i = id - b * nb;
        int k = i & (ls - 1);
        V x[R];
#pragma unroll
        for (int j = 0; j < R; ++j) x[j] = src[b * bstride + i + j * nb];
        if (ls > 1) {
#pragma unroll
            for (int j = 1; j < R; ++j) x[j] = cmul(x[j], twid<DIR>(tw, (int64_t)(j * k) * step));
        }
        dft<R, DIR>(x);
        int base = (i - k) * R + k;
#pragma unroll
        for (int j = 0; j < R; ++j) dst[b * bstride + base + j * ls] = x[j];
    }
}

// Runtime-size block FFT with ping-pong buffers a/b; returns the buffer
// holding the result.  Ends with __syncthreads().
template <typename T, int DIR>
__device__ cv<T> *block_fft_rt(cv<T> *a, cv<T> *b, int n, int batch, int bstride, const cv<T> *__restrict__ tw,
                               int64_t TW) {
    cv<T> *src = a, *dst = b;
    int ls = 1;
    while (ls < n) {
        int R = next_radix(n, ls);
        switch (R) {
        case 2: stockham_pass_rt<T, 2, DIR>(src, dst, n, ls, batch, bstride, tw, TW); break;
        case 4: stockham_pass_rt<T, 4, DIR>(src, dst, n, ls, batch, bstride, tw, TW); break;
        case 8: stockham_pass_rt<T, 8, DIR>(src, dst, n, ls, batch, bstride, tw, TW); break;
        default: stockham_pass_rt<T, 16, DIR>(src, dst, n, ls, batch, bstride, tw, TW); break;
        }
        __syncthreads();
        ls *= R;
        cv<T> *t = src; src = dst; dst = t;
    }
    return src;
}

}  // namespace mci

// ---------------------------------------------------------------------------------------
// Compile-time two-stage codelets (radix 32 = 4 x 8, radix 64 = 8 x 8) with constant
// twiddles from a 64th-root table (exact zeros/ones at the quadrant points).
namespace mci {
namespace cl {
// cos(2 pi e / 64), e = 0..16 (rounded from long double)
constexpr double C64[17] = {
    1.0, 0.99518472667219688624, 0.98078528040323044913, 0.95694033573220886494, 0.92387953251128675613,
    0.88192126434835502971, 0.83146961230254523708, 0.77301045336273696081, 0.70710678118654752440,
    0.63439328416364549822, 0.55557023301960222474, 0.47139673682599764856, 0.38268343236508977173,
    0.29028467725446236764, 0.19509032201612826785, 0.09801714032956060199, 0.0};
constexpr double cos64(int e) {
    e = ((e % 64) + 64) % 64;
    return e <= 16 ? C64[e] : (e <= 32 ? -C64[32 - e] : (e <= 48 ? -C64[e - 32] : C64[64 - e]));
}
constexpr double sin64(int e) { return cos64(e - 16); }

template <int B, int E, typename F> __device__ __forceinline__ void static_for(F &&f) {
    if constexpr (B < E) {
        f(std::integral_constant<int, B>{});
        static_for<B + 1, E>(f);
    }
}

// v * e^{DIR 2 pi i E / R}, R | 64, E compile-time
template <int R, int E, int DIR, typename V> __device__ __forceinline__ V twc(V v) {
    using S = decltype(v.x);
    constexpr int e64 = (((E % R) + R) % R) * (64 / R);
    if constexpr (e64 == 0) return v;
    else if constexpr (e64 == 16) return rot<DIR>(v);
    else if constexpr (e64 == 32) return V{-v.x, -v.y};
    else if constexpr (e64 == 48) return rot<-DIR>(v);
    else {
        constexpr S c = (S)cos64(e64);
        constexpr S s = (S)(DIR * sin64(e64));
        return V{v.x * c - v.y * s, v.x * s + v.y * c};
    }
}

// DFT of size R1*R2 on x[n1 + R1 n2] -> natural order x[k], k = k2 + R2 k1.
template <int R1, int R2, int DIR, typename V> __device__ __forceinline__ void dft2s(V *x) {
    constexpr int R = R1 * R2;
    V y[R];
    static_for<0, R1>([&](auto n1c) {
        constexpr int n1 = decltype(n1c)::value;
        V t[R2];
#pragma unroll
        for (int n2 = 0; n2 < R2; ++n2) t[n2] = x[n1 + R1 * n2];
        dft<R2, DIR>(t);
        static_for<0, R2>([&](auto k2c) {
            constexpr int k2 = decltype(k2c)::value;
            y[n1 + R1 * k2] = twc<R, n1 * k2, DIR>(t[k2]);
        });
    });
#pragma unroll
    for (int k2 = 0; k2 < R2; ++k2) {
        V t[R1];
#pragma unroll
        for (int n1 = 0; n1 < R1; ++n1) t[n1] = y[n1 + R1 * k2];
        dft<R1, DIR>(t);
#pragma unroll
        for (int k1 = 0; k1 < R1; ++k1) x[k2 + R2 * k1] = t[k1];
    }
}

template <int R, int DIR, typename V> __device__ __forceinline__ void dft_big(V *x) {
    if constexpr (R == 32) dft2s<4, 8, DIR>(x);
    else if constexpr (R == 64) dft2s<8, 8, DIR>(x);
    else dft<R, DIR>(x);
}
}  // namespace cl
}  // namespace mci
