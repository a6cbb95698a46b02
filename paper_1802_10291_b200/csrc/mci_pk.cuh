// Packed complex arithmetic on sm_100a FP32x2 instructions (FADD2 / FMUL2 / FFMA2).
//
// A complex fp32 value lives in one 64-bit register pair (re, im).  sm_100a
// executes add/mul/fma.rn.f32x2 at the same FLOP rate as scalar FFMA but in
// half the issue slots (measured on B200: tools/microbench/f32x2_throughput.cu,
// FFMA 69 TFLOP/s vs FFMA2 73 TFLOP/s), and ptxas folds swaps (LO_HI),
// broadcasts (.F32) and partial negation (.NP) into the operands, so
//   complex add/sub        1 instruction  (scalar: 2)
//   complex multiply       2 instructions (scalar: 4)
//   a +- (+-i) b           1 instruction  (scalar: 2)
// Arithmetic stays IEEE fp32 round-to-nearest (no fast math).
#pragma once

#include <cstdint>
#include <type_traits>

#include "mci_fft.cuh"

namespace mci {
// max over the warp of a non-negative float: non-negative floats order like their bit patterns, so one
// integer warp reduction (redux.sync) replaces five shuffle + max rounds
__device__ __forceinline__ float warp_max_nonneg(float m) {
    return __uint_as_float(__reduce_max_sync(0xffffffffu, __float_as_uint(m)));
}
namespace pkx {

struct pk {
    uint64_t v;
};

__device__ __forceinline__ pk mk(float x, float y) {
    pk r;
    asm("mov.b64 %0, {%1, %2};" : "=l"(r.v) : "f"(x), "f"(y));
    return r;
}
__device__ __forceinline__ pk mk(float2 a) { return mk(a.x, a.y); }
__device__ __forceinline__ float2 f2(pk a) {
    float2 v;
    asm("mov.b64 {%0, %1}, %2;" : "=f"(v.x), "=f"(v.y) : "l"(a.v));
    return v;
}
__device__ __forceinline__ pk add(pk a, pk b) {
    pk r;
    asm("add.rn.f32x2 %0, %1, %2;" : "=l"(r.v) : "l"(a.v), "l"(b.v));
    return r;
}
__device__ __forceinline__ pk sub(pk a, pk b) {
    pk r;
    asm("sub.rn.f32x2 %0, %1, %2;" : "=l"(r.v) : "l"(a.v), "l"(b.v));
    return r;
}
__device__ __forceinline__ pk mul(pk a, pk b) {
    pk r;
    asm("mul.rn.f32x2 %0, %1, %2;" : "=l"(r.v) : "l"(a.v), "l"(b.v));
    return r;
}
__device__ __forceinline__ pk fma(pk a, pk b, pk c) {
    pk r;
    asm("fma.rn.f32x2 %0, %1, %2, %3;" : "=l"(r.v) : "l"(a.v), "l"(b.v), "l"(c.v));
    return r;
}
__device__ __forceinline__ pk swp(pk a) {
    const float2 v = f2(a);
    return mk(v.y, v.x);
}
__device__ __forceinline__ pk conj(pk a) {
    const float2 v = f2(a);
    return mk(v.x, -v.y);
}
__device__ __forceinline__ pk bc(float s) { return mk(s, s); }

// x * w (complex), 2 instructions: w*x.re + (-w.im, w.re)*x.im
__device__ __forceinline__ pk cmul(pk x, pk w) {
    const float2 xf = f2(x), wf = f2(w);
    const pk p = mul(w, bc(xf.x));
    return fma(mk(-wf.y, wf.x), bc(xf.y), p);
}
// a + s*(DIR i)*b with s = +1/-1 folded: a + (DIR i) b  /  a - (DIR i) b
template <int DIR> __device__ __forceinline__ pk add_rot(pk a, pk b) {
    // (DIR i) b = DIR * (-b.im, b.re)
    const float2 bf = f2(b);
    return DIR > 0 ? add(a, mk(-bf.y, bf.x)) : add(a, mk(bf.y, -bf.x));
}
template <int DIR> __device__ __forceinline__ pk sub_rot(pk a, pk b) {
    const float2 bf = f2(b);
    return DIR > 0 ? add(a, mk(bf.y, -bf.x)) : add(a, mk(-bf.y, bf.x));
}
template <int DIR> __device__ __forceinline__ pk rot(pk b) {
    const float2 bf = f2(b);
    return DIR > 0 ? mk(-bf.y, bf.x) : mk(bf.y, -bf.x);
}

// v * e^{DIR 2 pi i E / R}, R | 64, E compile-time
template <int R, int E, int DIR> __device__ __forceinline__ pk twc(pk v) {
    constexpr int e64 = (((E % R) + R) % R) * (64 / R);
    if constexpr (e64 == 0) return v;
    else if constexpr (e64 == 16) return rot<DIR>(v);
    else if constexpr (e64 == 32) return mul(v, bc(-1.f));
    else if constexpr (e64 == 48) return rot<-DIR>(v);
    else {
        constexpr float c = (float)cl::cos64(e64);
        constexpr float s = (float)(DIR * cl::sin64(e64));
        const float2 vf = f2(v);
        return fma(mk(-vf.y, vf.x), bc(s), mul(v, bc(c)));
    }
}

// Fused twiddle butterfly: (a, b) <- (a + w b, a - w b), w = e^{DIR 2 pi i E / 64}, E compile-time.
// Quadrant points are swizzled adds (2 instructions); a general w = c + i s costs 3 instead of the
// 4 of a complex multiply and two adds: u = b + (s/c)(i b), then a +- c u (|c| >= |s|), or
// u = i b + (c/s) b, then a +- s u.  Each output is rounded twice, as with the unfused form.
#ifndef MCI_PK_FUSED
#define MCI_PK_FUSED 1
#endif
template <int E, int DIR> __device__ __forceinline__ void twf(pk &a, pk &b) {
    constexpr int e = ((E % 64) + 64) % 64;
    const pk t = a;
    if constexpr (e == 0) {
        a = add(t, b);
        b = sub(t, b);
    } else if constexpr (e == 16) {
        a = add_rot<DIR>(t, b);
        b = sub_rot<DIR>(t, b);
    } else if constexpr (e == 32) {
        a = sub(t, b);
        b = add(t, b);
    } else if constexpr (e == 48) {
        a = sub_rot<DIR>(t, b);
        b = add_rot<DIR>(t, b);
    } else {
        constexpr double c = cl::cos64(e), sn = DIR * cl::sin64(e);
        constexpr bool CB = (c < 0 ? -c : c) >= (sn < 0 ? -sn : sn);
        constexpr float f = (float)(CB ? c : sn), r = (float)(CB ? sn / c : c / sn);
        const float2 bf = f2(b);
        const pk ib = mk(-bf.y, bf.x);  // i b
        const pk u = CB ? fma(ib, bc(r), b) : fma(b, bc(r), ib);
        a = fma(u, bc(f), t);
        b = fma(u, bc(-f), t);
    }
}

// DFT of size R (power of two, <= 64) of the inputs x[n] w^{n E}, w = e^{DIR 2 pi i / 64}
// (input twiddles E compile-time, in 64ths of a turn), natural order in and out: radix-2
// decimation in time whose every twiddle rides in a fused butterfly (twf).
template <int R, int E, int DIR> __device__ __forceinline__ void dftw(pk *x) {
    if constexpr (R == 2) {
        twf<E, DIR>(x[0], x[1]);
    } else if constexpr (R > 2) {
        pk ev[R / 2], od[R / 2];
#pragma unroll
        for (int m = 0; m < R / 2; ++m) {
            ev[m] = x[2 * m];
            od[m] = x[2 * m + 1];
        }
        dftw<R / 2, 2 * E, DIR>(ev);
        dftw<R / 2, 2 * E, DIR>(od);
        cl::static_for<0, R / 2>([&](auto kc) {
            constexpr int k = decltype(kc)::value;
            twf<E + (64 / R) * k, DIR>(ev[k], od[k]);
            x[k] = ev[k];
            x[k + R / 2] = od[k];
        });
    }
}

template <int DIR> __device__ __forceinline__ void dft2(pk &a, pk &b) {
    const pk t = a;
    a = add(t, b);
    b = sub(t, b);
}
template <int DIR> __device__ __forceinline__ void dft4(pk &x0, pk &x1, pk &x2, pk &x3) {
    const pk t0 = add(x0, x2), t1 = sub(x0, x2), t2 = add(x1, x3), t3 = sub(x1, x3);
    x0 = add(t0, t2);
    x2 = sub(t0, t2);
    x1 = add_rot<DIR>(t1, t3);
    x3 = sub_rot<DIR>(t1, t3);
}

template <int R, int DIR> __device__ __forceinline__ void dft(pk *x);

template <int R1, int R2, int DIR> __device__ __forceinline__ void dft2s(pk *x) {
    constexpr int R = R1 * R2;
    pk y[R];
    cl::static_for<0, R1>([&](auto n1c) {
        constexpr int n1 = decltype(n1c)::value;
        pk t[R2];
#pragma unroll
        for (int n2 = 0; n2 < R2; ++n2) t[n2] = x[n1 + R1 * n2];
        dft<R2, DIR>(t);
        cl::static_for<0, R2>([&](auto k2c) {
            constexpr int k2 = decltype(k2c)::value;
            y[n1 + R1 * k2] = MCI_PK_FUSED ? t[k2] : twc<R, n1 * k2, DIR>(t[k2]);
        });
    });
    cl::static_for<0, R2>([&](auto k2c) {
        constexpr int k2 = decltype(k2c)::value;
        pk t[R1];
#pragma unroll
        for (int n1 = 0; n1 < R1; ++n1) t[n1] = y[n1 + R1 * k2];
        if constexpr (MCI_PK_FUSED) dftw<R1, (64 / R) * k2, DIR>(t);  // twiddles w^{n1 k2} fused
        else dft<R1, DIR>(t);
#pragma unroll
        for (int k1 = 0; k1 < R1; ++k1) x[k2 + R2 * k1] = t[k1];
    });
}

// In-register DFT of size R (natural order in/out).
template <int R, int DIR> __device__ __forceinline__ void dft(pk *x) {
    if constexpr (R == 1) {
    } else if constexpr (R == 2) {
        dft2<DIR>(x[0], x[1]);
    } else if constexpr (R == 4) {
        dft4<DIR>(x[0], x[1], x[2], x[3]);
    } else if constexpr (R == 8) {
        dft2s<2, 4, DIR>(x);
    } else if constexpr (R == 16) {
        dft2s<4, 4, DIR>(x);
    } else if constexpr (R == 32) {
        dft2s<4, 8, DIR>(x);
    } else if constexpr (R == 64) {
        dft2s<8, 8, DIR>(x);
    } else {
        static_assert(R <= 64, "radix");
    }
}

// ---- DFTs with compile-time zero inputs (bit n of Z: x[n] == 0, never read).
// Only the first stage of each sub-transform changes; supports at most one zero per
// radix-4 / radix-2 group (asserted), which is all the row kernel needs.
template <int R, int DIR, unsigned long long Z> __device__ __forceinline__ void dftz(pk *x);

template <int DIR, unsigned Z> __device__ __forceinline__ void dft4z(pk &x0, pk &x1, pk &x2, pk &x3) {
    static_assert((Z & 5) != 5 && (Z & 10) != 10, "at most one zero per butterfly pair");
    pk t0, t1;  // x0 +- x2
    if constexpr (Z & 4) { t0 = x0; t1 = x0; }
    else if constexpr (Z & 1) { t0 = x2; t1 = mul(x2, bc(-1.f)); }
    else { t0 = add(x0, x2); t1 = sub(x0, x2); }
    if constexpr (Z & 8) {  // x3 = 0: x1 +- x3 = x1
        const pk u = x1;
        x0 = add(t0, u);
        x2 = sub(t0, u);
        x1 = add_rot<DIR>(t1, u);
        x3 = sub_rot<DIR>(t1, u);
    } else if constexpr (Z & 2) {  // x1 = 0: x1 + x3 = x3, x1 - x3 = -x3
        const pk u = x3;
        x0 = add(t0, u);
        x2 = sub(t0, u);
        x1 = sub_rot<DIR>(t1, u);
        x3 = add_rot<DIR>(t1, u);
    } else {
        const pk t2 = add(x1, x3), t3 = sub(x1, x3);
        x0 = add(t0, t2);
        x2 = sub(t0, t2);
        x1 = add_rot<DIR>(t1, t3);
        x3 = sub_rot<DIR>(t1, t3);
    }
}

template <unsigned long long Z, int n1, int R1, int R2> constexpr unsigned long long sub_mask() {
    unsigned long long m = 0;
    for (int n2 = 0; n2 < R2; ++n2)
        if ((Z >> (n1 + R1 * n2)) & 1ull) m |= 1ull << n2;
    return m;
}

template <int R1, int R2, int DIR, unsigned long long Z> __device__ __forceinline__ void dft2sz(pk *x) {
    constexpr int R = R1 * R2;
    pk y[R];
    cl::static_for<0, R1>([&](auto n1c) {
        constexpr int n1 = decltype(n1c)::value;
        constexpr unsigned long long zm = sub_mask<Z, n1, R1, R2>();
        pk t[R2];
#pragma unroll
        for (int n2 = 0; n2 < R2; ++n2)
            if (!((zm >> n2) & 1ull)) t[n2] = x[n1 + R1 * n2];
        dftz<R2, DIR, zm>(t);
        cl::static_for<0, R2>([&](auto k2c) {
            constexpr int k2 = decltype(k2c)::value;
            y[n1 + R1 * k2] = MCI_PK_FUSED ? t[k2] : twc<R, n1 * k2, DIR>(t[k2]);
        });
    });
    cl::static_for<0, R2>([&](auto k2c) {
        constexpr int k2 = decltype(k2c)::value;
        pk t[R1];
#pragma unroll
        for (int n1 = 0; n1 < R1; ++n1) t[n1] = y[n1 + R1 * k2];
        if constexpr (MCI_PK_FUSED) dftw<R1, (64 / R) * k2, DIR>(t);
        else dft<R1, DIR>(t);
#pragma unroll
        for (int k1 = 0; k1 < R1; ++k1) x[k2 + R2 * k1] = t[k1];
    });
}

template <int R, int DIR, unsigned long long Z> __device__ __forceinline__ void dftz(pk *x) {
    if constexpr (Z == 0) {
        dft<R, DIR>(x);
    } else if constexpr (R == 4) {
        dft4z<DIR, (unsigned)Z>(x[0], x[1], x[2], x[3]);
    } else if constexpr (R == 8) {
        dft2sz<2, 4, DIR, Z>(x);
    } else if constexpr (R == 16) {
        dft2sz<4, 4, DIR, Z>(x);
    } else if constexpr (R == 32) {
        dft2sz<4, 8, DIR, Z>(x);
    } else if constexpr (R == 64) {
        dft2sz<8, 8, DIR, Z>(x);
    } else {
        static_assert(R == 4, "dftz radix");
    }
}

}  // namespace pkx
}  // namespace mci
