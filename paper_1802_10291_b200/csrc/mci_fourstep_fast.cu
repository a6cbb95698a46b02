// Packed-FP32x2 four-step kernels for the config-4 shape (N = N1 * N2 with
// N1 = 1024, N2 = 256; S = N1 * S2 with S2 = 1024; M in {3, 4}; R = 4).
// Same decomposition and workspace layout as mci_fourstep.cu (FA / FB / IC;
// see the header comment there), with register radix-32 / radix-16 two-pass
// FFTs (packed complex arithmetic, mci_pk.cuh), padded shared buffers and
// coalesced 32-64 byte global runs.  Selected by launch_fourstep when the
// shape matches; the generic kernels remain the fallback.
#include <cstdlib>

#include "mci_fourstep.cuh"
#include "mci_pk.cuh"

#ifndef MCI_FSF_B32
#define MCI_FSF_B32 1  // 0: phase B of FB with 64-bit indices and three table lookups per class (A/B)
#endif

namespace mci {

namespace fsf {
constexpr int N2 = 256, S2 = 1024;  // N1 = 1024 from mci_fourstep.cuh
__device__ __forceinline__ int pad5(int a) { return a + (a >> 5); }
__device__ __forceinline__ int pad4(int a) { return a + (a >> 4); }
__device__ __forceinline__ float pow2f(int e) { return __int_as_float((127 + e) << 23); }
// one bulk copy (cp.async.bulk + mbarrier transaction count) of a CTA's twiddle tables from
// the plan block into shared memory; issued by thread 0, awaited by each thread before use
__device__ __forceinline__ uint32_t su32(const void *p) { return (uint32_t)__cvta_generic_to_shared(p); }
__device__ __forceinline__ void tab_copy(void *dst, const void *src, uint32_t bytes, uint64_t *mb) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(su32(mb)) : "memory");
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(su32(mb)), "r"(bytes) : "memory");
    asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
                     su32(dst)),
                 "l"(src), "r"(bytes), "r"(su32(mb))
                 : "memory");
}
__device__ __forceinline__ void tab_wait(uint64_t *mb) {
    uint32_t done = 0;
    while (!done)
        asm volatile("{ .reg .pred p; mbarrier.try_wait.parity.shared::cta.b64 p, [%1], 0; selp.u32 %0, 1, 0, p; }"
                     : "=r"(done)
                     : "r"(su32(mb))
                     : "memory");
}
// e^{2 pi i E / 128} as a compile-time constant (half-angle from the 64th-root table)
constexpr double csqrt(double x) {
    double r = x > 1 ? x : 1;
    for (int it = 0; it < 80; ++it) r = 0.5 * (r + x / r);
    return r;
}
constexpr double cos128(int e) {
    e = ((e % 128) + 128) % 128;
    if (e % 2 == 0) return cl::cos64(e / 2);
    const double m = csqrt(0.5 * (1.0 + cl::cos64(e)));  // |cos(a)|, cos(2a) = cos64(e)
    return (e <= 32 || e >= 96) ? m : -m;
}
constexpr double sin128(int e) { return cos128(e - 32); }
template <int E> __device__ __forceinline__ pkx::pk c128() {
    constexpr float c = (float)cos128(E), s = (float)sin128(E);
    return pkx::mk(c, s);
}
}  // namespace fsf

using pkx::pk;

// ---- FA: COLS FFTs of length N1 over n1 for COLS consecutive residues n2 ----------------------
// COLS = 8 (256 threads, 32-byte input runs, 64-byte T runs, 76 KB) or 16 (512 threads, 64 / 128-byte
// runs, 143 KB, one CTA per SM); lane = COLS il + t2: FFT t2 (n2 = tile * COLS + t2), butterfly i
template <int COLS>
__global__ void __launch_bounds__(32 * COLS) mci_fsf_fa(const FSArgs<float> a) {
    using namespace fsf;
    using namespace pkx;
    extern __shared__ __align__(16) unsigned char smem[];
    constexpr int BS = COLS == 8 ? 1056 + 2 : 1056 + 1;  // per-FFT stride: conflict-free per half-warp
    constexpr int NT = 32 * COLS, LB = COLS == 8 ? 3 : 4;
    float2 *bufs = reinterpret_cast<float2 *>(smem);
    float2 *tw = bufs + COLS * BS;  // [32][32] e^{-2 pi i j i / 1024}
    __shared__ __align__(8) uint64_t tmb;
    if (a.fbt) {
        if (threadIdx.x == 0) tab_copy(tw, a.fbt + 256, 1024 * 8, &tmb);
    } else {
        for (int q = threadIdx.x; q < 1024; q += NT) tw[q] = __ldg(a.twF + (((q >> 5) * (q & 31)) & 1023));
    }
    __syncthreads();
    const int ntiles = N2 / COLS;
    const int tile = blockIdx.x % ntiles;
    const int c = (blockIdx.x / ntiles) % a.npair;
    const int64_t sl = blockIdx.x / ((int64_t)ntiles * a.npair);
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int t2 = lane & (COLS - 1), i = (32 / COLS) * warp + (lane >> LB);
    const int n2 = tile * COLS + t2;
    const float *g0 = a.g + (a.sig0 + sl) * (int64_t)a.M * a.N + (int64_t)(2 * c) * a.N;
    const float *g1 = g0 + a.N;
    const bool has1 = 2 * c + 1 < a.M;
    const pk sc = mk(pow2f(-chan_exp(a, sl, 2 * c)), pow2f(-chan_exp(a, sl, 2 * c + 1)));
    float2 *buf = bufs + t2 * BS;
    pk x[32];
#pragma unroll
    for (int j = 0; j < 32; ++j) {
        const int64_t n = (int64_t)(i + 32 * j) * N2 + n2;
        x[j] = mul(mk(__ldg(g0 + n), has1 ? __ldg(g1 + n) : 0.f), sc);
    }
    dft<32, -1>(x);
#pragma unroll
    for (int j = 0; j < 32; ++j) buf[pad5(32 * i + j)] = f2(x[j]);
    __syncthreads();
#pragma unroll
    for (int j = 0; j < 32; ++j) x[j] = mk(buf[pad5(i + 32 * j)]);
    if (a.fbt) tab_wait(&tmb);
#pragma unroll
    for (int j = 1; j < 32; ++j) x[j] = pkx::cmul(x[j], mk(tw[j * 32 + i]));
    dft<32, -1>(x);
    float2 *out = reinterpret_cast<float2 *>(a.Tw + (sl * a.npair + c) * (int64_t)N1 * N2);
#pragma unroll
    for (int j = 0; j < 32; ++j) {
        const int q1 = i + 32 * j;
        out[q1 * N2 + n2] = f2(pkx::cmul(x[j], mk(a.twN.at32(n2 * q1))));  // n2 q1 < 2^18: 32-bit indices
    }
}

// ---- FB: forward step 2 + solve + assembly + inverse step 1 for the residue pair --------------
__global__ void __launch_bounds__(128, 5) mci_fsf_fb(const FSArgs<float> a) {
    using namespace fsf;
    using namespace pkx;
    extern __shared__ __align__(16) unsigned char smem[];
    constexpr int GB = 272 + 1;   // forward buffer stride (4 FFTs of 256, pad4)
    constexpr int IB = 1056 + 4;  // inverse buffer stride (4 FFTs of 1024, pad5); == 4 mod 16
    const int64_t xl = a.K / N1 + 2;
    // the inverse buffers (phase C) alias the forward buffers (phases A-B), which are dead after
    // the barrier that follows the solve; the radix-16 / radix-32 twiddles are read through L1
    // from the plan block (not staged per CTA): 43 KB per CTA, 5 CTAs (20 warps) per SM
    float2 *fb = reinterpret_cast<float2 *>(smem);  // 4 x GB
    float2 *G = fb + 4 * GB;                         // [4][256] natural order
    float2 *ib = fb;                                 // 4 x IB (phase C)
    float2 *Xl = fb + 4 * IB;                        // [2][xl]  (4 IB >= 4 GB + 4 x 256)
    const float2 *gt16 = a.fbt, *gt32 = a.fbt + 256;  // plan block: [16][16] e^{-2 pi i j b/256}, [32][32] e^{-2 pi i j i/1024}
    float2 *tw128 = Xl + 2 * xl;                     // [3][32] e^{2 pi i e j / 128}, e = 1, 2, 3
    float2 *twE = tw128 + 96;                        // [2][32] e^{2 pi i 32 res_r j / S}
    __shared__ __align__(8) uint64_t tmb;
    const int q1 = blockIdx.x % (N1 / 2 + 1);
    if (a.fbt) {  // plan block: [tw16 256][tw32 1024][tw128 96]
        if (threadIdx.x == 0) tab_copy(tw128, a.fbt + 256 + 1024, 96 * 8, &tmb);
    } else {
        for (int q = threadIdx.x; q < 96; q += 128) {  // e^{+2 pi i e j / 128} = conj(twF[8 e j])
            const float2 v = __ldg(a.twF + ((8 * ((q >> 5) + 1) * (q & 31)) & 1023));
            tw128[q] = make_float2(v.x, -v.y);
        }
    }
#if MCI_FSF_B32
    // warps 2-3, idle during phase A, fill the phase-C table; warps 0-1 go straight to their loads
    // (the tables are first read after the barrier that ends phase A)
    if (threadIdx.x >= 64) {
        const int q = threadIdx.x - 64;
        const int rq = (q >> 5) == 0 ? q1 : N1 - q1;
        twE[q] = a.twS((int64_t)32 * rq * (q & 31));
    }
#else
    for (int q = threadIdx.x; q < 64; q += 128) {
        const int rq = (q >> 5) == 0 ? q1 : N1 - q1;
        twE[q] = a.twS((int64_t)32 * rq * (q & 31));
    }
#endif
    const int64_t sl = blockIdx.x / (N1 / 2 + 1);
    const int nres = (q1 == 0 || q1 == N1 / 2) ? 1 : 2;
    const int res[2] = {q1, N1 - q1};
    const int64_t N = a.N, K = a.K;
    const int M = a.M, npair = a.npair, tid = threadIdx.x;
#if MCI_FSF_B32
    // phase C's per-thread factor w^{res + N1 i}: its two table loads overlap phases A-B
    const pk P1early = mk(a.twL((int64_t)res[(tid >> 6) < nres ? (tid >> 6) : 0] + (int64_t)N1 * (tid & 31)));
    float sup[4];  // channel scales: their loads overlap phase A
#pragma unroll
    for (int m = 0; m < 4; ++m) sup[m] = 0.5f * pow2f(chan_exp(a, sl, m));
    if (!a.fbt) __syncthreads();  // (generic table fill above used every thread)
#else
    __syncthreads();
#endif
    // -- A: 4 forward FFTs of length 256 (residue r, pair c): radix 16 x 16 on 64 threads
    if (tid < 64) {
        const int fi = tid >> 4, b = tid & 15, r = fi >> 1, c = fi & 1;
        if (r < nres) {
            const float2 *trow = reinterpret_cast<const float2 *>(a.Tw) + ((sl * npair + c) * N1 + res[r]) * (int64_t)N2;
            float2 *buf = fb + fi * GB;
            pk x[16];
#pragma unroll
            for (int j = 0; j < 16; ++j) x[j] = mk(trow[b + 16 * j]);
            dft<16, -1>(x);
#pragma unroll
            for (int j = 0; j < 16; ++j) buf[pad4(16 * b + j)] = f2(x[j]);
            __syncwarp();
            asm volatile("bar.sync 1, 64;" ::: "memory");
#pragma unroll
            for (int j = 0; j < 16; ++j) x[j] = mk(buf[pad4(b + 16 * j)]);
#pragma unroll
            for (int j = 1; j < 16; ++j)
                x[j] = pkx::cmul(x[j], mk(a.fbt ? __ldg(gt16 + j * 16 + b) : __ldg(a.twF + ((4 * j * b) & 1023))));
            dft<16, -1>(x);
#pragma unroll
            for (int j = 0; j < 16; ++j) G[fi * 256 + b + 16 * j] = f2(x[j]);
        } else {
            asm volatile("bar.sync 1, 64;" ::: "memory");
        }
    }
    __syncthreads();
    // -- B: solve classes q = res_r + N1 q2 <= N/2 and assemble X at p = +-res mod N1
#if !MCI_FSF_B32
    float sup[4];
#pragma unroll
    for (int m = 0; m < 4; ++m) sup[m] = 0.5f * pow2f(chan_exp(a, sl, m));
#endif
#if MCI_FSF_B32
    // 32-bit index arithmetic (every index of this shape is below 2^23: N = 2^18, K = 2^19, L = 2^22) and
    // the delay phases e^{-i j tau_m}, m = 1..3, as powers of one table value instead of three lookups
    // (phase B took 32 % of the kernel's samples for 48 packed FP instructions out of ~600: 64-bit
    // index arithmetic and the table round trips)
    {
        const int Ni = (int)N, Ki = (int)K, Kmodi = (int)a.Kmod, lmni = (int)a.lmn, xli = (int)xl;
        const unsigned lmask = (unsigned)a.twL.mask, lolen = (1u << a.twL.lob) - 1u;
        const int lob = a.twL.lob;
        auto twL32 = [&](int m) {
            const unsigned mm = (unsigned)m & lmask;
            return pkx::cmul(mk(__ldg(a.twL.hi + (mm >> lob))), mk(__ldg(a.twL.lo + (mm & lolen))));
        };
        for (int idx = tid; idx < nres * N2; idx += 128) {
            const int r = idx >> 8, q2 = idx & (N2 - 1);
            const int q = res[r] + N1 * q2;
            if (q > Ni / 2) continue;
            const int rm = (nres == 1) ? 0 : 1 - r;
            const int q2m = (res[r] == 0) ? ((N2 - q2) & (N2 - 1)) : (N2 - 1 - q2);
            int jt = q + Kmodi;
            if (jt >= Ni) jt -= Ni;
            const int jq = -Ki + jt;
            pk gm[4];
#pragma unroll
            for (int m = 0; m < 4; ++m) {
                if (m < M) {
                    const int c = m >> 1;
                    const pk zc = mk(G[(r * 2 + c) * 256 + q2]), zm = pkx::conj(mk(G[(rm * 2 + c) * 256 + q2m]));
                    gm[m] = (m & 1) ? mul(rot<-1>(sub(zc, zm)), bc(sup[m])) : mul(add(zc, zm), bc(sup[m]));
                } else {
                    gm[m] = mk(0.f, 0.f);
                }
            }
            pk v[4];
            if (a.delay_uniform) {
                const float s = 1.f / (float)(M * Ni);
                const pk w1 = pkx::conj(twL32(jq * lmni));  // e^{-i j tau_1}
                const pk w2 = pkx::cmul(w1, w1), w3 = pkx::cmul(w2, w1);
                pk u[4];
                u[0] = mul(gm[0], bc(s));
                u[1] = mul(pkx::cmul(gm[1], w1), bc(s));
                u[2] = mul(pkx::cmul(gm[2], w2), bc(s));
                u[3] = mul(pkx::cmul(gm[3], w3), bc(s));
                const pk t0 = add(u[0], u[2]), t1 = sub(u[0], u[2]), t2 = add(u[1], u[3]), t3 = sub(u[1], u[3]);
                v[0] = add(t0, t2);
                v[2] = sub(t0, t2);
                v[1] = add_rot<-1>(t1, t3);
                v[3] = sub_rot<-1>(t1, t3);
            } else {
                const float2 *Qq = reinterpret_cast<const float2 *>(a.Qt) + (int64_t)q * M * M;
#pragma unroll
                for (int l = 0; l < 4; ++l) {
                    pk acc = mk(0.f, 0.f);
#pragma unroll
                    for (int m = 0; m < 4; ++m)
                        if (m < M && l < M) acc = add(acc, pkx::cmul(gm[m], mk(__ldg(Qq + m * M + l))));
                    v[l] = acc;
                }
            }
            const bool selfm = (q == 0) || (2 * q == Ni);
#pragma unroll
            for (int l = 0; l < 4; ++l) {
                if (l >= M) break;
                const int k = jq + l * Ni;
                int p = -1;
                float2 val;
                if (!selfm) {
                    p = k > 0 ? k : -k;
                    val = k > 0 ? f2(v[l]) : f2(pkx::conj(v[l]));
                } else {
                    const int lm = -k - jq;
                    const bool neg_in = (lm >= 0) && (lm % Ni == 0) && (lm / Ni < M);
                    if (k >= 0 || !neg_in) {
                        p = k >= 0 ? k : -k;
                        pk ap = mk(0.f, 0.f), an = mk(0.f, 0.f);
                        const int lp = p - jq, ln = -p - jq;
#pragma unroll
                        for (int l2 = 0; l2 < 4; ++l2) {
                            if (l2 < M && lp == l2 * Ni) ap = v[l2];
                            if (l2 < M && ln == l2 * Ni) an = v[l2];
                        }
                        val = f2(mul(add(ap, pkx::conj(an)), bc(0.5f)));
                    }
                }
                if (p >= 0) Xl[((p & (N1 - 1)) == res[0] ? 0 : 1) * xli + (p >> 10)] = val;
            }
        }
    }
#else
    for (int idx = tid; idx < nres * N2; idx += 128) {
        const int r = idx / N2, q2 = idx % N2;
        const int64_t q = res[r] + (int64_t)N1 * q2;
        if (q > N / 2) continue;
        const int rm = (nres == 1) ? 0 : 1 - r;
        const int q2m = (res[r] == 0) ? ((N2 - q2) % N2) : (N2 - 1 - q2);
        int64_t jt = q + a.Kmod;
        if (jt >= N) jt -= N;
        const int64_t jq = -K + jt;
        pk gm[4];
#pragma unroll
        for (int m = 0; m < 4; ++m) {
            if (m < M) {
                const int c = m >> 1;
                const pk zc = mk(G[(r * 2 + c) * 256 + q2]), zm = pkx::conj(mk(G[(rm * 2 + c) * 256 + q2m]));
                gm[m] = (m & 1) ? mul(rot<-1>(sub(zc, zm)), bc(sup[m])) : mul(add(zc, zm), bc(sup[m]));
            } else {
                gm[m] = mk(0.f, 0.f);
            }
        }
        pk v[4];
        if (a.delay_uniform) {
            // H^{-1}/N = diag(e^{-i j tau_m}) W^H / (M N): twiddle, then a 4-point DFT
            const float s = 1.f / (float)(M * N);
            pk u[4];
            u[0] = mul(gm[0], bc(s));
#pragma unroll
            for (int m = 1; m < 4; ++m) {
                const float2 w = a.twL(jq * m * a.lmn);  // e^{+i j tau_m}
                u[m] = mul(pkx::cmul(gm[m], mk(w.x, -w.y)), bc(s));
            }
            const pk t0 = add(u[0], u[2]), t1 = sub(u[0], u[2]), t2 = add(u[1], u[3]), t3 = sub(u[1], u[3]);
            v[0] = add(t0, t2);
            v[2] = sub(t0, t2);
            v[1] = add_rot<-1>(t1, t3);  // u0 - i u1 - u2 + i u3
            v[3] = sub_rot<-1>(t1, t3);
        } else {
            const float2 *Qq = reinterpret_cast<const float2 *>(a.Qt) + q * M * M;
#pragma unroll
            for (int l = 0; l < 4; ++l) {
                pk acc = mk(0.f, 0.f);
#pragma unroll
                for (int m = 0; m < 4; ++m)
                    if (m < M && l < M) acc = add(acc, pkx::cmul(gm[m], mk(__ldg(Qq + m * M + l))));
                v[l] = acc;
            }
        }
        const bool selfm = (q == 0) || (2 * q == N);
#pragma unroll
        for (int l = 0; l < 4; ++l) {
            if (l >= M) break;
            const int64_t k = jq + (int64_t)l * N;
            int64_t p = -1;
            float2 val;
            if (!selfm) {
                p = k > 0 ? k : -k;
                val = k > 0 ? f2(v[l]) : f2(pkx::conj(v[l]));
            } else {
                const int64_t lm = -k - jq;
                const bool neg_in = (lm >= 0) && (lm % N == 0) && (lm / N < M);
                if (k >= 0 || !neg_in) {
                    p = k >= 0 ? k : -k;
                    pk ap = mk(0.f, 0.f), an = mk(0.f, 0.f);
                    const int64_t lp = p - jq, ln = -p - jq;
#pragma unroll
                    for (int l2 = 0; l2 < 4; ++l2) {
                        if (l2 < M && lp == (int64_t)l2 * N) ap = v[l2];
                        if (l2 < M && ln == (int64_t)l2 * N) an = v[l2];
                    }
                    val = f2(mul(add(ap, pkx::conj(an)), bc(0.5f)));
                }
            }
            if (p >= 0) Xl[((int)(p % N1) == res[0] ? 0 : 1) * xl + p / N1] = val;
        }
    }
#endif
    __syncthreads();
    // -- C: inverse step 1, 4 FFTs (residue r, pair ip) of length S2 over k1: radix 32 x 32 on 128 threads.
    //    k' = res + N1 k1, k1 = i + 32 j.  With S = 2K: k' < K (j < 16) is k = k' (positive);
    //    k' > K (j >= 16) is k = k' - S (negative, Y = conj X[S - k'], w^k = -i w^k'); k' = K
    //    (res = 0, k1 = 512) carries both.  w^{k'} = w^{res + N1 i} e^{2 pi i j / 128}.
    //    Zin(k') = W_{pa}(k) + i W_{pb}(k), W_p(k) = Y(k) w^{k p}, (pa, pb) = (2 ip, 2 ip + 1).
    if (a.fbt) tab_wait(&tmb);  // complete long ago; every reading thread observes it
    if (tid < 128) {
        const int fi = tid >> 5, i = tid & 31, r = fi >> 1, ip = fi & 1;
        float2 *buf = ib + fi * IB;
        const bool act = r < nres;
        pk x[32];
        if (act) {
            const int rr = res[r];
            const int ro = (rr == 0) ? 0 : ((nres == 1) ? 0 : 1 - r);  // slot of residue N1 - rr
            const float2 *Xp = Xl + r * xl, *Xn = Xl + ro * xl;
#if MCI_FSF_B32
            const pk P1 = P1early;  // w^{res + N1 i}, looked up before phase A
#else
            const pk P1 = mk(a.twL((int64_t)rr + (int64_t)N1 * i));   // w^{res + N1 i}
#endif
            const pk P2 = pkx::cmul(P1, P1), P3 = pkx::cmul(P2, P1);
#if MCI_FSF_B32
            // (the factors e^{2 pi i e j / 128} are compile-time constants: immediates of the packed
            // multiplies instead of shared-memory table reads)
            cl::static_for<0, 32>([&](auto jc) {
                constexpr int j = decltype(jc)::value;
                const int k1 = i + 32 * j;
                const pk w1 = pkx::cmul(fsf::c128<j>(), P1);           // w^{k'} = w^{res + N1 i} e^{2 pi i j / 128}
                pk acc;
                if (j < 16) {  // positive frequencies: Y = X[k1] (slot r)
                    const pk X = mk(Xp[k1]);
                    if (ip == 0) {
                        acc = add_rot<1>(X, pkx::cmul(X, w1));  // X + i X w
                    } else {
                        const pk w2 = pkx::cmul(fsf::c128<2 * j>(), P2), w3 = pkx::cmul(fsf::c128<3 * j>(), P3);
                        acc = add_rot<1>(pkx::cmul(X, w2), pkx::cmul(X, w3));
                    }
                } else {  // negative frequencies: Y = conj X[S - k'] (slot ro)
                    const int idx = (rr == 0) ? (N1 - k1) : (N1 - 1 - k1);
                    const pk Xc = pkx::conj(mk(Xn[idx]));
                    if (ip == 0) {
                        acc = add(Xc, pkx::cmul(Xc, w1));  // conj X + i conj X (-i w)
                    } else {
                        const pk w2 = pkx::cmul(fsf::c128<2 * j>(), P2), w3 = pkx::cmul(fsf::c128<3 * j>(), P3);
                        acc = mul(add(pkx::cmul(Xc, w2), pkx::cmul(Xc, w3)), bc(-1.f));
                    }
                    if (rr == 0 && k1 == 512) {  // k' = K: add the k = +K term, Y = X[K]
                        const pk X = mk(Xp[512]);
                        if (ip == 0) {
                            acc = add(acc, add_rot<1>(X, pkx::cmul(X, w1)));
                        } else {
                            const pk w2 = pkx::cmul(fsf::c128<2 * j>(), P2), w3 = pkx::cmul(fsf::c128<3 * j>(), P3);
                            acc = add(acc, add_rot<1>(pkx::cmul(X, w2), pkx::cmul(X, w3)));
                        }
                    }
                }
                x[j] = acc;
            });
#else
#pragma unroll
            for (int j = 0; j < 32; ++j) {
                const int k1 = i + 32 * j;
                const pk c1 = mk(tw128[j]);                            // e^{2 pi i j / 128}
                const pk w1 = pkx::cmul(P1, c1);                         // w^{k'}
                pk acc;
                if (j < 16) {  // positive frequencies: Y = X[k1] (slot r)
                    const pk X = mk(Xp[k1]);
                    if (ip == 0) {
                        acc = add_rot<1>(X, pkx::cmul(X, w1));  // X + i X w
                    } else {
                        const pk w2 = pkx::cmul(P2, mk(tw128[32 + j])), w3 = pkx::cmul(P3, mk(tw128[64 + j]));
                        acc = add_rot<1>(pkx::cmul(X, w2), pkx::cmul(X, w3));
                    }
                } else {  // negative frequencies: Y = conj X[S - k'] (slot ro)
                    const int idx = (rr == 0) ? (N1 - k1) : (N1 - 1 - k1);
                    const pk Xc = pkx::conj(mk(Xn[idx]));
                    if (ip == 0) {
                        acc = add(Xc, pkx::cmul(Xc, w1));  // conj X + i conj X (-i w)
                    } else {
                        const pk w2 = pkx::cmul(P2, mk(tw128[32 + j])), w3 = pkx::cmul(P3, mk(tw128[64 + j]));
                        acc = mul(add(pkx::cmul(Xc, w2), pkx::cmul(Xc, w3)), bc(-1.f));
                    }
                    if (rr == 0 && k1 == 512) {  // k' = K: add the k = +K term, Y = X[K]
                        const pk X = mk(Xp[512]);
                        if (ip == 0) {
                            acc = add(acc, add_rot<1>(X, pkx::cmul(X, w1)));
                        } else {
                            const pk w2 = pkx::cmul(P2, mk(tw128[32 + j])), w3 = pkx::cmul(P3, mk(tw128[64 + j]));
                            acc = add(acc, add_rot<1>(pkx::cmul(X, w2), pkx::cmul(X, w3)));
                        }
                    }
                }
                x[j] = acc;
            }
#endif
            dft<32, 1>(x);
#pragma unroll
            for (int j = 0; j < 32; ++j) buf[pad5(32 * i + j)] = f2(x[j]);
        }
        __syncthreads();
        if (act) {
#pragma unroll
            for (int j = 0; j < 32; ++j) x[j] = mk(buf[pad5(i + 32 * j)]);
#pragma unroll
            for (int j = 1; j < 32; ++j)
                x[j] = pkx::cmul(x[j], pkx::conj(mk(a.fbt ? __ldg(gt32 + j * 32 + i) : __ldg(a.twF + ((j * i) & 1023)))));
            dft<32, 1>(x);
            // twiddle e^{2 pi i res u / S}, u = i + 32 j: base(i) * E[j], E[j] = e^{2 pi i 32 res j / S}
            const pk B = mk(a.twS((int64_t)res[r] * i));
            const float2 *E = twE + r * 32;
            float2 *urow = reinterpret_cast<float2 *>(a.Uw) + ((sl * a.npi + ip) * N1 + res[r]) * (int64_t)S2;
#pragma unroll
            for (int j = 0; j < 32; ++j) urow[i + 32 * j] = f2(pkx::cmul(x[j], pkx::cmul(B, mk(E[j]))));
        }
    }
}

// ---- IC: 16 FFTs (pair ip, 8 consecutive u) of length N1 over k2; output runs of 128 B ----------
// lane = 16 il + 8 ip + t: butterfly i = 2 warp + il
// COLS = 8 (default): 512 threads, 16 FFTs (8 columns x 2 residue pairs), 143 KB of shared memory: one
// CTA per SM (measured 3.85 TB/s, lg_throttle 46 % of the stall samples at 25 % occupancy).  COLS = 4
// (MCI_FS_IC_COLS=4, A/B): 256 threads, 8 FFTs, 76 KB, three CTAs per SM in different phases, but loads
// in 32-byte runs and stores in 64-byte runs instead of 64 / 128: measured slower (0.362 vs 0.325 ms).
template <int COLS>
__global__ void __launch_bounds__(64 * COLS, COLS == 4 ? 3 : 1) mci_fsf_ic(const FSArgs<float> a) {
    using namespace fsf;
    using namespace pkx;
    extern __shared__ __align__(16) unsigned char smem[];
    // per-FFT stride: == 1 (mod 16) for 16 FFTs per half-warp, == 2 (mod 16) for 8 FFTs x 2 butterflies
    constexpr int BS = COLS == 8 ? 1056 + 1 : 1056 + 2;
    constexpr int NT = 64 * COLS, LB = COLS == 8 ? 3 : 2;  // lane bits of the column index
    float2 *bufs = reinterpret_cast<float2 *>(smem);
    float2 *tw = bufs + 2 * COLS * BS;  // [32][32] e^{-2 pi i j i/1024}
    __shared__ __align__(8) uint64_t tmb;
    if (a.fbt) {
        if (threadIdx.x == 0) tab_copy(tw, a.fbt + 256, 1024 * 8, &tmb);
    } else {
        for (int q = threadIdx.x; q < 1024; q += NT) tw[q] = __ldg(a.twF + (((q >> 5) * (q & 31)) & 1023));
    }
    __syncthreads();
    const int ntiles = S2 / COLS;
    const int tile = blockIdx.x % ntiles;
    const int64_t sl = blockIdx.x / ntiles;
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int t = lane & (COLS - 1), ip = (lane >> LB) & 1, i = (32 / (2 * COLS)) * warp + (lane >> (LB + 1));
    const int u = tile * COLS + t;
    float2 *buf = bufs + (ip * COLS + t) * BS;
    const float2 *ucol = reinterpret_cast<const float2 *>(a.Uw) + (sl * a.npi + ip) * (int64_t)N1 * S2 + u;
    pk x[32];
#pragma unroll
    for (int j = 0; j < 32; ++j) x[j] = mk(ucol[(int64_t)(i + 32 * j) * S2]);
    dft<32, 1>(x);
#pragma unroll
    for (int j = 0; j < 32; ++j) buf[pad5(32 * i + j)] = f2(x[j]);
    __syncthreads();
#pragma unroll
    for (int j = 0; j < 32; ++j) x[j] = mk(buf[pad5(i + 32 * j)]);
    if (a.fbt) tab_wait(&tmb);
#pragma unroll
    for (int j = 1; j < 32; ++j) x[j] = pkx::cmul(x[j], pkx::conj(mk(tw[j * 32 + i])));
    dft<32, 1>(x);
    // y[u + S2 v] = f[4 p2 + 2 ip + {0,1}], p2 = u + S2 v, v = i + 32 j
    float2 *fo = reinterpret_cast<float2 *>(a.f + (a.sig0 + sl) * a.L);
#pragma unroll
    for (int j = 0; j < 32; ++j) {
        const int64_t p2 = u + (int64_t)S2 * (i + 32 * j);
        __stcs(fo + 2 * p2 + ip, f2(x[j]));
    }
}

bool fourstep_fast_ok(const Axis1D &ax) {
    return ax.dtype == MCI_F32 && ax.N / 1024 == fsf::N2 && ax.S / 1024 == fsf::S2 && (ax.M == 3 || ax.M == 4) &&
           ax.R == 4;
}

cudaError_t fourstep_fast_chunk(const FSArgs<float> &a, int64_t ns, cudaStream_t st) {
    using namespace fsf;
    // MCI_FS_FA_COLS (launch time): 16 = the 512-thread FA kernel (64-byte input runs), default 8
    const int fa_cols = getenv("MCI_FS_FA_COLS") ? atoi(getenv("MCI_FS_FA_COLS")) : 8;
    const size_t fa_sm = fa_cols == 16 ? (size_t)(16 * 1057 + 1024) * 8 : (size_t)(8 * (1056 + 2) + 1024) * 8;
    const int64_t xl = a.K / N1 + 2;
    const size_t fb_sm = (size_t)(4 * 1060 + 2 * xl + 96 + 64) * 8;  // ib aliases fb + G
    // MCI_FS_IC_COLS (launch time): 4 = the 256-thread IC kernel (three CTAs per SM; measured slower,
    // config 4 0.362 vs 0.325 ms: its 32-byte read runs cost more than the occupancy returns), default 8
    const int ic_cols = getenv("MCI_FS_IC_COLS") ? atoi(getenv("MCI_FS_IC_COLS")) : 8;
    const size_t ic_sm = ic_cols == 8 ? (size_t)(16 * 1057 + 1024) * 8 : (size_t)(8 * 1058 + 1024) * 8;
    cudaError_t e;
    if ((e = cudaFuncSetAttribute(mci_fsf_fa<8>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)(8 * 1058 + 1024) * 8))) return e;
    if ((e = cudaFuncSetAttribute(mci_fsf_fa<16>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)(16 * 1057 + 1024) * 8))) return e;
    if ((e = cudaFuncSetAttribute(mci_fsf_fb, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)fb_sm))) return e;
    if ((e = cudaFuncSetAttribute(mci_fsf_ic<8>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)(16 * 1057 + 1024) * 8))) return e;
    if ((e = cudaFuncSetAttribute(mci_fsf_ic<4>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)(8 * 1058 + 1024) * 8))) return e;
    if (fa_cols == 16) mci_fsf_fa<16><<<(unsigned)(ns * a.npair * (N2 / 16)), 512, fa_sm, st>>>(a);
    else mci_fsf_fa<8><<<(unsigned)(ns * a.npair * (N2 / 8)), 256, fa_sm, st>>>(a);
    mci_fsf_fb<<<(unsigned)(ns * (N1 / 2 + 1)), 128, fb_sm, st>>>(a);
    if (ic_cols == 8) mci_fsf_ic<8><<<(unsigned)(ns * (S2 / 8)), 512, ic_sm, st>>>(a);
    else mci_fsf_ic<4><<<(unsigned)(ns * (S2 / 4)), 256, ic_sm, st>>>(a);
    return cudaGetLastError();
}

}  // namespace mci
