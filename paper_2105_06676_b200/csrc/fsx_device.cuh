// Device building blocks for the sm_100a StencilFFT-P path.
//
//   * fp64 complex helpers on double2 (re, im)
//   * register-resident radix-2/4/8/16 DFT butterflies with folded constants
//   * LineFFT<N, SIGN>: a Stockham autosort FFT of one pow2 line executed by
//     N/R threads (R = min(16, N) elements per thread held in registers);
//     the passes exchange through a bank-swizzled shared-memory line buffer.
//
// Conventions follow the reference FFT (proj/src/fft.cpp:143-155): forward is
// X[k] = sum_n x[n] exp(-2 pi i n k / N), unnormalized; SIGN = -1 forward,
// +1 inverse (normalization is folded into the spectral multiply by the
// callers, see fsx_kernels.cu).
#pragma once

#include <cstdint>
#include <type_traits>
#include <cuda_runtime.h>

#include "fsx_kernels.h"

namespace fsx {

using i64 = long long;
using u64 = unsigned long long;

__host__ __device__ constexpr int ilog2c(long long n) { return n <= 1 ? 0 : 1 + ilog2c(n >> 1); }

// ------------------------------------------------------------------ complex
__device__ __forceinline__ double2 cadd(double2 a, double2 b) { return make_double2(a.x + b.x, a.y + b.y); }
__device__ __forceinline__ double2 csub(double2 a, double2 b) { return make_double2(a.x - b.x, a.y - b.y); }
__device__ __forceinline__ double2 cmul(double2 a, double2 b) {
    return make_double2(fma(a.x, b.x, -a.y * b.y), fma(a.x, b.y, a.y * b.x));
}
// a * conj(b)
__device__ __forceinline__ double2 cmulc(double2 a, double2 b) {
    return make_double2(fma(a.x, b.x, a.y * b.y), fma(a.y, b.x, -a.x * b.y));
}
__device__ __forceinline__ double2 cconj(double2 a) { return make_double2(a.x, -a.y); }
__device__ __forceinline__ double2 cscale(double2 a, double s) { return make_double2(a.x * s, a.y * s); }
// multiply by SIGN * i   (SIGN = -1: -i, +1: +i)
template <int SIGN>
__device__ __forceinline__ double2 cmul_si(double2 a) {
    return SIGN < 0 ? make_double2(a.y, -a.x) : make_double2(-a.y, a.x);
}
// a * w^SIGN-direction: forward uses the table value w, inverse its conjugate
template <int SIGN>
__device__ __forceinline__ double2 ctw(double2 a, double2 w) {
    return SIGN < 0 ? cmul(a, w) : cmulc(a, w);
}

// The same helpers on float2 (the fp32 arithmetic of the fp32 mode's fused
// pass; the line-FFT engine below is templated on the complex type CT).
__device__ __forceinline__ float2 cadd(float2 a, float2 b) { return make_float2(a.x + b.x, a.y + b.y); }
__device__ __forceinline__ float2 csub(float2 a, float2 b) { return make_float2(a.x - b.x, a.y - b.y); }
__device__ __forceinline__ float2 cmul(float2 a, float2 b) {
    return make_float2(fmaf(a.x, b.x, -a.y * b.y), fmaf(a.x, b.y, a.y * b.x));
}
__device__ __forceinline__ float2 cmulc(float2 a, float2 b) {
    return make_float2(fmaf(a.x, b.x, a.y * b.y), fmaf(a.y, b.x, -a.x * b.y));
}
__device__ __forceinline__ float2 cconj(float2 a) { return make_float2(a.x, -a.y); }
__device__ __forceinline__ float2 cscale(float2 a, float s) { return make_float2(a.x * s, a.y * s); }
template <int SIGN>
__device__ __forceinline__ float2 cmul_si(float2 a) {
    return SIGN < 0 ? make_float2(a.y, -a.x) : make_float2(-a.y, a.x);
}
template <int SIGN>
__device__ __forceinline__ float2 ctw(float2 a, float2 w) {
    return SIGN < 0 ? cmul(a, w) : cmulc(a, w);
}
// fp64 <-> fp32 complex conversions (widen exactly, narrow to nearest)
__device__ __forceinline__ double2 to_d2(double2 a) { return a; }
__device__ __forceinline__ double2 to_d2(float2 a) { return make_double2(a.x, a.y); }
template <class TO>
__device__ __forceinline__ TO from_d2(double2 a) {
    if constexpr (sizeof(TO) == 16) return a;
    else return make_float2((float)a.x, (float)a.y);
}

template <class CT>
struct CScalar;
template <>
struct CScalar<double2> {
    using T = double;
    __device__ __forceinline__ static double2 make(double x, double y) { return make_double2(x, y); }
};
template <>
struct CScalar<float2> {
    using T = float;
    __device__ __forceinline__ static float2 make(float x, float y) { return make_float2(x, y); }
};

// compile-time unrolled loop: f(std::integral_constant<int, I>) for I in [B, E)
template <int B, int E, class F>
__device__ __forceinline__ void static_for(F&& f) {
    if constexpr (B < E) {
        f(std::integral_constant<int, B>{});
        static_for<B + 1, E>(f);
    }
}

// ------------------------------------------------------------------ constant twiddles
// cos(2 pi j / 32) for j = 0..8 (quarter wave); everything else by symmetry.
__device__ __forceinline__ constexpr double cos32q(int j) {
    return j == 0 ? 1.0
         : j == 1 ? 0.98078528040323044913
         : j == 2 ? 0.92387953251128673848
         : j == 3 ? 0.83146961230254523708
         : j == 4 ? 0.70710678118654752440
         : j == 5 ? 0.55557023301960222474
         : j == 6 ? 0.38268343236508977173
         : j == 7 ? 0.19509032201612826785
                  : 0.0;
}

// Multiply a by exp(SIGN * 2 pi i * J / R) with J, R compile-time (R divides
// 32); the trivial angles are folded to swaps/negations.
template <int J, int R, int SIGN, class CT>
__device__ __forceinline__ CT cmul_const(CT a) {
    static_assert(32 % R == 0, "cmul_const: R must divide 32");
    using T = typename CScalar<CT>::T;
    constexpr int j32 = ((J * 32 / R) % 32 + 32) % 32;  // angle in 32nds
    if constexpr (j32 == 0) return a;
    else if constexpr (j32 == 16) return CScalar<CT>::make(-a.x, -a.y);
    else if constexpr (j32 == 8) return cmul_si<SIGN>(a);
    else if constexpr (j32 == 24) return cmul_si<-SIGN>(a);
    else {
        // exp(i theta) with theta = 2 pi j32 / 32 (then conj for SIGN = -1)
        constexpr int q = j32 % 8, quad = j32 / 8;
        constexpr double c0 = cos32q(q), s0 = cos32q(8 - q);  // cos, sin in the first quadrant
        constexpr T c = (T)(quad == 0 ? c0 : quad == 1 ? -s0 : quad == 2 ? -c0 : s0);
        constexpr T s = (T)(quad == 0 ? s0 : quad == 1 ? c0 : quad == 2 ? -s0 : -c0);
        constexpr T ss = SIGN < 0 ? -s : s;
        if constexpr (q == 4) {
            // c, s = +-1/sqrt2
            return CScalar<CT>::make(c * a.x - ss * a.y, c * a.y + ss * a.x);
        } else {
            return CScalar<CT>::make(fma(c, a.x, -ss * a.y), fma(c, a.y, ss * a.x));
        }
    }
}

// ------------------------------------------------------------------ DFT butterflies
// In-place DFT of v[0..R) in natural order.  Written as Cooley-Tukey
// R = R1 * R2 with the inner twiddles folded at compile time.
template <int R, int SIGN>
struct Dft;

template <int SIGN>
struct Dft<1, SIGN> {
    template <class CT>
    __device__ __forceinline__ static void run(CT*) {}
};

template <int SIGN>
struct Dft<2, SIGN> {
    template <class CT>
    __device__ __forceinline__ static void run(CT* v) {
        const CT a = v[0], b = v[1];
        v[0] = cadd(a, b);
        v[1] = csub(a, b);
    }
};

template <int SIGN>
struct Dft<4, SIGN> {
    template <class CT>
    __device__ __forceinline__ static void run(CT* v) {
        const CT t0 = cadd(v[0], v[2]), t1 = csub(v[0], v[2]);
        const CT t2 = cadd(v[1], v[3]), t3 = cmul_si<SIGN>(csub(v[1], v[3]));
        v[0] = cadd(t0, t2);
        v[2] = csub(t0, t2);
        v[1] = cadd(t1, t3);
        v[3] = csub(t1, t3);
    }
};

// R = R1 * R2: X[k1 + R1 k2] = sum_n2 W_R2^(n2 k2) W_R^(n2 k1) sum_n1 x[R2 n1 + n2] W_R1^(n1 k1)
template <int R1, int R2, int SIGN>
struct DftCT {
    static constexpr int R = R1 * R2;
    template <int N2, int K1, class CT>
    __device__ __forceinline__ static void tw(CT (&y)[R2][R1]) {
        if constexpr (N2 < R2) {
            if constexpr (K1 < R1) {
                y[N2][K1] = cmul_const<N2 * K1, R, SIGN>(y[N2][K1]);
                tw<N2, K1 + 1, CT>(y);
            } else {
                tw<N2 + 1, 0, CT>(y);
            }
        }
    }
    template <class CT>
    __device__ __forceinline__ static void run(CT* v) {
        CT y[R2][R1];
#pragma unroll
        for (int n2 = 0; n2 < R2; ++n2) {
#pragma unroll
            for (int n1 = 0; n1 < R1; ++n1) y[n2][n1] = v[R2 * n1 + n2];
            Dft<R1, SIGN>::run(y[n2]);
        }
        tw<0, 0, CT>(y);
#pragma unroll
        for (int k1 = 0; k1 < R1; ++k1) {
            CT z[R2];
#pragma unroll
            for (int n2 = 0; n2 < R2; ++n2) z[n2] = y[n2][k1];
            Dft<R2, SIGN>::run(z);
#pragma unroll
            for (int k2 = 0; k2 < R2; ++k2) v[k1 + R1 * k2] = z[k2];
        }
    }
};

template <int SIGN>
struct Dft<8, SIGN> {
    template <class CT>
    __device__ __forceinline__ static void run(CT* v) { DftCT<2, 4, SIGN>::run(v); }
};
template <int SIGN>
struct Dft<16, SIGN> {
    template <class CT>
    __device__ __forceinline__ static void run(CT* v) { DftCT<4, 4, SIGN>::run(v); }
};

// ------------------------------------------------------------------ radix-16 with the pass twiddles folded in
// X[k] = sum_u a[u] w^u W16^(u k), w = the pass twiddle of this item (the
// table value for SIGN = -1, its conjugate for +1), as four radix-2 layers in
// which the twiddle rides on the butterfly: with u = u' + 8 b,
//   X[p + 2 k'] = sum_u' (w W16^p)^u' W8^(u' k') (a[u'] + (-1)^p w^8 a[u' + 8]),
// an 8-point transform of the same form with base twiddle w W16^p, and so on.
// Layer 1 multiplies by w^8, layer 2 by w^4 (SIGN i)^p, layer 3 by
// w^2 W8^p (SIGN i)^p', layer 4 by w W16^(p + 2 p') (SIGN i)^p''.  Each
// butterfly is s = a + m b (4 FMA), d = 2 a - s (2 FMA): 32 x 6 + 4 constant
// products = 208 FP64 instructions against 264 for twiddles (15 products + 11
// derived powers) followed by the plain transform.  Only w, w^2, w^4, w^8 are
// needed -- the four values the gathered tables hold.  Output in natural order
// (the bit reversal is a compile-time renaming).
#ifndef FSX_FUSED16
#define FSX_FUSED16 0  // 1: measured slower (cfg3 0.983 -> 1.017 ms, r04e): fewer FP64 instructions, longer FMA chains
#endif
template <class CT>
__device__ __forceinline__ void bfly_tw(CT& a, CT& b, typename CScalar<CT>::T mx, typename CScalar<CT>::T my) {
    using T = typename CScalar<CT>::T;
    const T sx = fma(mx, b.x, fma(-my, b.y, a.x));
    const T sy = fma(mx, b.y, fma(my, b.x, a.y));
    b = CScalar<CT>::make(fma((T)2, a.x, -sx), fma((T)2, a.y, -sy));
    a = CScalar<CT>::make(sx, sy);
}

template <int SIGN, class CT>
__device__ __forceinline__ void dft16_tw_fused(CT (&a)[16], CT w1, CT w2, CT w4, CT w8) {
    if constexpr (SIGN > 0) {
        w1 = cconj(w1);
        w2 = cconj(w2);
        w4 = cconj(w4);
        w8 = cconj(w8);
    }
    // layer 1: (u, u + 8), multiplier w^8
#pragma unroll
    for (int u = 0; u < 8; ++u) bfly_tw(a[u], a[u + 8], w8.x, w8.y);
    // layer 2: group p, (u, u + 4), multiplier w^4 (SIGN i)^p
    {
        const CT m1 = cmul_si<SIGN>(w4);
#pragma unroll
        for (int u = 0; u < 4; ++u) {
            bfly_tw(a[u], a[u + 4], w4.x, w4.y);
            bfly_tw(a[8 + u], a[12 + u], m1.x, m1.y);
        }
    }
    // layer 3: group (p, p'), (u, u + 2), multiplier w^2 W8^p (SIGN i)^p'
    {
        const CT m0 = w2, m1 = cmul_const<1, 8, SIGN>(w2);
        const CT m0i = cmul_si<SIGN>(m0), m1i = cmul_si<SIGN>(m1);
#pragma unroll
        for (int u = 0; u < 2; ++u) {
            bfly_tw(a[u], a[u + 2], m0.x, m0.y);
            bfly_tw(a[4 + u], a[6 + u], m0i.x, m0i.y);
            bfly_tw(a[8 + u], a[10 + u], m1.x, m1.y);
            bfly_tw(a[12 + u], a[14 + u], m1i.x, m1i.y);
        }
    }
    // layer 4: group (p, p', p''), (0, 1), multiplier w W16^(p + 2 p') (SIGN i)^p''
    {
        const CT n0 = w1, n1 = cmul_const<1, 16, SIGN>(w1), n2 = cmul_const<2, 16, SIGN>(w1),
                 n3 = cmul_const<3, 16, SIGN>(w1);
        const CT n0i = cmul_si<SIGN>(n0), n1i = cmul_si<SIGN>(n1), n2i = cmul_si<SIGN>(n2), n3i = cmul_si<SIGN>(n3);
        // index 8 p + 4 p' + 2 p'': j = p + 2 p'
        bfly_tw(a[0], a[1], n0.x, n0.y);
        bfly_tw(a[2], a[3], n0i.x, n0i.y);
        bfly_tw(a[4], a[5], n2.x, n2.y);
        bfly_tw(a[6], a[7], n2i.x, n2i.y);
        bfly_tw(a[8], a[9], n1.x, n1.y);
        bfly_tw(a[10], a[11], n1i.x, n1i.y);
        bfly_tw(a[12], a[13], n3.x, n3.y);
        bfly_tw(a[14], a[15], n3i.x, n3i.y);
    }
    // position 8 p + 4 p' + 2 p'' + p''' holds X[p + 2 p' + 4 p'' + 8 p''']
    CT t;
    t = a[1], a[1] = a[8], a[8] = t;
    t = a[2], a[2] = a[4], a[4] = t;
    t = a[3], a[3] = a[12], a[12] = t;
    t = a[5], a[5] = a[10], a[10] = t;
    t = a[7], a[7] = a[14], a[14] = t;
    t = a[11], a[11] = a[13], a[13] = t;
}

// ------------------------------------------------------------------ smem swizzle
// 16-byte elements: 8 per 128-byte bank row.  XOR the low 3 bits with bits
// 3..5 and 4..6 so the Stockham scatter strides 2, 4, 8, 16 and the unit
// stride gathers are all conflict-free per quarter warp.
__device__ __forceinline__ int swz(int p) { return p ^ (((p >> 3) ^ (p >> 4)) & 7); }

// ------------------------------------------------------------------ line FFT
// One pow2 line of N complex values, transformed by TPL = N/R threads.
// Thread t holds v[q] = x[t + q * TPL] on entry and X[t + q * TPL] on exit.
// `line` is this line's shared-memory buffer (N elements, swizzled index);
// `tw` is the twiddle table for N: tw[x] = exp(-2 pi i x / N), x < N.
// Every thread of the CTA must call run() together (it contains
// __syncthreads); lines of one CTA are transformed concurrently.
//
// PF = true hoists the next pass's twiddle loads above the exchange barrier
// (their L1/L2 latency then overlaps the barrier wait and the shared-memory
// round trip); it costs R-1 extra live double2 registers, so it is used by
// the persistent kernels that run 8 warps per SM with the full register file.
//
// PAIR = true (only meaningful when the last pass has radix 8, i.e. two
// items per thread) gives the last pass the items {t, N/8 - t} (thread 0:
// {0, N/16}) instead of {t, t + TPL}: every output position p of the thread
// then has its mirror N - p in the same thread, which lets a real-to-complex
// split run in registers.  Output convention with PAIR: v[i + u * 2] holds
// X[item(t, i) + u * N / 8].
// FT (bit S set: pass S): read every twiddle of that pass from the gathered
// table (no derived products: fewer FP64 instructions, more L1 loads).
// NB > 0: the exchanges synchronize NB-thread groups with named barriers
// (id 1 + threadIdx.x / NB) instead of the whole CTA, so independent groups
// of one CTA (e.g. the two half-columns of the 8192-point pass) drift apart.
template <int NB>
__device__ __forceinline__ void group_sync() {
    if constexpr (NB == 0) __syncthreads();
    else asm volatile("bar.sync %0, %1;\n" ::"r"(1 + (int)(threadIdx.x / NB)), "n"(NB) : "memory");
}

// CT: the complex element type (double2; float2 for the fp32 mode's fused
// pass, with a float2 copy of the twiddle tables).
// LPF = true: the four base twiddles (W^1, W^2, W^4, W^8) of the next radix-16
// derived-twiddle pass are loaded before the exchange barrier (8 extra live
// registers instead of PF's 30), so their latency overlaps the barrier wait.
template <int N, int SIGN, bool PF = false, bool PAIR = false, int FT = 0, int NB = 0, class CT = double2,
          bool LPF = false>
struct LineFFT {
    static constexpr int LOGN = ilog2c(N);
    static constexpr int R = N < 16 ? N : 16;
    static constexpr int TPL = N / R;
    static constexpr int P16 = N < 16 ? 0 : LOGN / 4;
    static constexpr int REM = N < 16 ? LOGN : LOGN % 4;
    static constexpr int NPASS = P16 + (REM > 0 ? 1 : 0);
    static constexpr int EXCHANGES = NPASS - 1;

    template <int S>
    __host__ __device__ static constexpr int radix() { return S < P16 ? 16 : (1 << REM); }
    template <int S>
    __host__ __device__ static constexpr int ns() {
        if constexpr (S == 0) return 1;
        else return ns<S - 1>() * radix<S - 1>();
    }
    static constexpr bool PAIRED = PAIR && NPASS >= 2 && R / (1 << REM) == 2 && REM == 3;

    // index j of item i of thread t in pass S
    template <int S>
    __device__ __forceinline__ static int item(int t, int i) {
        if constexpr (PAIRED && S == NPASS - 1) return i == 0 ? t : (t == 0 ? TPL : 2 * TPL - t);
        else return t + i * TPL;
    }

    // twiddles of pass S for this thread: w[i * r + u] = W_{Ns r}^{u k(i)}, u >= 1,
    // from the per-pass gathered table (kPassTabBase: row u - 1, contiguous in
    // k, so a warp's load touches consecutive lines instead of one line per
    // thread).  Without FT only the power-of-two exponents u = 1, 2, 4, 8 are
    // read; the others are products of at most two loaded/derived values
    // (<= 3 roundings).
    template <int S>
    __device__ __forceinline__ static void load_tw(int t, const CT* __restrict__ tw, CT (&w)[R]) {
        constexpr int r = radix<S>();
        constexpr int Ns = ns<S>();
        constexpr int C = R / r;
        // Last pass (Ns r = N, several items per thread): item i sits at
        // t + i N/16, so W_N^(u (t + i N/16)) = W_N^(u t) W_16^(u i) -- only
        // item 0 is read, the others are exact-constant rotations of it.
        constexpr bool LAST_DERIVE = Ns * r == N && C > 1 && !(PAIRED && S == NPASS - 1);
        if constexpr (Ns > 1) {
#pragma unroll
            for (int i = 0; i < (LAST_DERIVE ? 1 : C); ++i) {
                const int k = item<S>(t, i) & (Ns - 1);
                CT* wi = w + i * r;
                const CT* pt = tw + (kPassTabBase + 15 * N + 16 * Ns);  // tw = tw_all + N
                if constexpr (((FT >> S) & 1) != 0) {
#pragma unroll
                    for (int u = 1; u < r; ++u) wi[u] = __ldg(pt + (u - 1) * Ns + k);
                    continue;
                }
#pragma unroll
                for (int u = 1; u < r; u <<= 1) wi[u] = __ldg(pt + (u - 1) * Ns + k);
                if constexpr (r >= 4) wi[3] = cmul(wi[1], wi[2]);
                if constexpr (r >= 8) {
                    wi[5] = cmul(wi[1], wi[4]);
                    wi[6] = cmul(wi[2], wi[4]);
                    wi[7] = cmul(wi[3], wi[4]);
                }
                if constexpr (r >= 16) {
#pragma unroll
                    for (int u = 9; u < 16; ++u) wi[u] = cmul(wi[u - 8], wi[8]);
                }
            }
            if constexpr (LAST_DERIVE) {
                static_for<1, C>([&](auto I) {
                    constexpr int i = decltype(I)::value;
                    static_for<1, r>([&](auto U) {
                        constexpr int u = decltype(U)::value;
                        w[i * r + u] = cmul_const<u * i, 16, -1>(w[u]);
                    });
                });
            }
        }
    }

    // One radix-16 item (C == 1) with derived twiddles, applied as they are
    // formed: W^1, W^2, W^4, W^8 are read, and every product is consumed right
    // away, so at most a handful of twiddles are live (the 15-entry w[] array
    // of the generic path costs 60 registers and spilled at 128).  The products
    // are the generic path's (w3 = w1 w2, w5 = w1 w4, w6 = w2 w4, w7 = w3 w4,
    // w(u + 8) = w(u) w8): bitwise the same results.
    template <int S>
    __device__ __forceinline__ static void tw16_base(int t, const CT* __restrict__ tw, CT (&b)[4]) {
        constexpr int Ns = ns<S>();
        const int k = item<S>(t, 0) & (Ns - 1);
        const CT* pt = tw + (kPassTabBase + 15 * N + 16 * Ns) + k;
        b[0] = __ldg(pt);
        b[1] = __ldg(pt + Ns);
        b[2] = __ldg(pt + 3 * Ns);
        b[3] = __ldg(pt + 7 * Ns);
    }

    template <int S>
    __device__ __forceinline__ static void tw16_apply(CT (&a)[16], int t, const CT* __restrict__ tw,
                                                      const CT* pre = nullptr) {
        CT b[4];
        if (pre) {
#pragma unroll
            for (int i = 0; i < 4; ++i) b[i] = pre[i];
        } else {
            tw16_base<S>(t, tw, b);
        }
        const CT w1 = b[0], w2 = b[1], w4 = b[2], w8 = b[3];
        a[1] = ctw<SIGN>(a[1], w1);
        a[2] = ctw<SIGN>(a[2], w2);
        a[4] = ctw<SIGN>(a[4], w4);
        a[8] = ctw<SIGN>(a[8], w8);
        a[9] = ctw<SIGN>(a[9], cmul(w1, w8));
        a[10] = ctw<SIGN>(a[10], cmul(w2, w8));
        a[12] = ctw<SIGN>(a[12], cmul(w4, w8));
        const CT w3 = cmul(w1, w2);
        a[3] = ctw<SIGN>(a[3], w3);
        a[11] = ctw<SIGN>(a[11], cmul(w3, w8));
        const CT w5 = cmul(w1, w4);
        a[5] = ctw<SIGN>(a[5], w5);
        a[13] = ctw<SIGN>(a[13], cmul(w5, w8));
        const CT w6 = cmul(w2, w4);
        a[6] = ctw<SIGN>(a[6], w6);
        a[14] = ctw<SIGN>(a[14], cmul(w6, w8));
        const CT w7 = cmul(w3, w4);
        a[7] = ctw<SIGN>(a[7], w7);
        a[15] = ctw<SIGN>(a[15], cmul(w7, w8));
    }

    template <int S>
    __host__ __device__ static constexpr bool inc_pass() {
        return !PF && radix<S>() == 16 && R / radix<S>() == 1 && ns<S>() > 1 && ((FT >> S) & 1) == 0 &&
               !(PAIRED && S == NPASS - 1);
    }

    template <int S>
    __device__ __forceinline__ static void pass(CT (&v)[R], int t, CT* line, const CT* __restrict__ tw, CT (&w)[R],
                                                const CT* pre = nullptr) {
        constexpr int r = radix<S>();
        constexpr int Ns = ns<S>();
        constexpr int C = R / r;
        // radix-16 items with derived twiddles: formed and applied on the fly
        constexpr bool INC = inc_pass<S>();
        if constexpr (!PF && !INC) load_tw<S>(t, tw, w);
#pragma unroll
        for (int i = 0; i < C; ++i) {
            CT a[r];
#pragma unroll
            for (int u = 0; u < r; ++u) a[u] = v[i + u * C];
            if constexpr (INC && FSX_FUSED16 != 0) {
                CT b[4];
                if (pre) {
#pragma unroll
                    for (int q = 0; q < 4; ++q) b[q] = pre[q];
                } else {
                    tw16_base<S>(t, tw, b);
                }
                dft16_tw_fused<SIGN>(a, b[0], b[1], b[2], b[3]);
            } else {
                if constexpr (INC) {
                    tw16_apply<S>(a, t, tw, pre);
                } else if constexpr (Ns > 1) {
#pragma unroll
                    for (int u = 1; u < r; ++u) a[u] = ctw<SIGN>(a[u], w[i * r + u]);
                }
                Dft<r, SIGN>::run(a);
            }
#pragma unroll
            for (int u = 0; u < r; ++u) v[i + u * C] = a[u];
        }
        if constexpr (S + 1 < NPASS) {
            if constexpr (PF) load_tw<S + 1>(t, tw, w);
            CT nb[4];
            constexpr bool LP = LPF && inc_pass<S + 1>();
            if constexpr (LP) tw16_base<S + 1>(t, tw, nb);
            group_sync<NB>();
#pragma unroll
            for (int i = 0; i < C; ++i) {
                const int j = t + i * TPL;
                const int k = j & (Ns - 1);
                const int base = (j - k) * r + k;
#pragma unroll
                for (int u = 0; u < r; ++u) line[swz(base + u * Ns)] = v[i + u * C];
            }
            group_sync<NB>();
            constexpr int r2 = radix<S + 1>();
            constexpr int C2 = R / r2;
#pragma unroll
            for (int i = 0; i < C2; ++i) {
                const int j = item<S + 1>(t, i);
#pragma unroll
                for (int u = 0; u < r2; ++u) v[i + u * C2] = line[swz(j + u * (N / r2))];
            }
            if constexpr (LP) pass<S + 1>(v, t, line, tw, w, nb);
            else pass<S + 1>(v, t, line, tw, w);
        }
    }

    __device__ __forceinline__ static void run(CT (&v)[R], int t, CT* line, const CT* __restrict__ tw) {
        CT w[R];
        if constexpr (NPASS > 0) pass<0>(v, t, line, tw, w);
    }
};


}  // namespace fsx
