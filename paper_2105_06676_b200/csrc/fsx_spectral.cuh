// Device-side symbol / power helpers shared by the fused spectral passes.
//
// lam(k) = sum_taps c * exp(+2 pi i sum_a k_a o_a / n_a) is the transform of
// the reference's generator column (proj/src/spectrum.cpp:21-45) evaluated
// analytically with exact integer phase reduction; the power is the
// reference's binary exponentiation loop (proj/src/spectrum.cpp:53-64).
#pragma once

#include "fsx_device.cuh"
#include "fsx_kernels.h"

namespace fsx {

// exp(-2 pi i x / n) for x in [0, n) from a (two-level) phase table
__device__ __forceinline__ double2 phase_at(const PhaseTable& t, i64 x) {
    if (t.shift == 0) return __ldg(t.lo + x);
    return cmul(__ldg(t.hi + (x >> t.shift)), __ldg(t.lo + (x & t.mask)));
}

// any lane's `bad` sets the solve's non-finite flag (realize_checked)
__device__ __forceinline__ void flag_nonfinite(bool bad, Flags* f) {
    const unsigned any = __ballot_sync(0xffffffffu, bad);
    if (any && (threadIdx.x & 31) == 0) atomicOr(&f->nonfinite, 1u);
}

// exp(+2 pi i x / n) for pow2 n from the exact table: conj(tw_all[n + (x mod n)])
__device__ __forceinline__ double2 eplus_tab(const double2* tw_all, i64 n, i64 x) {
    return cconj(__ldg(tw_all + n + (x & (n - 1))));
}

// The product of a finite u with a zero multiplier, as the fused passes form it:
//   real symbol     cscale(u, 0.0 * scale)             = (0 * u.x, 0 * u.y)
//   complex symbol  cscale(cmul((0, 0), u), scale),  cmul = (fma(0, u.x, -(0 * u.y)), fma(0, u.y, 0 * u.x))
// with scale > 0.  Every result is a zero; only its sign depends on u: 0 * x carries x's sign, and a
// sum of two zeros is -0 only when both are.  So the signs follow from u's sign bits alone, without
// touching the FP64 pipe (96 of its instructions per thread in a zero column otherwise).  A non-finite
// u would give NaN in the full evaluation; it cannot hide here, because its whole row and therefore
// the always-evaluated column 0 is non-finite too (the solve raises NumericError either way).
__device__ __forceinline__ double2 zero_products(double2 u, bool real_symbol) {
    const unsigned sx = (unsigned)__double2hiint(u.x), sy = (unsigned)__double2hiint(u.y);
    const unsigned rx = real_symbol ? sx : (sx & ~sy);  // complex: (+-0 of u.x) + (-+0 of u.y)
    const unsigned ry = real_symbol ? sy : (sx & sy);   //          (+-0 of u.y) + (+-0 of u.x)
    return make_double2(__hiloint2double((int)(rx & 0x80000000u), 0), __hiloint2double((int)(ry & 0x80000000u), 0));
}

// e * i^m for m in 0..3 (exact: swaps and sign flips)
__device__ __forceinline__ double2 rot_quarter(double2 e, int m) {
    const double x = (m & 1) ? e.y : e.x, y = (m & 1) ? e.x : e.y;
    return make_double2((m == 1 || m == 2) ? -x : x, (m >= 2) ? -y : y);
}

// exp(+2 pi i og k0 / N) for a thread's 16 frequencies k0 = t + q N/16:
// with q = 4a + b this is e_b * i^(og a), so four table reads give all 16
// (the other twelve are exact quarter turns).  f(q, e) is called per q.
template <int N, class F>
__device__ __forceinline__ void eplus16(const double2* tw_all, int t, i64 og, F&& f) {
    double2 eb[4];
#pragma unroll
    for (int b = 0; b < 4; ++b) eb[b] = eplus_tab(tw_all, N, (i64)(t + b * (N / 16)) * og);
    const int mo = (int)(og & 3);
#pragma unroll
    for (int a = 0; a < 4; ++a) {
        const int m = (mo * a) & 3;
#pragma unroll
        for (int b = 0; b < 4; ++b) f(4 * a + b, rot_quarter(eb[b], m));
    }
}

// |lam|^T < 2^-1100 short cut: below every representable contribution (the
// reference's own repeated squaring underflows to 0 / subnormal there).
__device__ __forceinline__ bool negligible_power(double mag2, u64 T) {
    if (!(mag2 < 1.0)) return false;
    int e;
    const double mant = frexp(mag2, &e);
    const float l2 = (float)e + __log2f((float)mant);
    return l2 * (0.5f * (float)T) < -2200.0f;
}

__device__ __forceinline__ double2 pow_complex(double2 lam, u64 T, double neg_mag2) {
    if (fma(lam.x, lam.x, lam.y * lam.y) < neg_mag2) return make_double2(0.0, 0.0);
    double2 acc = make_double2(1.0, 0.0), sq = lam;
    u64 t = T;
    while (t) {
        if (t & 1) acc = cmul(acc, sq);
        t >>= 1;
        if (t) sq = make_double2(fma(sq.x, sq.x, -sq.y * sq.y), (sq.x + sq.x) * sq.y);
    }
    return acc;
}

// neg_mag2 = 2^(-2200/T) from the host (FusedSymbol): the same short cut as
// negligible_power with one compare instead of frexp + log2
__device__ __forceinline__ double pow_realv(double lam, u64 T, double neg_mag2) {
    if (lam * lam < neg_mag2) return 0.0;
    double acc = 1.0, sq = lam;
    u64 t = T;
    while (t) {
        if (t & 1) acc *= sq;
        t >>= 1;
        if (t) sq *= sq;
    }
    return acc;
}

// Element-parallel versions of pow_realv / pow_complex (the same loop per
// element): the loop over the bits of T is uniform, and CH independent
// elements per step give the FP64 pipe CH-way ILP instead of one latency
// chain per element.  No underflow short cut here: the loop runs for every
// element anyway, and where |lam|^T < 2^-1100 its own product underflows to 0
// (or a subnormal) exactly as the reference's loop does -- the frexp/log2
// test cost ~13 % of the fused pass's issue slots.
template <int R, int CH = R>
__device__ __forceinline__ void pow_real_vec(double (&x)[R], u64 T) {
    static_assert(R % CH == 0, "chunk must divide R");
#pragma unroll
    for (int c = 0; c < R; c += CH) {
        double acc[CH];
#pragma unroll
        for (int q = 0; q < CH; ++q) acc[q] = 1.0;
        u64 t = T;
        while (t) {
            if (t & 1) {
#pragma unroll
                for (int q = 0; q < CH; ++q) acc[q] *= x[c + q];
            }
            t >>= 1;
            if (t) {
#pragma unroll
                for (int q = 0; q < CH; ++q) x[c + q] *= x[c + q];
            }
        }
#pragma unroll
        for (int q = 0; q < CH; ++q) x[c + q] = acc[q];
    }
}

template <int R, int CH = R>
__device__ __forceinline__ void pow_complex_vec(double2 (&x)[R], u64 T) {
    static_assert(R % CH == 0, "chunk must divide R");
#pragma unroll
    for (int c = 0; c < R; c += CH) {
        double2 acc[CH];
#pragma unroll
        for (int q = 0; q < CH; ++q) acc[q] = make_double2(1.0, 0.0);
        u64 t = T;
        while (t) {
            if (t & 1) {
#pragma unroll
                for (int q = 0; q < CH; ++q) acc[q] = cmul(acc[q], x[c + q]);
            }
            t >>= 1;
            if (t) {
#pragma unroll
                for (int q = 0; q < CH; ++q) {
                    const double2 sq = x[c + q];
                    x[c + q] = make_double2(fma(sq.x, sq.x, -sq.y * sq.y), (sq.x + sq.x) * sq.y);
                }
            }
        }
#pragma unroll
        for (int q = 0; q < CH; ++q) x[c + q] = acc[q];
    }
}

// pow_real_vec with the underflow short cut at warp granularity: elements
// with |lam|^2 < neg_mag2 (host: 2^(-2200/T)) are 0; a chunk whose elements
// are negligible in every lane of the warp skips the power loop (a compare
// and a vote instead of the per-element frexp/log2 test).
template <int R, int CH>
__device__ __forceinline__ void pow_real_vec_skip(double (&x)[R], u64 T, double neg_mag2) {
    static_assert(R % CH == 0, "chunk must divide R");
#pragma unroll
    for (int c = 0; c < R; c += CH) {
        bool neg[CH], all = true;
#pragma unroll
        for (int q = 0; q < CH; ++q) {
            neg[q] = x[c + q] * x[c + q] < neg_mag2;
            all &= neg[q];
        }
        if (__all_sync(0xffffffffu, all)) {
#pragma unroll
            for (int q = 0; q < CH; ++q) x[c + q] = 0.0;
            continue;
        }
        double acc[CH];
#pragma unroll
        for (int q = 0; q < CH; ++q) acc[q] = 1.0;
        u64 t = T;
        while (t) {
            if (t & 1) {
#pragma unroll
                for (int q = 0; q < CH; ++q) acc[q] *= x[c + q];
            }
            t >>= 1;
            if (t) {
#pragma unroll
                for (int q = 0; q < CH; ++q) x[c + q] *= x[c + q];
            }
        }
#pragma unroll
        for (int q = 0; q < CH; ++q) x[c + q] = neg[q] ? 0.0 : acc[q];
    }
}

// pow_complex for R elements with the same warp-level short cut: the loop
// over T's bits is uniform and CH independent elements per step give CH-way
// ILP (the per-element pow_complex is one latency chain per element and
// diverges on its own early out).  Per element the operations are those of
// pow_complex, so the results are bitwise identical.
template <int R, int CH>
__device__ __forceinline__ void pow_complex_vec_skip(double2 (&x)[R], u64 T, double neg_mag2) {
    static_assert(R % CH == 0, "chunk must divide R");
#pragma unroll
    for (int c = 0; c < R; c += CH) {
        bool neg[CH], all = true;
#pragma unroll
        for (int q = 0; q < CH; ++q) {
            neg[q] = fma(x[c + q].x, x[c + q].x, x[c + q].y * x[c + q].y) < neg_mag2;
            all &= neg[q];
        }
        if (__all_sync(0xffffffffu, all)) {
#pragma unroll
            for (int q = 0; q < CH; ++q) x[c + q] = make_double2(0.0, 0.0);
            continue;
        }
        double2 acc[CH];
#pragma unroll
        for (int q = 0; q < CH; ++q) acc[q] = make_double2(1.0, 0.0);
        u64 t = T;
        while (t) {
            if (t & 1) {
#pragma unroll
                for (int q = 0; q < CH; ++q) acc[q] = cmul(acc[q], x[c + q]);
            }
            t >>= 1;
            if (t) {
#pragma unroll
                for (int q = 0; q < CH; ++q) {
                    const double2 sq = x[c + q];
                    x[c + q] = make_double2(fma(sq.x, sq.x, -sq.y * sq.y), (sq.x + sq.x) * sq.y);
                }
            }
        }
#pragma unroll
        for (int q = 0; q < CH; ++q) x[c + q] = neg[q] ? make_double2(0.0, 0.0) : acc[q];
    }
}

// Real symbol lam(k0) for k0 = t + q * TPL (no power, no scale), over the
// groups of one tap set (set 0: the stencil S; set 1: an implicit solve's Q).
template <int N, int R, int TPL, class AC>
__device__ __forceinline__ void symbol_real_set(double (&lam)[R], int t, const FusedSymbol& sym,
                                                const double2* __restrict__ tw_all, AC acoef, int set) {
#pragma unroll
    for (int q = 0; q < R; ++q) lam[q] = 0.0;
    for (int gi = 0; gi < sym.ngroups; ++gi) {
        if (sym.group_set[gi] != set) continue;
        if (sym.group_partner[gi] < 0) continue;  // -og of a symmetric pair: counted with +og below
        double2 a = acoef(gi);
        const i64 og = sym.group_off[gi];
        if (og == 0) {  // exp(0) = 1: no table read
#pragma unroll
            for (int q = 0; q < R; ++q) lam[q] += a.x;
            continue;
        }
        // symmetric taps: A_{-og} = conj(A_og) and exp(-i phi) = conj(exp(i phi)), so the pair
        // contributes 2 Re(A_og exp(i phi)) -- one set of phase reads for both
        if (sym.group_partner[gi] > 0) a = make_double2(2.0 * a.x, 2.0 * a.y);
        if constexpr (R == 16 && TPL * 16 == N) {
            eplus16<N>(tw_all, t, og, [&](int q, double2 e) { lam[q] = fma(a.x, e.x, fma(-a.y, e.y, lam[q])); });
        } else {
#pragma unroll
            for (int q = 0; q < R; ++q) {
                const double2 e = eplus_tab(tw_all, N, (i64)(t + q * TPL) * og);
                lam[q] = fma(a.x, e.x, fma(-a.y, e.y, lam[q]));
            }
        }
    }
}

template <int N, int R, int TPL, bool IMPL = false, class AC>
__device__ __forceinline__ void symbol_real(double (&lam)[R], int t, const FusedSymbol& sym,
                                            const double2* __restrict__ tw_all, AC acoef) {
    symbol_real_set<N, R, TPL>(lam, t, sym, tw_all, acoef, 0);
    if constexpr (IMPL) {
        // solve_periodic_implicit (proj/src/periodic.cpp:108-124): lam = pinv(lamQ) lamS,
        // pinv(v) = |v| <= 1e-12 max|lamQ| ? 0 : 1/v (proj/src/spectrum.cpp:85-96)
        double lq[R];
        symbol_real_set<N, R, TPL>(lq, t, sym, tw_all, acoef, 1);
        const double eps = 1e-12 * __longlong_as_double((long long)*sym.qmax_bits);
#pragma unroll
        for (int q = 0; q < R; ++q) lam[q] = fabs(lq[q]) <= eps ? 0.0 : (1.0 / lq[q]) * lam[q];
    }
}

// One tap's contribution to the per-column group coefficient:
// c * exp(+2 pi i (kx o_last / L + ky o1 / n1)).
__device__ __forceinline__ double2 tap_term(const FusedSymbol& sym, const double2* tw_all, int j, i64 kx, i64 ky) {
    double2 e = eplus_tab(tw_all, sym.L, kx * (i64)sym.tap_olast[j]);
    if (sym.rank == 3) e = cmul(e, eplus_tab(tw_all, sym.n1, ky * (i64)sym.tap_o1[j]));
    return cscale(e, sym.tap_c[j]);
}

// v[q] (frequency k0 = t + q * TPL along axis 0) *= lam(k0)^T * scale, with
// lam = sum_g A_g exp(+2 pi i k0 O_g / N); A_g read from `acoef(g)`.
// Groups outer / elements inner so the 16 table reads of a group are
// independent (memory-level parallelism instead of a latency chain).
template <int N, int R, int TPL, class AC>
__device__ __forceinline__ void spectral_regs(double2 (&v)[R], int t, const FusedSymbol& sym,
                                              const double2* __restrict__ tw_all, AC acoef);

// Element q of this thread is frequency k0 = kbase + q * kstride.
template <int N, int R, class AC>
__device__ __forceinline__ void spectral_regs_at(double2 (&v)[R], int kbase, int kstride, const FusedSymbol& sym,
                                                 const double2* __restrict__ tw_all, AC acoef) {
    if (sym.real) {
        double lam[R];
#pragma unroll
        for (int q = 0; q < R; ++q) lam[q] = 0.0;
        for (int gi = 0; gi < sym.ngroups; ++gi) {
            const double2 a = acoef(gi);
            const i64 og = sym.group_off[gi];
            if (og == 0) {  // exp(0) = 1: no table read
#pragma unroll
                for (int q = 0; q < R; ++q) lam[q] += a.x;
                continue;
            }
#pragma unroll
            for (int q = 0; q < R; ++q) {
                const double2 e = eplus_tab(tw_all, N, (i64)(kbase + q * kstride) * og);
                lam[q] = fma(a.x, e.x, fma(-a.y, e.y, lam[q]));
            }
        }
#pragma unroll
        pow_real_vec_skip<R, (R % 4 == 0 ? 4 : R)>(lam, sym.T, sym.neg_mag2);
#pragma unroll
        for (int q = 0; q < R; ++q) v[q] = cscale(v[q], lam[q] * sym.scale);
    } else {
        // complex symbol: offset 0 needs no phase (a * 1 = a exactly), and a group
        // with offset -og shares the phase read of its partner +og
        // (exp(-i phi) = conj(exp(i phi)); FusedSymbol::group_partner)
        double2 lam[R];
#pragma unroll
        for (int q = 0; q < R; ++q) lam[q] = make_double2(0.0, 0.0);
        for (int gi = 0; gi < sym.ngroups; ++gi) {
            const int pg = sym.group_partner[gi] - 1;  // -1: none
            if (pg == -2) continue;                     // folded into its +og partner
            const double2 a = acoef(gi);
            const i64 og = sym.group_off[gi];
            if (og == 0) {
#pragma unroll
                for (int q = 0; q < R; ++q) lam[q] = cadd(lam[q], a);
                continue;
            }
            const double2 am = pg >= 0 ? acoef(pg) : make_double2(0.0, 0.0);
#pragma unroll
            for (int q = 0; q < R; ++q) {
                const double2 e = eplus_tab(tw_all, N, (i64)(kbase + q * kstride) * og);
                lam[q] = cadd(lam[q], cmul(a, e));
                if (pg >= 0) lam[q] = cadd(lam[q], cmul(am, cconj(e)));
            }
        }
#pragma unroll
        pow_complex_vec_skip<R, (R % 4 == 0 ? 4 : R)>(lam, sym.T, sym.neg_mag2);
#pragma unroll
        for (int q = 0; q < R; ++q) v[q] = cscale(cmul(lam[q], v[q]), sym.scale);
    }
}

template <int N, int R, int TPL, class AC>
__device__ __forceinline__ void spectral_regs(double2 (&v)[R], int t, const FusedSymbol& sym,
                                              const double2* __restrict__ tw_all, AC acoef) {
    if (sym.real) {
        double lam[R];
#pragma unroll
        for (int q = 0; q < R; ++q) lam[q] = 0.0;
        for (int gi = 0; gi < sym.ngroups; ++gi) {
            const double2 a = acoef(gi);
            const i64 og = sym.group_off[gi];
            if (og == 0) {
#pragma unroll
                for (int q = 0; q < R; ++q) lam[q] += a.x;
                continue;
            }
            if constexpr (R == 16 && TPL * 16 == N) {
                eplus16<N>(tw_all, t, og, [&](int q, double2 e) { lam[q] = fma(a.x, e.x, fma(-a.y, e.y, lam[q])); });
            } else {
#pragma unroll
                for (int q = 0; q < R; ++q) {
                    const double2 e = eplus_tab(tw_all, N, (i64)(t + q * TPL) * og);
                    lam[q] = fma(a.x, e.x, fma(-a.y, e.y, lam[q]));
                }
            }
        }
#pragma unroll
        pow_real_vec_skip<R, (R % 4 == 0 ? 4 : R)>(lam, sym.T, sym.neg_mag2);
#pragma unroll
        for (int q = 0; q < R; ++q) v[q] = cscale(v[q], lam[q] * sym.scale);
    } else if constexpr (R == 16 && TPL * 16 == N && N >= 4096) {
        // complex symbol, four elements q = 4 a + b (a = 0..3) per chunk b: one
        // phase read per group and chunk (e_b; the others are exact quarter
        // turns), and only four complex multipliers live next to the 16 data
        // values (the 16-wide multiplier array spilled at 128 registers)
#pragma unroll
        for (int b = 0; b < 4; ++b) {
            double2 lam[4];
#pragma unroll
            for (int a = 0; a < 4; ++a) lam[a] = make_double2(0.0, 0.0);
            for (int gi = 0; gi < sym.ngroups; ++gi) {
                const double2 c = acoef(gi);
                const i64 og = sym.group_off[gi];
                const double2 e = eplus_tab(tw_all, N, (i64)(t + b * (N / 16)) * og);
                const int mo = (int)(og & 3);
#pragma unroll
                for (int a = 0; a < 4; ++a) lam[a] = cadd(lam[a], cmul(c, rot_quarter(e, (mo * a) & 3)));
            }
            pow_complex_vec_skip<4, 4>(lam, sym.T, sym.neg_mag2);
#pragma unroll
            for (int a = 0; a < 4; ++a) v[4 * a + b] = cscale(cmul(lam[a], v[4 * a + b]), sym.scale);
        }
    } else {
        double2 lam[R];
#pragma unroll
        for (int q = 0; q < R; ++q) lam[q] = make_double2(0.0, 0.0);
        for (int gi = 0; gi < sym.ngroups; ++gi) {
            const double2 a = acoef(gi);
            const i64 og = sym.group_off[gi];
            if constexpr (R == 16 && TPL * 16 == N) {
                eplus16<N>(tw_all, t, og, [&](int q, double2 e) { lam[q] = cadd(lam[q], cmul(a, e)); });
            } else {
#pragma unroll
                for (int q = 0; q < R; ++q) {
                    const double2 e = eplus_tab(tw_all, N, (i64)(t + q * TPL) * og);
                    lam[q] = cadd(lam[q], cmul(a, e));
                }
            }
        }
#pragma unroll
        pow_complex_vec_skip<R, (R % 4 == 0 ? 4 : R)>(lam, sym.T, sym.neg_mag2);
#pragma unroll
        for (int q = 0; q < R; ++q) v[q] = cscale(cmul(lam[q], v[q]), sym.scale);
    }
}

}  // namespace fsx
