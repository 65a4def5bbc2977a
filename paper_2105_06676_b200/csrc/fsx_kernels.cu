// sm_100a kernels of the B200 StencilFFT-P path.
//
// Hot path (per BASELINE north_star; reference: proj/src/periodic.cpp:27-86,
// proj/src/fft.cpp:143-192, proj/src/spectrum.cpp:21-134):
//   k_r2c_rows      last-axis real -> half spectrum (packed pairs + split)
//   k_strided       C2C along a non-contiguous axis (optionally four-step twiddled)
//   k_fused_r2c     last forward axis pass + analytic symbol^T * x + first inverse pass
//   k_c2r_rows      half spectrum -> real, non-finite scan (realize_checked)
//   k_rowpair       1D four-step row stage fused with pairing + symbol^T + inverse rows
// General path (any dims / fields / non-pow2; still on the GPU):
//   k_contig / k_strided / k_direct_dft, k_spectral_general, k_promote, k_extract
//
// See DESIGN.md for the data layout and the roofline of each kernel.
#include <cfloat>

#include <map>
#include <mutex>

#include "fsx_async.cuh"
#include "fsx_device.cuh"
#include "fsx_kernels.h"
#include "fsx_spectral.cuh"

namespace fsx {

// ------------------------------------------------------------------ helpers
// a mod n for a power-of-two n (two's complement: exact for negative a too);
// the 1D row-pair symbols' phase indices (their lengths are powers of two) --
// the generic 64-bit modp is a ~40-instruction software sequence per call
__device__ __forceinline__ i64 modp2(i64 a, i64 n) { return a & (n - 1); }

__device__ __forceinline__ i64 modp(i64 a, i64 n) {
    const i64 r = a % n;
    return r < 0 ? r + n : r;
}

// exp(+2 pi i x / n) for the pow2 tables: conj(tw_all[n + (x mod n)])
__device__ __forceinline__ double2 eplus_pow2(const double2* tw_all, i64 n, i64 x) {
    return cconj(__ldg(tw_all + n + (x & (n - 1))));
}

template <int N>
struct Cfg {
    static constexpr int R = N < 16 ? N : 16;
    static constexpr int TPL = N / R;
    // strided tiles: W adjacent columns x N (64 KB of fp64 complex for N >= 512)
    static constexpr int W = N >= 4096 ? 1 : (4096 / N > 64 ? 64 : 4096 / N);
    // contiguous tiles: LINES lines x N, 256 threads
    static constexpr int LINES = N >= 4096 ? 1 : (256 / TPL);
    static constexpr int GW = W < 8 ? W : 8;                 // columns per quarter warp
    static constexpr int LSW = GW > 1 ? N + 8 / GW : N;      // smem line stride, strided tiles
    static constexpr int GL = TPL >= 8 ? 1 : 8 / TPL;        // lines per quarter warp
    static constexpr int LSL = GL > 1 ? N + 8 / GL : N;      // smem line stride, contiguous tiles
    // resident CTAs per SM the register budget is sized for (<= 128 regs at 256 threads)
    static constexpr int MINB_W = W * TPL <= 256 ? 2 : 1;
    static constexpr int MINB_L = LINES * TPL <= 256 ? 2 : 1;
};

// Binary exponentiation of a scalar symbol, the reference loop shape
// (proj/src/spectrum.cpp:53-64), with an exact-to-tolerance underflow
// short cut: |lam|^T < 2^-1100 is below every representable contribution
// (the reference's own product underflows to 0 / subnormal there).
__device__ __forceinline__ double2 pow_scalar(double2 lam, u64 T) {
    const double mag2 = fma(lam.x, lam.x, lam.y * lam.y);
    if (mag2 < 1.0) {
        int e;
        const double mant = frexp(mag2, &e);
        const float l2 = (float)e + __log2f((float)mant);
        if (l2 * (0.5f * (float)T) < -2200.0f) return make_double2(0.0, 0.0);
    }
    double2 acc = make_double2(1.0, 0.0), sq = lam;
    u64 t = T;
    while (t) {
        if (t & 1) acc = cmul(acc, sq);
        t >>= 1;
        if (t) sq = make_double2(fma(sq.x, sq.x, -sq.y * sq.y), (sq.x + sq.x) * sq.y);
    }
    return acc;
}

// Real symbol (symmetric stencil): same loop on one double.
__device__ __forceinline__ double pow_real(double lam, u64 T) {
    const double mag2 = lam * lam;
    if (mag2 < 1.0) {
        int e;
        const double mant = frexp(mag2, &e);
        const float l2 = (float)e + __log2f((float)mant);
        if (l2 * (0.5f * (float)T) < -2200.0f) return 0.0;
    }
    double acc = 1.0, sq = lam;
    u64 t = T;
    while (t) {
        if (t & 1) acc *= sq;
        t >>= 1;
        if (t) sq *= sq;
    }
    return acc;
}

template <int MM>
__device__ __forceinline__ void matmul_sq(const double2 (&a)[MM][MM], const double2 (&b)[MM][MM], double2 (&c)[MM][MM]) {
#pragma unroll
    for (int r = 0; r < MM; ++r)
#pragma unroll
        for (int col = 0; col < MM; ++col) {
            double2 acc = make_double2(0.0, 0.0);
#pragma unroll
            for (int t = 0; t < MM; ++t) {
                const double2 p = cmul(a[r][t], b[t][col]);
                acc = cadd(acc, p);
            }
            c[r][col] = acc;
        }
}

// acc = I, sq = lam; while t { if t&1 acc = acc*sq; t >>= 1; if t sq = sq*sq }
// (proj/src/spectrum.cpp:66-82)
template <int MM>
__device__ __forceinline__ void pow_block(double2 (&lam)[MM][MM], u64 T) {
    double2 acc[MM][MM], tmp[MM][MM];
#pragma unroll
    for (int r = 0; r < MM; ++r)
#pragma unroll
        for (int c = 0; c < MM; ++c) acc[r][c] = make_double2(r == c ? 1.0 : 0.0, 0.0);
    u64 t = T;
    while (t) {
        if (t & 1) {
            matmul_sq<MM>(acc, lam, tmp);
#pragma unroll
            for (int r = 0; r < MM; ++r)
#pragma unroll
                for (int c = 0; c < MM; ++c) acc[r][c] = tmp[r][c];
        }
        t >>= 1;
        if (t) {
            matmul_sq<MM>(lam, lam, tmp);
#pragma unroll
            for (int r = 0; r < MM; ++r)
#pragma unroll
                for (int c = 0; c < MM; ++c) lam[r][c] = tmp[r][c];
        }
    }
#pragma unroll
    for (int r = 0; r < MM; ++r)
#pragma unroll
        for (int c = 0; c < MM; ++c) lam[r][c] = acc[r][c];
}

// ------------------------------------------------------------------ C2C passes
// Contiguous lines: line l occupies in[l * pitch + 0 .. N).
template <int N, int SIGN>
__global__ void __launch_bounds__(Cfg<N>::LINES * Cfg<N>::TPL, Cfg<N>::MINB_L)
k_contig(const double2* in, double2* out, i64 nlines, i64 pitch, const double2* __restrict__ tw_all) {
    using C = Cfg<N>;
    using F = LineFFT<N, SIGN>;
    extern __shared__ double2 sm[];
    const int b = threadIdx.x / C::TPL, t = threadIdx.x % C::TPL;
    const i64 line = (i64)blockIdx.x * C::LINES + b;
    const bool ok = line < nlines;
    double2 v[C::R];
    const double2* src = in + line * pitch;
#pragma unroll
    for (int q = 0; q < C::R; ++q) v[q] = ok ? src[t + q * C::TPL] : make_double2(0.0, 0.0);
    F::run(v, t, sm + b * C::LSL, tw_all + N);
    if (ok) {
        double2* dst = out + line * pitch;
#pragma unroll
        for (int q = 0; q < C::R; ++q) dst[t + q * C::TPL] = v[q];
    }
}

// Strided lines: W adjacent columns per CTA, the axis in shared memory.
// TI / TO = float2: the fp32 storage mode's first / last pass of the 1D plan
// (the column pass reads the float grid, or writes it), fp64 arithmetic.
template <int N, int SIGN, int TWM, class TI = double2, class TO = double2>
__global__ void __launch_bounds__(Cfg<N>::W * Cfg<N>::TPL, Cfg<N>::MINB_W)
k_strided(const TI* in, TO* out, AxisGeom g, StepTwiddle st, const double2* __restrict__ tw_all,
          Flags* flags) {
    using C = Cfg<N>;
    using F = LineFFT<N, SIGN>;
    extern __shared__ double2 sm[];
    const int w = threadIdx.x % C::W, t = threadIdx.x / C::W;
    const i64 tiles = (g.ncols + C::W - 1) / C::W;
    const i64 o = (i64)blockIdx.x / tiles;
    const i64 c = ((i64)blockIdx.x % tiles) * C::W + w;
    const bool ok = c < g.ncols;
    const i64 base = o * g.block + c;
    double2 v[C::R];
#pragma unroll
    for (int q = 0; q < C::R; ++q)
        v[q] = ok ? to_d2(in[base + (i64)(t + q * C::TPL) * g.inner]) : make_double2(0.0, 0.0);
    // four-step twiddle W^(b (k kmul + o omul)) for k = t + q TPL: the
    // exponents of one thread form an arithmetic progression in q, so two
    // table reads (base, ratio) and a running product replace 16 two-level
    // lookups (<= 15 extra roundings; the per-element lookups were as much
    // L2 traffic as the data of the 1D plan's column passes)
    double2 tq = make_double2(1.0, 0.0), tr = tq;
    if constexpr (TWM != 0) {
        const i64 bq = c / st.col_div;
        tq = phase_at(st.tab, bq * ((i64)t * st.kmul + o * st.omul));
        tr = phase_at(st.tab, bq * (i64)C::TPL * st.kmul);
    }
    if constexpr (TWM == 2) {
#pragma unroll
        for (int q = 0; q < C::R; ++q) {
            v[q] = cmulc(v[q], tq);
            tq = cmul(tq, tr);
        }
    }
    F::run(v, t, sm + w * C::LSW, tw_all + N);
    if constexpr (TWM == 1) {
#pragma unroll
        for (int q = 0; q < C::R; ++q) {
            v[q] = cmul(v[q], tq);
            tq = cmul(tq, tr);
        }
    }
    bool bad = false;
#pragma unroll
    for (int q = 0; q < C::R; ++q) {
        const TO r = from_d2<TO>(v[q]);
        if (ok) out[base + (i64)(t + q * C::TPL) * g.inner] = r;
        bad |= ok && (!isfinite(r.x) || !isfinite(r.y));
    }
    if (flags) flag_nonfinite(bad, flags);  // last pass of a solve: the non-finite scan rides along (realize_checked)
}

// fp32 storage mode, 1D plan: the first forward column pass reading the float
// grid (SIGN -1, post-twiddle) and the last inverse one writing it (SIGN +1,
// pre-twiddle, non-finite scan), for the strided route (N <= 256).
template <int N>
static cudaError_t axis_f32_n(const void* in, void* out, const AxisGeom& g, int sign, const StepTwiddle& st,
                              const double2* tw, cudaStream_t s, Flags* flags) {
    using C = Cfg<N>;
    const size_t smem = (size_t)C::W * C::LSW * sizeof(double2);
    const i64 blocks = g.outer * ((g.ncols + C::W - 1) / C::W);
    if (sign < 0 && st.mode == 1) {
        auto kf = k_strided<N, -1, 1, float2, double2>;
        kernel_prepare((const void*)kf, smem);
        kf<<<(unsigned)blocks, C::W * C::TPL, smem, s>>>(static_cast<const float2*>(in), static_cast<double2*>(out), g,
                                                        st, tw, flags);
    } else if (sign > 0 && st.mode == 2) {
        auto kf = k_strided<N, +1, 2, double2, float2>;
        kernel_prepare((const void*)kf, smem);
        kf<<<(unsigned)blocks, C::W * C::TPL, smem, s>>>(static_cast<const double2*>(in), static_cast<float2*>(out), g,
                                                        st, tw, flags);
    } else {
        return cudaErrorInvalidValue;
    }
    return cudaGetLastError();
}

bool axis_f32_ok(const AxisGeom& g) { return g.inner > 1 && g.n >= 2 && g.n <= 256 && (g.n & (g.n - 1)) == 0; }

cudaError_t launch_axis_f32(const void* in, void* out, const AxisGeom& g, int sign, const StepTwiddle& st,
                            const double2* tw, cudaStream_t s, Flags* flags) {
    switch (g.n) {
        case 2: return axis_f32_n<2>(in, out, g, sign, st, tw, s, flags);
        case 4: return axis_f32_n<4>(in, out, g, sign, st, tw, s, flags);
        case 8: return axis_f32_n<8>(in, out, g, sign, st, tw, s, flags);
        case 16: return axis_f32_n<16>(in, out, g, sign, st, tw, s, flags);
        case 32: return axis_f32_n<32>(in, out, g, sign, st, tw, s, flags);
        case 64: return axis_f32_n<64>(in, out, g, sign, st, tw, s, flags);
        case 128: return axis_f32_n<128>(in, out, g, sign, st, tw, s, flags);
        case 256: return axis_f32_n<256>(in, out, g, sign, st, tw, s, flags);
        default: return cudaErrorInvalidValue;
    }
}

// Direct O(n^2) DFT for non-power-of-two axes (one line per CTA; the line
// staged in shared memory so the pass can run in place).
__global__ void k_direct_dft(const double2* in, double2* out, AxisGeom g, int sign, PhaseTable tab) {
    extern __shared__ double2 sm[];
    const i64 line = blockIdx.x;
    const i64 o = line / g.ncols, c = line % g.ncols;
    const i64 base = o * g.block + c;
    const i64 n = g.n;
    for (i64 p = threadIdx.x; p < n; p += blockDim.x) sm[p] = in[base + p * g.inner];
    __syncthreads();
    for (i64 k = threadIdx.x; k < n; k += blockDim.x) {
        double2 acc = make_double2(0.0, 0.0);
        i64 idx = 0;
        for (i64 j = 0; j < n; ++j) {
            const double2 w = phase_at(tab, idx);
            acc = cadd(acc, sign < 0 ? cmul(sm[j], w) : cmulc(sm[j], w));
            idx += k;
            if (idx >= n) idx -= n;
        }
        out[base + k * g.inner] = acc;
    }
}

// ------------------------------------------------------------------ real <-> half spectrum rows
// Row of L = 2M reals viewed as M complex z[j] = x[2j] + i x[2j+1];
// Z = DFT_M(z); X[k] = E[k] + W_L^k O[k] with E = (Z[k] + conj Z[M-k]) / 2,
// O = -i (Z[k] - conj Z[M-k]) / 2; X[M] = Re Z[0] - Im Z[0].
template <int M>
__global__ void __launch_bounds__(Cfg<M>::LINES * Cfg<M>::TPL, Cfg<M>::MINB_L)
k_r2c_rows(const double* __restrict__ x, double2* __restrict__ H, i64 nrows, i64 L, RowLayout lay,
           const double2* __restrict__ tw_all) {
    using C = Cfg<M>;
    using F = LineFFT<M, -1>;
    extern __shared__ double2 sm[];
    const int b = threadIdx.x / C::TPL, t = threadIdx.x % C::TPL;
    const i64 row = (i64)blockIdx.x * C::LINES + b;
    const bool ok = row < nrows;
    double2* line = sm + b * C::LSL;
    const double2* src = reinterpret_cast<const double2*>(x + row * L);
    double2 v[C::R];
#pragma unroll
    for (int q = 0; q < C::R; ++q) v[q] = ok ? src[t + q * C::TPL] : make_double2(0.0, 0.0);
    F::run(v, t, line, tw_all + M);
    __syncthreads();
#pragma unroll
    for (int q = 0; q < C::R; ++q) line[swz(t + q * C::TPL)] = v[q];
    __syncthreads();
    if (!ok) return;
#pragma unroll
    for (int q = 0; q < C::R; ++q) {
        const int k = t + q * C::TPL;
        const double2 zk = v[q];
        const double2 zm = cconj(line[swz((M - k) & (M - 1))]);
        const double2 e = cscale(cadd(zk, zm), 0.5);
        const double2 od = cscale(cmul_si<-1>(csub(zk, zm)), 0.5);
        const double2 w = __ldg(tw_all + 2 * M + k);  // exp(-2 pi i k / L)
        *lay.ptr(H, row, k) = cadd(e, cmul(w, od));
        if (k == 0) *lay.ptr(H, row, M) = make_double2(zk.x - zk.y, 0.0);
    }
    if (lay.peers) __threadfence_system();  // remote (NVLink) stores ordered before the rank barrier
}

// Inverse: Z[k] = (X[k] + conj X[M-k]) + i conj(W_L^k) (X[k] - conj X[M-k]),
// unnormalized inverse DFT_M, x[2j] = Re z[j], x[2j+1] = Im z[j] (times L;
// the 1/N of the inverse transform is folded into the spectral multiply).
template <int M>
__global__ void __launch_bounds__(Cfg<M>::LINES * Cfg<M>::TPL, Cfg<M>::MINB_L)
k_c2r_rows(const double2* __restrict__ H, double* __restrict__ x, i64 nrows, i64 L, RowLayout lay,
           const double2* __restrict__ tw_all, Flags* flags) {
    using C = Cfg<M>;
    using F = LineFFT<M, +1>;
    extern __shared__ double2 sm[];
    __shared__ double2 nyq[C::LINES];
    const int b = threadIdx.x / C::TPL, t = threadIdx.x % C::TPL;
    const i64 row = (i64)blockIdx.x * C::LINES + b;
    const bool ok = row < nrows;
    double2* line = sm + b * C::LSL;
    double2 v[C::R];
#pragma unroll
    for (int q = 0; q < C::R; ++q) {
        v[q] = ok ? *lay.ptr(H, row, t + q * C::TPL) : make_double2(0.0, 0.0);
        line[swz(t + q * C::TPL)] = v[q];
    }
    if (t == 0) nyq[b] = ok ? *lay.ptr(H, row, M) : make_double2(0.0, 0.0);
    __syncthreads();
#pragma unroll
    for (int q = 0; q < C::R; ++q) {
        const int k = t + q * C::TPL;
        const double2 xm = cconj(k == 0 ? nyq[b] : line[swz(M - k)]);
        const double2 e = cadd(v[q], xm);
        const double2 od = cmulc(csub(v[q], xm), __ldg(tw_all + 2 * M + k));
        v[q] = cadd(e, cmul_si<+1>(od));
    }
    F::run(v, t, line, tw_all + M);
    bool bad = false;
    if (ok) {
        double2* dst = reinterpret_cast<double2*>(x + row * L);
#pragma unroll
        for (int q = 0; q < C::R; ++q) {
            dst[t + q * C::TPL] = v[q];
            bad |= !isfinite(v[q].x) || !isfinite(v[q].y);
        }
    }
    flag_nonfinite(bad, flags);
}

// ------------------------------------------------------------------ fused spectral pass (R2C layout)
// Last forward axis (axis 0, strided) -> lam(k)^T * X(k) / N -> first inverse
// axis pass, one tile in registers + shared memory.  lam(k) is the analytic
// symbol sum_taps c * exp(+2 pi i sum_a k_a o_a / n_a) (the transform of the
// reference's generator column, proj/src/spectrum.cpp:21-45), grouped by the
// axis-0 offset: A_g(column) is formed once per column, then per element
// lam = sum_g A_g * exp(+2 pi i k0 O_g / n0).
template <int N, int W, int MINB>
__global__ void __launch_bounds__(W * Cfg<N>::TPL, MINB)
k_fused_r2c(double2* H, AxisGeom g, FusedSymbol sym, const double2* __restrict__ tw_all) {
    using C = Cfg<N>;
    using FF = LineFFT<N, -1>;
    using FI = LineFFT<N, +1>;
    constexpr int GW = W < 8 ? W : 8;
    constexpr int LSW = GW > 1 ? N + 8 / GW : N;
    constexpr bool PAR = W <= 8;  // per-tap terms in parallel (smem for ntaps x W terms)
    extern __shared__ double2 sm[];
    __shared__ double2 acoef[kMaxGroups][W];
    __shared__ double2 tapterm[PAR ? kMaxFusedTaps : 1][PAR ? W : 1];
    const int w = threadIdx.x % W, t = threadIdx.x / W;
    const i64 tiles = (g.ncols + W - 1) / W;
    const i64 o = (i64)blockIdx.x / tiles;
    const i64 c = ((i64)blockIdx.x % tiles) * W + w;
    i64 kx, ky;
    fused_col_freqs(sym, c, kx, ky);
    const bool ok = c < g.ncols && kx <= sym.M;
    const i64 base = o * g.block + c;
    double2 v[C::R];
#pragma unroll
    for (int q = 0; q < C::R; ++q)
        v[q] = ok ? H[base + (i64)(t + q * C::TPL) * g.inner] : make_double2(0.0, 0.0);
    // per-column symbol coefficients: tap terms issued before the FFT so
    // their table reads overlap it
    if constexpr (PAR) {
        for (int j = t; j < sym.ntaps; j += C::TPL) tapterm[j][w] = tap_term(sym, tw_all, j, kx, ky);
    }
    double2* line = sm + w * LSW;
    FF::run(v, t, line, tw_all + N);
    __syncthreads();
    for (int gi = t; gi < sym.ngroups; gi += C::TPL) {
        double2 a = make_double2(0.0, 0.0);
        for (int j = 0; j < sym.ntaps; ++j)
            if (sym.tap_group[j] == gi) a = cadd(a, PAR ? tapterm[PAR ? j : 0][PAR ? w : 0] : tap_term(sym, tw_all, j, kx, ky));
        acoef[gi][w] = a;
    }
    __syncthreads();
    spectral_regs<N, C::R, C::TPL>(v, t, sym, tw_all, [&](int gi) { return acoef[gi][w]; });
    FI::run(v, t, line, tw_all + N);
    if (ok) {
#pragma unroll
        for (int q = 0; q < C::R; ++q) H[base + (i64)(t + q * C::TPL) * g.inner] = v[q];
    }
}

// ------------------------------------------------------------------ 1D row-pair fused pass
// z holds the four-step intermediate [N1][N2] (row r, col c = frequency
// r + N1 c after the row FFT).  One CTA owns rows r and N1 - r, so every
// frequency k meets its partner M - k (mode 0, real packing) or N - k
// (mode 1, two-for-one) inside the CTA.
__device__ __forceinline__ double2 sym1(const RowPairArgs& a, i64 k, i64 n) {
    double2 lam = make_double2(0.0, 0.0);
    for (int j = 0; j < a.ntaps; ++j) {
        const double2 e = cconj(phase_at(a.wk, modp2(k * (i64)a.tap_off[j], n)));
        lam = make_double2(fma(a.tap_b[j][0], e.x, lam.x), fma(a.tap_b[j][0], e.y, lam.y));
    }
    return lam;
}

__device__ __forceinline__ void pair_mode0(const RowPairArgs& a, double2& zk, double2& zp, i64 k, i64 M) {
    // k in [0, M); partner kp = M - k in (0, M]; for k == 0 the partner is the Nyquist bin.
    const i64 L = 2 * M, kp = M - k;
    const double2 cz = cconj(zp);
    const double2 e = cscale(cadd(zk, cz), 0.5);
    const double2 od = cscale(cmul_si<-1>(csub(zk, cz)), 0.5);
    const double2 wk = phase_at(a.wk, k);
    const double2 wp = phase_at(a.wk, kp);
    const double2 xk = cadd(e, cmul(wk, od));
    const double2 xp = cadd(cconj(e), cmul(wp, cconj(od)));
    double2 yk, yp;
    if (a.real) {
        yk = cscale(xk, pow_realv(sym1(a, k, L).x, a.T, a.neg_mag2) * a.scale);
        yp = cscale(xp, pow_realv(sym1(a, kp, L).x, a.T, a.neg_mag2) * a.scale);
    } else {
        yk = cscale(cmul(pow_scalar(sym1(a, k, L), a.T), xk), a.scale);
        yp = cscale(cmul(pow_scalar(sym1(a, kp, L), a.T), xp), a.scale);
    }
    const double2 cyp = cconj(yp), cyk = cconj(yk);
    zk = cadd(cadd(yk, cyp), cmul_si<+1>(cmulc(csub(yk, cyp), wk)));
    if (k != 0) zp = cadd(cadd(yp, cyk), cmul_si<+1>(cmulc(csub(yp, cyk), wp)));
}

// pair_mode0 for a real (symmetric) symbol, four frequencies k at once (the
// partners kp = M - k come with them): the phase reads of all four are issued
// together and the eight powers run element-parallel with the warp-level
// underflow skip, where pair_mode0 is one latency chain per frequency (cfg1's
// row-pair pass ran at ~7 warps per SM on those chains).  With L = 2M,
// cos(2 pi kp o / L) = (-1)^o cos(2 pi k o / L) and W_L^kp = -conj(W_L^k), so
// the partners need no reads of their own.  k != 0 (the k = 0 / Nyquist pair
// stays on pair_mode0).
__device__ __forceinline__ void pair_mode0_real_x4(const RowPairArgs& a, double2 (&zk)[4], double2 (&zp)[4],
                                                   const i64 (&k)[4], i64 M) {
    const i64 L = 2 * M;
    double2 wk[4];
    double x[8];
#pragma unroll
    for (int i = 0; i < 4; ++i) {
        wk[i] = phase_at(a.wk, k[i]);
        x[i] = x[4 + i] = 0.0;
    }
    int last = 0;  // cos is even in o: offset 0 reads nothing, +-o share one read
    double lastc[4] = {1.0, 1.0, 1.0, 1.0};
    for (int j = 0; j < a.ntaps; ++j) {
        const int o = a.tap_off[j], ao = o < 0 ? -o : o;
        const double b = a.tap_b[j][0], bp = (o & 1) ? -b : b;
        if (ao != 0 && ao != last) {
#pragma unroll
            for (int i = 0; i < 4; ++i) lastc[i] = phase_at(a.wk, modp2(k[i] * (i64)ao, L)).x;
            last = ao;
        }
#pragma unroll
        for (int i = 0; i < 4; ++i) {
            const double c = ao == 0 ? 1.0 : lastc[i];
            x[i] = fma(b, c, x[i]);
            x[4 + i] = fma(bp, c, x[4 + i]);
        }
    }
    pow_real_vec_skip<8, 4>(x, a.T, a.neg_mag2);
#pragma unroll
    for (int i = 0; i < 4; ++i) {
        const double2 cz = cconj(zp[i]);
        const double2 e = cscale(cadd(zk[i], cz), 0.5);
        const double2 od = cscale(cmul_si<-1>(csub(zk[i], cz)), 0.5);
        const double2 wp = make_double2(-wk[i].x, wk[i].y);
        const double2 xk = cadd(e, cmul(wk[i], od));
        const double2 xp = cadd(cconj(e), cmul(wp, cconj(od)));
        const double2 yk = cscale(xk, x[i] * a.scale);
        const double2 yp = cscale(xp, x[4 + i] * a.scale);
        const double2 cyp = cconj(yp), cyk = cconj(yk);
        zk[i] = cadd(cadd(yk, cyp), cmul_si<+1>(cmulc(csub(yk, cyp), wk[i])));
        zp[i] = cadd(cadd(yp, cyk), cmul_si<+1>(cmulc(csub(yp, cyk), wp)));
    }
}

// Real 2x2 symbol power by Cayley-Hamilton, NX independent chains.
// A^n = p_n A + q_n I (A^2 = t A - d I, t = trace, d = det), tracked as
// (p_n, tr_n = trace A^n, d^n) by left-to-right binary exponentiation:
//   A^2n  : p <- p tr,             tr <- tr^2 - 2 d^n,      d^n <- (d^n)^2
//   A^n+1 : p' = (p t + tr) / 2,   tr <- p' t - 2 d p,      d^n <- d^n d
// and q_T = (tr_T - p_T t) / 2 at the end.  4 ops per squaring and 5 per
// multiply against the matrix loop's 6 and 8 (proj/src/spectrum.cpp:66-82);
// for det A = 1 (area-preserving schemes: cfg5's leapfrog) d^n stays 1 and a
// squaring is 2 ops -- the same arithmetic as the general branch, so the fast
// branch changes no bit.  Accuracy: near a double eigenvalue (the wave
// equation's low frequencies) the matrix product cancels n^2-sized terms
// while tr_n stays bounded; against an exact (60-digit) power of the same
// fp64 symbol the worst relative error at cfg5 (N = 2^26, T = 1e6) is 6.4e-5
// here and 12 for the matrix loop (scripts/pow_accuracy.py).
template <int NX>
__device__ __forceinline__ void pow_real2_ch(const double (&l)[NX][4], u64 T, double (&acc)[NX][4]) {
    if (T == 0) {
#pragma unroll
        for (int i = 0; i < NX; ++i) {
            acc[i][0] = acc[i][3] = 1.0;
            acc[i][1] = acc[i][2] = 0.0;
        }
        return;
    }
    double t[NX], m2d[NX], p[NX], tr[NX], dn[NX];
    bool unit = true;
#pragma unroll
    for (int i = 0; i < NX; ++i) {
        t[i] = l[i][0] + l[i][3];
        const double d = fma(l[i][0], l[i][3], -(l[i][1] * l[i][2]));
        m2d[i] = -2.0 * d;
        p[i] = 1.0;
        tr[i] = t[i];
        dn[i] = d;
        unit = unit && d == 1.0;
    }
    const int top = 63 - __clzll((long long)T);
    if (unit) {
#pragma unroll 1
        for (int b = top - 1; b >= 0; --b) {
#pragma unroll
            for (int i = 0; i < NX; ++i) {
                p[i] *= tr[i];
                tr[i] = fma(tr[i], tr[i], -2.0);
            }
            if ((T >> b) & 1) {
#pragma unroll
                for (int i = 0; i < NX; ++i) {
                    const double pn = 0.5 * fma(p[i], t[i], tr[i]);
                    tr[i] = fma(pn, t[i], -2.0 * p[i]);
                    p[i] = pn;
                }
            }
        }
    } else {
#pragma unroll 1
        for (int b = top - 1; b >= 0; --b) {
#pragma unroll
            for (int i = 0; i < NX; ++i) {
                p[i] *= tr[i];
                tr[i] = fma(tr[i], tr[i], -2.0 * dn[i]);
                dn[i] *= dn[i];
            }
            if ((T >> b) & 1) {
#pragma unroll
                for (int i = 0; i < NX; ++i) {
                    const double pn = 0.5 * fma(p[i], t[i], tr[i]);
                    tr[i] = fma(pn, t[i], m2d[i] * p[i]);
                    p[i] = pn;
                    dn[i] *= -0.5 * m2d[i];
                }
            }
        }
    }
#pragma unroll
    for (int i = 0; i < NX; ++i) {
        const double q = 0.5 * fma(-p[i], t[i], tr[i]);
        acc[i][0] = fma(p[i], l[i][0], q);
        acc[i][1] = p[i] * l[i][1];
        acc[i][2] = p[i] * l[i][2];
        acc[i][3] = fma(p[i], l[i][3], q);
    }
}

__device__ __forceinline__ void pair_mode1(const RowPairArgs& a, double2& zk, double2& zp, i64 k, i64 N) {
    const double2 cz = cconj(zp);
    const double2 u = cscale(cadd(zk, cz), 0.5);
    const double2 vv = cscale(cmul_si<-1>(csub(zk, cz)), 0.5);
    if (a.real) {
        // symmetric block stencil: lam(k) = sum B cos(2 pi k o / N) is a real 2x2
        // matrix, raised by the Cayley-Hamilton chain in real arithmetic
        double l[1][4] = {{0.0, 0.0, 0.0, 0.0}}, A[1][4];
        for (int j = 0; j < a.ntaps; ++j) {
            const double c = phase_at(a.wk, modp2(k * (i64)a.tap_off[j], N)).x;
#pragma unroll
            for (int e = 0; e < 4; ++e) l[0][e] = fma(a.tap_b[j][e], c, l[0][e]);
        }
        pow_real2_ch<1>(l, a.T, A);
        const double a00 = A[0][0], a01 = A[0][1], a10 = A[0][2], a11 = A[0][3];
        const double sc = a.scale;
        const double2 u2 = make_double2(sc * fma(a00, u.x, a01 * vv.x), sc * fma(a00, u.y, a01 * vv.y));
        const double2 v2 = make_double2(sc * fma(a10, u.x, a11 * vv.x), sc * fma(a10, u.y, a11 * vv.y));
        zk = cadd(u2, cmul_si<+1>(v2));
        zp = cadd(cconj(u2), cmul_si<+1>(cconj(v2)));
        return;
    }
    double2 lam[2][2] = {{make_double2(0, 0), make_double2(0, 0)}, {make_double2(0, 0), make_double2(0, 0)}};
    for (int j = 0; j < a.ntaps; ++j) {
        const double2 e = cconj(phase_at(a.wk, modp2(k * (i64)a.tap_off[j], N)));
#pragma unroll
        for (int r = 0; r < 2; ++r)
#pragma unroll
            for (int cc = 0; cc < 2; ++cc) {
                const double bb = a.tap_b[j][r * 2 + cc];
                lam[r][cc] = make_double2(fma(bb, e.x, lam[r][cc].x), fma(bb, e.y, lam[r][cc].y));
            }
    }
    pow_block<2>(lam, a.T);
    const double2 u2 = cscale(cadd(cmul(lam[0][0], u), cmul(lam[0][1], vv)), a.scale);
    const double2 v2 = cscale(cadd(cmul(lam[1][0], u), cmul(lam[1][1], vv)), a.scale);
    zk = cadd(u2, cmul_si<+1>(v2));
    zp = cadd(cconj(u2), cmul_si<+1>(cconj(v2)));
}

// Real 2x2 block symbols, NX frequencies per call (independent power chains:
// the row-pair pass of cfg5 is bound by this arithmetic at T = 1e6).  The host
// folds the +-o taps of a symmetric stencil into one cosine term per |o|
// (rowpair_args), so offset 0 needs no table read and every other term one.
__device__ __forceinline__ void real_block_symbol(const RowPairArgs& a, i64 k, i64 N, double (&l)[4]) {
    l[0] = l[1] = l[2] = l[3] = 0.0;
    for (int j = 0; j < a.ntaps; ++j) {
        const int o = a.tap_off[j];
        const double c = o == 0 ? 1.0 : phase_at(a.wk, modp2(k * (i64)o, N)).x;
#pragma unroll
        for (int e = 0; e < 4; ++e) l[e] = fma(a.tap_b[j][e], c, l[e]);
    }
}

template <int NX>
__device__ __forceinline__ void pair_mode1_real_xn(const RowPairArgs& a, double2 (&zk)[NX], double2 (&zp)[NX],
                                                   const i64 (&k)[NX], i64 N) {
    double l[NX][4], acc[NX][4];
#pragma unroll
    for (int i = 0; i < NX; ++i) real_block_symbol(a, k[i], N, l[i]);
    pow_real2_ch<NX>(l, a.T, acc);
    const double sc = a.scale;
#pragma unroll
    for (int i = 0; i < NX; ++i) {
        const double2 cz = cconj(zp[i]);
        const double2 u = cscale(cadd(zk[i], cz), 0.5);
        const double2 vv = cscale(cmul_si<-1>(csub(zk[i], cz)), 0.5);
        const double2 u2 = make_double2(sc * fma(acc[i][0], u.x, acc[i][1] * vv.x), sc * fma(acc[i][0], u.y, acc[i][1] * vv.y));
        const double2 v2 = make_double2(sc * fma(acc[i][2], u.x, acc[i][3] * vv.x), sc * fma(acc[i][2], u.y, acc[i][3] * vv.y));
        zk[i] = cadd(u2, cmul_si<+1>(v2));
        zp[i] = cadd(cconj(u2), cmul_si<+1>(cconj(v2)));
    }
}

#ifndef FSX_RP_NX
#define FSX_RP_NX 4  // cfg5: 4 chains 1.85 ms vs 2 chains 1.90 ms (same box)
#endif
template <int N2>
__global__ void __launch_bounds__(2 * Cfg<N2>::TPL)
k_rowpair(RowPairArgs a) {
    using C = Cfg<N2>;
    using FF = LineFFT<N2, -1>;
    using FI = LineFFT<N2, +1>;
    constexpr int LS = N2 + ((C::TPL >= 8) ? 0 : 8 / (8 / C::TPL > 2 ? 2 : 8 / C::TPL));
    extern __shared__ double2 sm[];
    const i64 N1 = a.N1, M = a.N1 * a.N2;
    const i64 ra = blockIdx.x;
    const i64 rb = (N1 - ra) % N1;
    const bool self = ra == rb;
    const int b = threadIdx.x / C::TPL, t = threadIdx.x % C::TPL;
    const i64 fr = b == 0 ? ra : rb;  // frequency row k1
    // storage row: k1 itself, or its digit-reversed position after a split column FFT
    const i64 row = a.row_split ? (fr % (N1 / a.row_split)) * a.row_split + fr / (N1 / a.row_split) : fr;
    const bool ok = b == 0 || !self;
    double2* line = sm + b * LS;
    double2* src = a.z + row * N2;
    double2 v[C::R];
#pragma unroll
    for (int q = 0; q < C::R; ++q) v[q] = ok ? src[t + q * C::TPL] : make_double2(0.0, 0.0);
    FF::run(v, t, line, a.tw_all + N2);
    __syncthreads();
#pragma unroll
    for (int q = 0; q < C::R; ++q) line[swz(t + q * C::TPL)] = v[q];
    __syncthreads();
    double2* la = sm;
    double2* lb = self ? sm : sm + LS;
    const int nth = blockDim.x;
    if (!self) {
        int cpos = threadIdx.x;
        if (a.mode == 0 && a.real && nth >= 32) {  // four frequencies (+ partners) per step (full warps: vote)
            for (; cpos + 3 * nth < N2; cpos += 4 * nth) {
                double2 zk[4], zp[4];
                i64 k[4];
#pragma unroll
                for (int i = 0; i < 4; ++i) {
                    zk[i] = la[swz(cpos + i * nth)];
                    zp[i] = lb[swz(N2 - 1 - (cpos + i * nth))];
                    k[i] = ra + N1 * (cpos + i * nth);
                }
                pair_mode0_real_x4(a, zk, zp, k, M);
#pragma unroll
                for (int i = 0; i < 4; ++i) {
                    la[swz(cpos + i * nth)] = zk[i];
                    lb[swz(N2 - 1 - (cpos + i * nth))] = zp[i];
                }
            }
        }
        if (a.mode == 1 && a.real) {  // FSX_RP_NX independent power chains per step
            for (; cpos + (FSX_RP_NX - 1) * nth < N2; cpos += FSX_RP_NX * nth) {
                double2 zk[FSX_RP_NX], zp[FSX_RP_NX];
                i64 k[FSX_RP_NX];
#pragma unroll
                for (int i = 0; i < FSX_RP_NX; ++i) {
                    zk[i] = la[swz(cpos + i * nth)];
                    zp[i] = lb[swz(N2 - 1 - (cpos + i * nth))];
                    k[i] = ra + N1 * (cpos + i * nth);
                }
                pair_mode1_real_xn<FSX_RP_NX>(a, zk, zp, k, M);
#pragma unroll
                for (int i = 0; i < FSX_RP_NX; ++i) {
                    la[swz(cpos + i * nth)] = zk[i];
                    lb[swz(N2 - 1 - (cpos + i * nth))] = zp[i];
                }
            }
        }
        for (; cpos < N2; cpos += nth) {
            const int cp = N2 - 1 - cpos;
            double2 zk = la[swz(cpos)], zp = lb[swz(cp)];
            const i64 k = ra + N1 * cpos;
            if (a.mode == 0) pair_mode0(a, zk, zp, k, M);
            else pair_mode1(a, zk, zp, k, M);
            la[swz(cpos)] = zk;
            lb[swz(cp)] = zp;
        }
    } else if (ra == 0) {
        for (int cpos = threadIdx.x; cpos <= N2 / 2; cpos += nth) {
            const int cp = (N2 - cpos) % N2;
            double2 zk = la[swz(cpos)], zp = la[swz(cp)];
            const i64 k = N1 * (i64)cpos;
            if (a.mode == 0) pair_mode0(a, zk, zp, k, M);
            else pair_mode1(a, zk, zp, k, M);
            if (cp != cpos) la[swz(cp)] = zp;
            la[swz(cpos)] = zk;
        }
    } else {  // ra == N1 / 2
        for (int cpos = threadIdx.x; cpos < N2 / 2; cpos += nth) {
            const int cp = N2 - 1 - cpos;
            double2 zk = la[swz(cpos)], zp = la[swz(cp)];
            const i64 k = ra + N1 * (i64)cpos;
            if (a.mode == 0) pair_mode0(a, zk, zp, k, M);
            else pair_mode1(a, zk, zp, k, M);
            la[swz(cpos)] = zk;
            la[swz(cp)] = zp;
        }
    }
    __syncthreads();
#pragma unroll
    for (int q = 0; q < C::R; ++q) v[q] = line[swz(t + q * C::TPL)];
    FI::run(v, t, line, a.tw_all + N2);
    if (ok) {
#pragma unroll
        for (int q = 0; q < C::R; ++q) src[t + q * C::TPL] = v[q];
    }
}

// ------------------------------------------------------------------ general path
__global__ void k_promote(const double* __restrict__ x, double2* __restrict__ z, i64 n) {
    for (i64 i = (i64)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (i64)gridDim.x * blockDim.x)
        z[i] = make_double2(x[i], 0.0);
}

__device__ __forceinline__ void atomic_max_nonneg(unsigned long long* addr, double v) {
    atomicMax(addr, (unsigned long long)__double_as_longlong(v));
}

__device__ __forceinline__ double warp_max(double v) {
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) v = fmax(v, __shfl_xor_sync(0xffffffffu, v, o));
    return v;
}

// realize_checked (proj/src/periodic.cpp:49-65): real part out, finite scan,
// max |re| and max |im| for the residue test (decided on the host).
__global__ void k_extract(const double2* __restrict__ z, double* __restrict__ x, i64 n, Flags* flags) {
    double mre = 0.0, mim = 0.0;
    bool bad = false;
    for (i64 i = (i64)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (i64)gridDim.x * blockDim.x) {
        const double2 v = z[i];
        x[i] = v.x;
        bad |= !isfinite(v.x) || !isfinite(v.y);
        mre = fmax(mre, fabs(v.x));
        mim = fmax(mim, fabs(v.y));
    }
    flag_nonfinite(bad, flags);
    mre = warp_max(mre);
    mim = warp_max(mim);
    if ((threadIdx.x & 31) == 0) {
        atomic_max_nonneg(&flags->max_re_bits, mre);
        atomic_max_nonneg(&flags->max_im_bits, mim);
    }
}

__global__ void k_finite(const double* __restrict__ x, i64 n, Flags* flags) {
    bool bad = false;
    for (i64 i = (i64)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (i64)gridDim.x * blockDim.x)
        bad |= !isfinite(x[i]);
    flag_nonfinite(bad, flags);
}

// position -> frequency along each axis (four-step split axes are stored
// in [k1][k2] order = frequency k1 + n1 k2)
__device__ __forceinline__ void cell_freqs(const GeneralSymbol& s, i64 cell, i64* k) {
    for (int a = s.rank - 1; a >= 0; --a) {
        const i64 n = s.dims[a];
        const i64 p = cell % n;
        cell /= n;
        if (s.split[a]) {
            const i64 n1 = s.split[a], n2 = n / n1;
            k[a] = p / n2 + n1 * (p % n2);
        } else {
            k[a] = p;
        }
    }
}

// sum_taps B * exp(+2 pi i sum_a k_a o_a / n_a)
template <int MM>
__device__ __forceinline__ void symbol_at(const GeneralSymbol& s, const i64* k, int ntaps, const long long* offs,
                                          const double* blocks, double2 (&lam)[MM][MM], int m) {
#pragma unroll
    for (int r = 0; r < MM; ++r)
#pragma unroll
        for (int c = 0; c < MM; ++c) lam[r][c] = make_double2(0.0, 0.0);
    for (int j = 0; j < ntaps; ++j) {
        double2 e = make_double2(1.0, 0.0);
        for (int a = 0; a < s.rank; ++a) {
            const i64 o = offs[j * s.rank + a];
            if (o == 0) continue;
            e = cmul(e, cconj(phase_at(s.tab[a], modp(k[a] * o, s.dims[a]))));
        }
#pragma unroll
        for (int r = 0; r < MM; ++r)
#pragma unroll
            for (int c = 0; c < MM; ++c) {
                if (r < m && c < m) {
                    const double bb = blocks[(j * m + r) * m + c];
                    lam[r][c] = make_double2(fma(bb, e.x, lam[r][c].x), fma(bb, e.y, lam[r][c].y));
                }
            }
    }
}

__device__ __forceinline__ double2 crecip(double2 v) {
    const double d = fma(v.x, v.x, v.y * v.y);
    return make_double2(v.x / d, -v.y / d);
}

template <int MM>
__global__ void k_spectral_general(double2* z, GeneralSymbol s) {
    for (i64 cell = (i64)blockIdx.x * blockDim.x + threadIdx.x; cell < s.cells;
         cell += (i64)gridDim.x * blockDim.x) {
        i64 k[kMaxRank];
        cell_freqs(s, cell, k);
        double2 lam[MM][MM];
        symbol_at<MM>(s, k, s.ntaps, s.offsets, s.blocks, lam, MM);
        if constexpr (MM == 1) {
            if (s.implicit) {
                double2 lq[1][1];
                symbol_at<1>(s, k, s.ntaps_q, s.offsets_q, s.blocks_q, lq, 1);
                const double eps = 1e-12 * s.qmax[0];
                const double mag = hypot(lq[0][0].x, lq[0][0].y);
                const double2 inv = mag <= eps ? make_double2(0.0, 0.0) : crecip(lq[0][0]);
                lam[0][0] = cmul(inv, lam[0][0]);
            }
            double2 acc = make_double2(1.0, 0.0), sq = lam[0][0];
            u64 t = s.T;
            while (t) {
                if (t & 1) acc = cmul(acc, sq);
                t >>= 1;
                if (t) sq = cmul(sq, sq);
            }
            for (i64 b = 0; b < s.batch; ++b) {  // stacked grids share the symbol
                double2* zc = z + b * s.cells + cell;
                *zc = cscale(cmul(acc, *zc), s.scale);
            }
        } else {
            pow_block<MM>(lam, s.T);
            for (i64 b = 0; b < s.batch; ++b) {
                double2* zc = z + (b * s.cells + cell) * MM;
                double2 x[MM], y[MM];
#pragma unroll
                for (int f = 0; f < MM; ++f) x[f] = zc[f];
#pragma unroll
                for (int r = 0; r < MM; ++r) {
                    double2 acc = make_double2(0.0, 0.0);
#pragma unroll
                    for (int c = 0; c < MM; ++c) acc = cadd(acc, cmul(lam[r][c], x[c]));
                    y[r] = cscale(acc, s.scale);
                }
#pragma unroll
                for (int f = 0; f < MM; ++f) zc[f] = y[f];
            }
        }
    }
}

// spectrum_from_kernel export: blocks at natural-order frequencies.
template <int MM>
__global__ void k_symbol_blocks(double2* out, GeneralSymbol s, int which_q) {
    for (i64 cell = (i64)blockIdx.x * blockDim.x + threadIdx.x; cell < s.cells;
         cell += (i64)gridDim.x * blockDim.x) {
        i64 k[kMaxRank];
        cell_freqs(s, cell, k);
        double2 lam[MM][MM];
        if (which_q) symbol_at<MM>(s, k, s.ntaps_q, s.offsets_q, s.blocks_q, lam, MM);
        else symbol_at<MM>(s, k, s.ntaps, s.offsets, s.blocks, lam, MM);
#pragma unroll
        for (int r = 0; r < MM; ++r)
#pragma unroll
            for (int c = 0; c < MM; ++c) out[(cell * MM + r) * MM + c] = lam[r][c];
    }
}

__global__ void k_symbol_absmax(GeneralSymbol s, unsigned long long* out_bits) {
    double mx = 0.0;
    for (i64 cell = (i64)blockIdx.x * blockDim.x + threadIdx.x; cell < s.cells;
         cell += (i64)gridDim.x * blockDim.x) {
        i64 k[kMaxRank];
        cell_freqs(s, cell, k);
        double2 lam[1][1];
        symbol_at<1>(s, k, s.ntaps_q, s.offsets_q, s.blocks_q, lam, 1);
        mx = fmax(mx, hypot(lam[0][0].x, lam[0][0].y));
    }
    mx = warp_max(mx);
    if ((threadIdx.x & 31) == 0) atomic_max_nonneg(out_bits, mx);
}

template <int MM>
__global__ void k_pow_blocks(const double2* in, double2* out, i64 cells, u64 T) {
    for (i64 cell = (i64)blockIdx.x * blockDim.x + threadIdx.x; cell < cells; cell += (i64)gridDim.x * blockDim.x) {
        if constexpr (MM == 1) {
            double2 acc = make_double2(1.0, 0.0), sq = in[cell];
            u64 t = T;
            while (t) {
                if (t & 1) acc = cmul(acc, sq);
                t >>= 1;
                if (t) sq = cmul(sq, sq);
            }
            out[cell] = acc;
        } else {
            double2 lam[MM][MM];
#pragma unroll
            for (int r = 0; r < MM; ++r)
#pragma unroll
                for (int c = 0; c < MM; ++c) lam[r][c] = in[(cell * MM + r) * MM + c];
            pow_block<MM>(lam, T);
#pragma unroll
            for (int r = 0; r < MM; ++r)
#pragma unroll
                for (int c = 0; c < MM; ++c) out[(cell * MM + r) * MM + c] = lam[r][c];
        }
    }
}

__global__ void k_absmax(const double2* in, i64 n, unsigned long long* out_bits) {
    double mx = 0.0;
    for (i64 i = (i64)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (i64)gridDim.x * blockDim.x)
        mx = fmax(mx, hypot(in[i].x, in[i].y));
    mx = warp_max(mx);
    if ((threadIdx.x & 31) == 0) atomic_max_nonneg(out_bits, mx);
}

// pseudo_inverse_spectrum (proj/src/spectrum.cpp:85-96)
__global__ void k_pinv(const double2* in, double2* out, i64 n, const double* maxabs) {
    const double eps = 1e-12 * maxabs[0];
    for (i64 i = (i64)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (i64)gridDim.x * blockDim.x) {
        const double2 v = in[i];
        out[i] = hypot(v.x, v.y) <= eps ? make_double2(0.0, 0.0) : crecip(v);
    }
}

template <int MM>
__global__ void k_block_mul(const double2* a, const double2* b, double2* out, i64 cells) {
    for (i64 cell = (i64)blockIdx.x * blockDim.x + threadIdx.x; cell < cells; cell += (i64)gridDim.x * blockDim.x) {
        double2 A[MM][MM], B[MM][MM], Cm[MM][MM];
#pragma unroll
        for (int r = 0; r < MM; ++r)
#pragma unroll
            for (int c = 0; c < MM; ++c) {
                A[r][c] = a[(cell * MM + r) * MM + c];
                B[r][c] = b[(cell * MM + r) * MM + c];
            }
        matmul_sq<MM>(A, B, Cm);
#pragma unroll
        for (int r = 0; r < MM; ++r)
#pragma unroll
            for (int c = 0; c < MM; ++c) out[(cell * MM + r) * MM + c] = Cm[r][c];
    }
}

// hadamard (proj/src/spectrum.cpp:111-134)
template <int MM>
__global__ void k_block_matvec(const double2* lam, const double2* x, double2* y, i64 cells) {
    for (i64 cell = (i64)blockIdx.x * blockDim.x + threadIdx.x; cell < cells; cell += (i64)gridDim.x * blockDim.x) {
#pragma unroll
        for (int r = 0; r < MM; ++r) {
            double2 acc = make_double2(0.0, 0.0);
#pragma unroll
            for (int c = 0; c < MM; ++c) acc = cadd(acc, cmul(lam[(cell * MM + r) * MM + c], x[cell * MM + c]));
            y[cell * MM + r] = acc;
        }
    }
}

// [outer][n1][n2][inner] <-> [outer][n2][n1][inner]
__global__ void k_transpose_split(const double2* in, double2* out, i64 outer, i64 n1, i64 n2, i64 inner,
                                  int to_natural) {
    const i64 total = outer * n1 * n2 * inner;
    for (i64 i = (i64)blockIdx.x * blockDim.x + threadIdx.x; i < total; i += (i64)gridDim.x * blockDim.x) {
        const i64 f = i % inner;
        i64 r = i / inner;
        // destination-major indexing
        if (to_natural) {  // dst [o][k2][k1][f] from src [o][k1][k2][f]
            const i64 k1 = r % n1;
            r /= n1;
            const i64 k2 = r % n2;
            const i64 o = r / n2;
            out[i] = in[((o * n1 + k1) * n2 + k2) * inner + f];
        } else {  // dst [o][k1][k2][f] from src [o][k2][k1][f]
            const i64 k2 = r % n2;
            r /= n2;
            const i64 k1 = r % n1;
            const i64 o = r / n1;
            out[i] = in[((o * n2 + k2) * n1 + k1) * inner + f];
        }
    }
}

// ================================================================== launchers
static int grid_for(i64 n, int threads) {
    i64 b = (n + threads - 1) / threads;
    if (b > 148 * 16) b = 148 * 16;
    return (int)(b < 1 ? 1 : b);
}

// ------------------------------------------------------------------ Bluestein (non-pow2 axes)
// The reference's Bluestein transform (proj/src/fft.cpp:103-139, chirp
// e^(-i pi n^2 / n_len) with n^2 reduced mod 2 n_len): the lines of an axis are
// gathered into a [lines][P] buffer (P = pow2 >= 2n - 1) premultiplied by the
// chirp, convolved with the chirp filter by pow2 FFTs (filter spectrum Bhat
// precomputed per plan), and scattered back postmultiplied by the chirp.
// Inverse = conj(forward(conj x)) (fft.cpp:151-154), unnormalized.
__global__ void k_blue_pre(const double2* __restrict__ Z, double2* __restrict__ buf, AxisGeom g, i64 P,
                           const double2* __restrict__ chirp, int conj_in) {
    const i64 total = g.outer * g.ncols * P;
    for (i64 i = (i64)blockIdx.x * blockDim.x + threadIdx.x; i < total; i += (i64)gridDim.x * blockDim.x) {
        const i64 l = i / P, n = i - l * P;
        double2 v = make_double2(0.0, 0.0);
        if (n < g.n) {
            const i64 o = l / g.ncols, c = l - o * g.ncols;
            double2 x = Z[o * g.block + c + n * g.inner];
            if (conj_in) x = cconj(x);
            v = cmul(x, chirp[n]);
        }
        buf[i] = v;
    }
}

__global__ void k_blue_mul(double2* __restrict__ buf, i64 total, i64 P, const double2* __restrict__ bhat) {
    for (i64 i = (i64)blockIdx.x * blockDim.x + threadIdx.x; i < total; i += (i64)gridDim.x * blockDim.x)
        buf[i] = cmul(buf[i], bhat[i % P]);
}

__global__ void k_blue_post(const double2* __restrict__ buf, double2* __restrict__ Z, AxisGeom g, i64 P,
                            const double2* __restrict__ chirp, double scale, int conj_out) {
    const i64 total = g.outer * g.ncols * g.n;
    for (i64 i = (i64)blockIdx.x * blockDim.x + threadIdx.x; i < total; i += (i64)gridDim.x * blockDim.x) {
        const i64 l = i / g.n, k = i - l * g.n;
        const i64 o = l / g.ncols, c = l - o * g.ncols;
        double2 v = cscale(cmul(buf[l * P + k], chirp[k]), scale);
        if (conj_out) v = cconj(v);
        Z[o * g.block + c + k * g.inner] = v;
    }
}

cudaError_t launch_blue_pre(const double2* Z, double2* buf, const AxisGeom& g, i64 P, const double2* chirp, int conj_in,
                            cudaStream_t s) {
    k_blue_pre<<<grid_for(g.outer * g.ncols * P, 256), 256, 0, s>>>(Z, buf, g, P, chirp, conj_in);
    return cudaGetLastError();
}

cudaError_t launch_blue_mul(double2* buf, i64 lines, i64 P, const double2* bhat, cudaStream_t s) {
    k_blue_mul<<<grid_for(lines * P, 256), 256, 0, s>>>(buf, lines * P, P, bhat);
    return cudaGetLastError();
}

cudaError_t launch_blue_post(const double2* buf, double2* Z, const AxisGeom& g, i64 P, const double2* chirp,
                             double scale, int conj_out, cudaStream_t s) {
    k_blue_post<<<grid_for(g.outer * g.ncols * g.n, 256), 256, 0, s>>>(buf, Z, g, P, chirp, scale, conj_out);
    return cudaGetLastError();
}


template <int N>
static cudaError_t axis_pow2_n(const double2* in, double2* out, const AxisGeom& g, int sign,
                               const StepTwiddle& st, const double2* tw, cudaStream_t s, Flags* flags) {
    using C = Cfg<N>;
    if (g.inner == 1 && st.mode == 0) {
        const size_t smem = (size_t)C::LINES * C::LSL * sizeof(double2);
        const int blocks = (int)((g.outer + C::LINES - 1) / C::LINES);
        auto kf = sign < 0 ? k_contig<N, -1> : k_contig<N, +1>;
        kernel_prepare((const void*)kf, smem);
        kf<<<blocks, C::LINES * C::TPL, smem, s>>>(in, out, g.outer, g.block, tw);
        if (flags) return launch_finite_check(reinterpret_cast<const double*>(out), 2 * g.outer * g.block, flags, s);
        return cudaGetLastError();
    }
    const size_t smem = (size_t)C::W * C::LSW * sizeof(double2);
    const i64 tiles = (g.ncols + C::W - 1) / C::W;
    const i64 blocks = g.outer * tiles;
    void (*kf)(const double2*, double2*, AxisGeom, StepTwiddle, const double2*, Flags*);
    if (sign < 0) kf = st.mode == 1 ? k_strided<N, -1, 1> : st.mode == 2 ? k_strided<N, -1, 2> : k_strided<N, -1, 0>;
    else kf = st.mode == 1 ? k_strided<N, +1, 1> : st.mode == 2 ? k_strided<N, +1, 2> : k_strided<N, +1, 0>;
    kernel_prepare((const void*)kf, smem);
    kf<<<(unsigned)blocks, C::W * C::TPL, smem, s>>>(in, out, g, st, tw, flags);
    return cudaGetLastError();
}

cudaError_t launch_axis_pow2(const double2* in, double2* out, const AxisGeom& g, int sign,
                             const StepTwiddle& st, const double2* tw, cudaStream_t s, Flags* flags) {
    {
        const cudaError_t e = launch_axis_tma(in, out, g, sign, st, tw, s, flags);
        if (e != cudaErrorNotSupported) return e;
    }
    if (pipe_enabled() && pipe_cols_ok(g.n) && g.inner > 1 && st.mode == 0 && in == out && !flags) {
        FusedSymbol none;
        return launch_cols_pipe(out, g, sign < 0 ? 0 : 1, none, tw, s);
    }
    switch (g.n) {
        case 2: return axis_pow2_n<2>(in, out, g, sign, st, tw, s, flags);
        case 4: return axis_pow2_n<4>(in, out, g, sign, st, tw, s, flags);
        case 8: return axis_pow2_n<8>(in, out, g, sign, st, tw, s, flags);
        case 16: return axis_pow2_n<16>(in, out, g, sign, st, tw, s, flags);
        case 32: return axis_pow2_n<32>(in, out, g, sign, st, tw, s, flags);
        case 64: return axis_pow2_n<64>(in, out, g, sign, st, tw, s, flags);
        case 128: return axis_pow2_n<128>(in, out, g, sign, st, tw, s, flags);
        case 256: return axis_pow2_n<256>(in, out, g, sign, st, tw, s, flags);
        case 512: return axis_pow2_n<512>(in, out, g, sign, st, tw, s, flags);
        case 1024: return axis_pow2_n<1024>(in, out, g, sign, st, tw, s, flags);
        case 2048: return axis_pow2_n<2048>(in, out, g, sign, st, tw, s, flags);
        case 4096: return axis_pow2_n<4096>(in, out, g, sign, st, tw, s, flags);
        case 8192: return axis_pow2_n<8192>(in, out, g, sign, st, tw, s, flags);
        default: return cudaErrorInvalidValue;
    }
}

cudaError_t launch_axis_direct(const double2* in, double2* out, const AxisGeom& g, int sign,
                               const PhaseTable& tab, cudaStream_t s) {
    const size_t smem = (size_t)g.n * sizeof(double2);
    kernel_prepare((const void*)k_direct_dft, smem);
    const i64 lines = g.outer * g.ncols;
    k_direct_dft<<<(unsigned)lines, 256, smem, s>>>(in, out, g, sign, tab);
    return cudaGetLastError();
}

template <int M>
static cudaError_t r2c_m(const double* x, double2* H, i64 nrows, i64 L, const RowLayout& P, const double2* tw,
                         cudaStream_t s) {
    using C = Cfg<M>;
    const size_t smem = (size_t)C::LINES * C::LSL * sizeof(double2);
    kernel_prepare((const void*)k_r2c_rows<M>, smem);
    k_r2c_rows<M><<<(unsigned)((nrows + C::LINES - 1) / C::LINES), C::LINES * C::TPL, smem, s>>>(x, H, nrows, L, P, tw);
    return cudaGetLastError();
}

template <int M>
static cudaError_t c2r_m(const double2* H, double* x, i64 nrows, i64 L, const RowLayout& P, const double2* tw, Flags* f,
                         cudaStream_t s) {
    using C = Cfg<M>;
    const size_t smem = (size_t)C::LINES * C::LSL * sizeof(double2);
    kernel_prepare((const void*)k_c2r_rows<M>, smem);
    k_c2r_rows<M><<<(unsigned)((nrows + C::LINES - 1) / C::LINES), C::LINES * C::TPL, smem, s>>>(H, x, nrows, L, P, tw, f);
    return cudaGetLastError();
}

bool pdl_enabled() {
    static int v = -1;
    if (v < 0) {
        const char* e = getenv("FSX_PDL");
        v = (e && e[0] == '0') ? 0 : 1;
    }
    return v == 1;
}

int cluster_policy() {
    static int v = -1;
    if (v < 0) {
        const char* e = getenv("FSX_CLUSTER_POLICY");
        v = e ? atoi(e) : 0;
    }
    return v;
}

int kernel_prepare(const void* fn, size_t smem, int threads) {
    struct Info {
        size_t smem = 0;
        int threads = -1, per_sm = 0;
    };
    static std::mutex mu;
    static std::map<std::pair<const void*, int>, Info> cache;
    int dev = 0;
    cudaGetDevice(&dev);
    std::lock_guard<std::mutex> lk(mu);
    Info& e = cache[{fn, dev}];
    if (e.smem != smem || e.threads != threads) {
        // always (static + dynamic > 48 KB needs the opt-in even when dynamic alone is below it)
        cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
        e.per_sm = 0;
        if (threads > 0) cudaOccupancyMaxActiveBlocksPerMultiprocessor(&e.per_sm, fn, threads, smem);
        e.smem = smem;
        e.threads = threads;
    }
    return e.per_sm;
}

// max |lamQ(k)| over the half spectrum for the implicit fused symbol: the
// pinv threshold of the reference (proj/src/spectrum.cpp:85-96) needs it
// before any multiplier is formed.  |lam(-k)| = |lam(k)| for real taps, so
// the half spectrum covers the full one.
__global__ void k_fused_qmax(FusedSymbol sym, i64 ncols, unsigned long long* out, const double2* __restrict__ tw_all) {
    double m = 0.0;
    const i64 total = sym.n0 * ncols;
    for (i64 i = (i64)blockIdx.x * blockDim.x + threadIdx.x; i < total; i += (i64)gridDim.x * blockDim.x) {
        const i64 k0 = i / ncols, c = i - k0 * ncols;
        i64 kx, ky;
        fused_col_freqs(sym, c, kx, ky);
        if (kx > sym.M) continue;
        double2 lam = make_double2(0.0, 0.0);
        for (int j = 0; j < sym.ntaps; ++j) {
            const int g = sym.tap_group[j];
            if (sym.group_set[g] != 1) continue;
            const double2 e = cmul(tap_term(sym, tw_all, j, kx, ky), eplus_tab(tw_all, sym.n0, k0 * (i64)sym.group_off[g]));
            lam = cadd(lam, e);
        }
        m = fmax(m, hypot(lam.x, lam.y));
    }
    m = warp_max(m);
    if ((threadIdx.x & 31) == 0) atomic_max_nonneg(out, m);
}

cudaError_t launch_fused_qmax(const FusedSymbol& sym, i64 ncols, unsigned long long* out, const double2* tw,
                              cudaStream_t s) {
    const i64 total = sym.n0 * ncols;
    i64 blocks = (total + 255) / 256;
    if (blocks > 148 * 16) blocks = 148 * 16;
    k_fused_qmax<<<(unsigned)blocks, 256, 0, s>>>(sym, ncols, out, tw);
    return cudaGetLastError();
}

#define FSX_POW2_CASES(MACRO) \
    MACRO(8) MACRO(16) MACRO(32) MACRO(64) MACRO(128) MACRO(256) MACRO(512) MACRO(1024) MACRO(2048) MACRO(4096) MACRO(8192)

cudaError_t launch_r2c_rows(const double* x, double2* H, i64 nrows, i64 L, const RowLayout& P, const double2* tw,
                            cudaStream_t s) {
    if (pipe_enabled() && pipe_rows_ok(L / 2) && rows_variant() == 3) return launch_r2c_bulk(x, H, nrows, L, P, tw, s);
    if (pipe_enabled() && pipe_rows_ok(L / 2) && (rows_variant() == 1 || rows_variant() == 3)) return launch_r2c_pipe(x, H, nrows, L, P, tw, s);
    switch (L / 2) {
#define C_(M) case M: return r2c_m<M>(x, H, nrows, L, P, tw, s);
        FSX_POW2_CASES(C_)
#undef C_
        default: return cudaErrorInvalidValue;
    }
}

cudaError_t launch_c2r_rows(const double2* H, double* x, i64 nrows, i64 L, const RowLayout& P, const double2* tw, Flags* f,
                            cudaStream_t s) {
    if (pipe_enabled() && pipe_rows_ok(L / 2) && rows_variant() == 3) return launch_c2r_bulk(H, x, nrows, L, P, tw, f, s);
    if (pipe_enabled() && pipe_rows_ok(L / 2) && (rows_variant() == 1 || rows_variant() == 3)) return launch_c2r_pipe(H, x, nrows, L, P, tw, f, s);
    switch (L / 2) {
#define C_(M) case M: return c2r_m<M>(H, x, nrows, L, P, tw, f, s);
        FSX_POW2_CASES(C_)
#undef C_
        default: return cudaErrorInvalidValue;
    }
}

template <int N, int W, int MINB>
static cudaError_t fused_nw(double2* H, const AxisGeom& g, const FusedSymbol& sym, const double2* tw, cudaStream_t s) {
    constexpr int GW = W < 8 ? W : 8;
    constexpr int LSW = GW > 1 ? N + 8 / GW : N;
    const size_t smem = (size_t)W * LSW * sizeof(double2);
    const i64 tiles = (g.ncols + W - 1) / W;
    kernel_prepare((const void*)k_fused_r2c<N, W, MINB>, smem);
    k_fused_r2c<N, W, MINB><<<(unsigned)(g.outer * tiles), W * Cfg<N>::TPL, smem, s>>>(H, g, sym, tw);
    return cudaGetLastError();
}

// FSX_FUSED_VARIANT (A/B measurements, N = 4096 only): 0 = W1 x 2 CTAs/SM
// (default), 1 = W1 x 1 CTA/SM (full register file), 2 = W2 x 1 CTA/SM.
static int fused_variant() {
    static int v = -1;
    if (v < 0) {
        const char* e = getenv("FSX_FUSED_VARIANT");
        v = e ? atoi(e) : 0;
    }
    return v;
}

template <int N>
static cudaError_t fused_n(double2* H, const AxisGeom& g, const FusedSymbol& sym, const double2* tw, cudaStream_t s) {
    using C = Cfg<N>;
    if constexpr (N == 4096) {
        const int var = fused_variant();
        if (var == 1) return fused_nw<N, 1, 1>(H, g, sym, tw, s);
        if (var == 2) return fused_nw<N, 2, 1>(H, g, sym, tw, s);
    }
    return fused_nw<N, C::W, C::MINB_W>(H, g, sym, tw, s);
}

cudaError_t launch_fused_r2c(double2* H, const AxisGeom& g, const FusedSymbol& sym, const double2* tw, cudaStream_t s) {
    if (pipe_enabled() && pipe_cols_ok(g.n)) return launch_cols_pipe(H, g, 2, sym, tw, s);
    switch (g.n) {
#define C_(N) case N: return fused_n<N>(H, g, sym, tw, s);
        FSX_POW2_CASES(C_)
#undef C_
        default: return cudaErrorInvalidValue;
    }
}

// ------------------------------------------------------------------ row pairs on a CTA pair
// k_rowpair holds rows r and N1 - r in one CTA (2 x 64 KB at N2 = 4096): one
// 512-thread CTA per SM, whose row loads, pairing and stores no other CTA
// overlaps (cfg5: 1.6 ms, FP64 pipe 42 %, warps 25 %).  Here a 2-CTA cluster
// takes the pair, one row per CTA (64 KB tile + 32 KB landing: two CTAs per
// SM), the row arriving by one bulk copy:
//   1. forward row FFT; thread th holds X[th + TPL q];
//   2. exchange 1 over DSMEM: each CTA sends the upper half of its row
//      (positions >= N2/2, q >= 8) into the peer's landing zone;
//   3. CTA h pairs its own positions p < N2/2 with the peer's N2 - 1 - p
//      (landing index N2/2 - 1 - p): CTA 0 (row r) owns frequencies
//      k = r + N1 p, CTA 1 (row N1 - r) their partners -- the same pair
//      arithmetic as k_rowpair, so the results are bitwise equal;
//   4. exchange 2: the partner's updated value goes back into the peer's tile
//      at N2 - 1 - p (its upper half, free once the peer reports its forward
//      FFT reads done);
//   5. inverse row FFT from registers (lower half) + tile (upper half), store.
// Rows 0 and N1 / 2 pair with themselves: cluster 0 runs them with
// k_rowpair's self-pairing loops, one row per CTA, no exchange.
template <int N2>
__global__ void __cluster_dims__(2, 1, 1) __launch_bounds__(N2 / 16, 2)
k_rowpair_c(RowPairArgs a) {
    using FF = LineFFT<N2, -1>;
    using FI = LineFFT<N2, +1>;
    constexpr int TPL = N2 / 16, R = 16, HALF = N2 / 2;
    extern __shared__ __align__(128) double2 tile[];  // [N2] row (+ FFT exchanges), [N2 / 2] landing
    double2* recv = tile + N2;
    __shared__ __align__(8) unsigned long long bar, bx1, bx2, bok;
    const int th = threadIdx.x;
    const unsigned h = cluster_rank(), peer = h ^ 1u;
    const i64 N1 = a.N1, M = a.N1 * a.N2;
    const i64 ci = (i64)(blockIdx.x >> 1);
    const bool self = ci == 0;  // rows 0 (CTA 0) and N1 / 2 (CTA 1)
    const i64 fr = self ? (h == 0 ? 0 : N1 / 2) : (h == 0 ? ci : N1 - ci);  // frequency row k1
    const i64 row = a.row_split ? (fr % (N1 / a.row_split)) * a.row_split + fr / (N1 / a.row_split) : fr;
    double2* src = a.z + row * N2;
    if (th == 0) {
        mbar_init(&bar, 1);
        mbar_init(&bx1, 1);
        mbar_init(&bx2, 1);
        mbar_init(&bok, 1);
        mbar_init_fence();
        mbar_expect_tx(&bx1, (unsigned)(HALF * sizeof(double2)));
        mbar_expect_tx(&bx2, (unsigned)(HALF * sizeof(double2)));
        pdl_wait();
        mbar_expect_tx(&bar, (unsigned)(N2 * sizeof(double2)));
        bulk_load(tile, src, (unsigned)(N2 * sizeof(double2)), &bar);
    }
    cluster_arrive_relaxed();
    cluster_wait();  // the peer's barriers exist
    mbar_wait(&bar, 0);
    double2 v[R];
#pragma unroll
    for (int q = 0; q < R; ++q) v[q] = tile[th + q * TPL];
    FF::run(v, th, tile, a.tw_all + N2);
    if (self) {
        // k_rowpair's self-paired rows, one row per CTA
        __syncthreads();
#pragma unroll
        for (int q = 0; q < R; ++q) tile[swz(th + q * TPL)] = v[q];
        __syncthreads();
        if (h == 0) {
            for (int cpos = th; cpos <= N2 / 2; cpos += TPL) {
                const int cp = (N2 - cpos) % N2;
                double2 zk = tile[swz(cpos)], zp = tile[swz(cp)];
                const i64 k = N1 * (i64)cpos;
                if (a.mode == 0) pair_mode0(a, zk, zp, k, M);
                else pair_mode1(a, zk, zp, k, M);
                if (cp != cpos) tile[swz(cp)] = zp;
                tile[swz(cpos)] = zk;
            }
        } else {
            for (int cpos = th; cpos < N2 / 2; cpos += TPL) {
                const int cp = N2 - 1 - cpos;
                double2 zk = tile[swz(cpos)], zp = tile[swz(cp)];
                const i64 k = fr + N1 * (i64)cpos;
                if (a.mode == 0) pair_mode0(a, zk, zp, k, M);
                else pair_mode1(a, zk, zp, k, M);
                tile[swz(cpos)] = zk;
                tile[swz(cp)] = zp;
            }
        }
        __syncthreads();
#pragma unroll
        for (int q = 0; q < R; ++q) v[q] = tile[swz(th + q * TPL)];
        __syncthreads();  // the inverse FFT's exchanges overwrite the tile
    } else {
        pdl_trigger();
        // exchange 1: the upper half of this row into the peer's landing zone
        {
            const unsigned dst = peer_smem(recv + th, peer), pbar = peer_smem(&bx1, peer);
#pragma unroll
            for (int b = 0; b < R / 2; ++b) st_async_peer(dst + (unsigned)(TPL * 16 * b), v[R / 2 + b], pbar);
        }
        __syncthreads();  // every thread is past the forward FFT's tile reads
        if (th == 0) mbar_arrive_peer(peer_smem(&bok, peer));  // the peer may write this tile's upper half
        // park the own lower half in the tile (positions the peer never writes)
        // so the pairing's power chains have the registers to themselves
#pragma unroll
        for (int q = 0; q < R / 2; ++q) tile[th + q * TPL] = v[q];
        mbar_wait(&bx1, 0);
        mbar_wait_cluster(&bok, 0);  // the peer's upper half is free for exchange 2
        // own positions p = th + TPL q (q < R/2) with the peer's N2 - 1 - p
        // (landing N2/2 - 1 - p); the partner's result goes straight back into
        // the peer's tile at N2 - 1 - p (exchange 2)
        const unsigned pbar = peer_smem(&bx2, peer);
        constexpr int NX = 4;
#pragma unroll 1
        for (int q0 = 0; q0 < R / 2; q0 += NX) {
            double2 zk[NX], zp[NX];
            i64 k[NX];
#pragma unroll
            for (int i = 0; i < NX; ++i) {
                const int p = th + TPL * (q0 + i);
                const double2 own = tile[p], oth = recv[HALF - 1 - p];
                zk[i] = h == 0 ? own : oth;
                zp[i] = h == 0 ? oth : own;
                k[i] = h == 0 ? fr + N1 * (i64)p : (N1 - fr) + N1 * (i64)(N2 - 1 - p);
            }
            if (a.mode == 1 && a.real) {
                pair_mode1_real_xn<NX>(a, zk, zp, k, M);
            } else if (a.mode == 0 && a.real) {
                pair_mode0_real_x4(a, zk, zp, k, M);
            } else {
#pragma unroll
                for (int i = 0; i < NX; ++i) {
                    if (a.mode == 0) pair_mode0(a, zk[i], zp[i], k[i], M);
                    else pair_mode1(a, zk[i], zp[i], k[i], M);
                }
            }
#pragma unroll
            for (int i = 0; i < NX; ++i) {
                const int p = th + TPL * (q0 + i);
                tile[p] = h == 0 ? zk[i] : zp[i];
                st_async_peer(peer_smem(tile + (N2 - 1 - p), peer), h == 0 ? zp[i] : zk[i], pbar);
            }
        }
        mbar_wait(&bx2, 0);
#pragma unroll
        for (int q = 0; q < R; ++q) v[q] = tile[th + q * TPL];
        __syncthreads();  // the inverse FFT's exchanges overwrite the tile
    }
    FI::run(v, th, tile, a.tw_all + N2);
#pragma unroll
    for (int q = 0; q < R; ++q) src[th + q * TPL] = v[q];
}

// FSX_ROWPAIR_C=0 keeps the one-CTA row-pair kernel for every N2 (A/B)
static bool rowpair_cluster() {
    static int v = -1;
    if (v < 0) {
        const char* e = getenv("FSX_ROWPAIR_C");
        v = e ? atoi(e) : 1;
    }
    return v != 0;
}

template <int N2>
static cudaError_t rowpair_n(const RowPairArgs& a, cudaStream_t s) {
    // measured: cfg5 (N2 = 4096) row-pair pass 1.62 -> 1.44 ms; cfg1 (N2 = 1024,
    // 64-thread CTAs) 28.8 -> 39.0 us, so only the 4096-point rows take the pair
    if constexpr (N2 == 4096) {
        if (rowpair_cluster() && a.N1 >= 4) {
            const size_t smem = (size_t)(N2 + N2 / 2) * sizeof(double2);
            kernel_prepare((const void*)k_rowpair_c<N2>, smem);
            return launch_pdl_cluster(k_rowpair_c<N2>, dim3((unsigned)a.N1), dim3(N2 / 16), smem, s, a);
        }
    }
    using C = Cfg<N2>;
    constexpr int LS = N2 + ((C::TPL >= 8) ? 0 : 8 / (8 / C::TPL > 2 ? 2 : 8 / C::TPL));
    const size_t smem = (size_t)2 * LS * sizeof(double2);
    kernel_prepare((const void*)k_rowpair<N2>, smem);
    const i64 ctas = a.N1 / 2 + 1;
    k_rowpair<N2><<<(unsigned)(a.N1 == 1 ? 1 : ctas), 2 * C::TPL, smem, s>>>(a);
    return cudaGetLastError();
}

cudaError_t launch_rowpair(const RowPairArgs& a, cudaStream_t s) {
    switch (a.N2) {
#define C_(N) case N: return rowpair_n<N>(a, s);
        FSX_POW2_CASES(C_)
#undef C_
        default: return cudaErrorInvalidValue;
    }
}

cudaError_t launch_promote(const double* x, double2* z, i64 n, cudaStream_t s) {
    k_promote<<<grid_for(n, 256), 256, 0, s>>>(x, z, n);
    return cudaGetLastError();
}

cudaError_t launch_extract(const double2* z, double* x, i64 n, Flags* f, cudaStream_t s) {
    k_extract<<<grid_for(n, 256), 256, 0, s>>>(z, x, n, f);
    return cudaGetLastError();
}

// fp32 storage mode around the fp64 plans that have no fp32 row kernels
__global__ void k_widen(const float* __restrict__ x, double* __restrict__ y, i64 n) {
    for (i64 i = blockIdx.x * (i64)blockDim.x + threadIdx.x; i < n; i += (i64)gridDim.x * blockDim.x) y[i] = x[i];
}
__global__ void k_narrow(const double* __restrict__ x, float* __restrict__ y, i64 n, Flags* flags) {
    bool bad = false;
    for (i64 i = blockIdx.x * (i64)blockDim.x + threadIdx.x; i < n; i += (i64)gridDim.x * blockDim.x) {
        const float f = (float)x[i];
        y[i] = f;
        bad |= !isfinite(f);
    }
    flag_nonfinite(bad, flags);
}

cudaError_t launch_widen(const float* x, double* y, i64 n, cudaStream_t s) {
    k_widen<<<grid_for(n, 256), 256, 0, s>>>(x, y, n);
    return cudaGetLastError();
}

cudaError_t launch_narrow(const double* x, float* y, i64 n, Flags* f, cudaStream_t s) {
    k_narrow<<<grid_for(n, 256), 256, 0, s>>>(x, y, n, f);
    return cudaGetLastError();
}

cudaError_t launch_finite_check(const double* x, i64 n, Flags* f, cudaStream_t s) {
    k_finite<<<grid_for(n, 256), 256, 0, s>>>(x, n, f);
    return cudaGetLastError();
}

__global__ void k_scale(double2* z, i64 n, double sc) {
    for (i64 i = (i64)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (i64)gridDim.x * blockDim.x)
        z[i] = cscale(z[i], sc);
}

cudaError_t launch_scale(double2* z, i64 n, double scale, cudaStream_t s) {
    k_scale<<<grid_for(n, 256), 256, 0, s>>>(z, n, scale);
    return cudaGetLastError();
}

cudaError_t launch_spectral_general(double2* z, const GeneralSymbol& sym, cudaStream_t s) {
    const int g = grid_for(sym.cells, 128);
    switch (sym.m) {
        case 1: k_spectral_general<1><<<g, 128, 0, s>>>(z, sym); break;
        case 2: k_spectral_general<2><<<g, 128, 0, s>>>(z, sym); break;
        case 3: k_spectral_general<3><<<g, 128, 0, s>>>(z, sym); break;
        case 4: k_spectral_general<4><<<g, 128, 0, s>>>(z, sym); break;
        case 5: k_spectral_general<5><<<g, 128, 0, s>>>(z, sym); break;
        case 6: k_spectral_general<6><<<g, 128, 0, s>>>(z, sym); break;
        case 7: k_spectral_general<7><<<g, 128, 0, s>>>(z, sym); break;
        case 8: k_spectral_general<8><<<g, 128, 0, s>>>(z, sym); break;
        default: return cudaErrorInvalidValue;
    }
    return cudaGetLastError();
}

cudaError_t launch_symbol_blocks(double2* out, const GeneralSymbol& sym, int which_q, cudaStream_t s) {
    const int g = grid_for(sym.cells, 128);
    switch (sym.m) {
        case 1: k_symbol_blocks<1><<<g, 128, 0, s>>>(out, sym, which_q); break;
        case 2: k_symbol_blocks<2><<<g, 128, 0, s>>>(out, sym, which_q); break;
        case 3: k_symbol_blocks<3><<<g, 128, 0, s>>>(out, sym, which_q); break;
        case 4: k_symbol_blocks<4><<<g, 128, 0, s>>>(out, sym, which_q); break;
        case 5: k_symbol_blocks<5><<<g, 128, 0, s>>>(out, sym, which_q); break;
        case 6: k_symbol_blocks<6><<<g, 128, 0, s>>>(out, sym, which_q); break;
        case 7: k_symbol_blocks<7><<<g, 128, 0, s>>>(out, sym, which_q); break;
        case 8: k_symbol_blocks<8><<<g, 128, 0, s>>>(out, sym, which_q); break;
        default: return cudaErrorInvalidValue;
    }
    return cudaGetLastError();
}

cudaError_t launch_symbol_absmax(const GeneralSymbol& sym, double* out_max, cudaStream_t s) {
    k_symbol_absmax<<<grid_for(sym.cells, 128), 128, 0, s>>>(sym, reinterpret_cast<unsigned long long*>(out_max));
    return cudaGetLastError();
}

cudaError_t launch_pow_blocks(const double2* in, double2* out, i64 cells, int m, u64 T, cudaStream_t s) {
    const int g = grid_for(cells, 128);
    switch (m) {
        case 1: k_pow_blocks<1><<<g, 128, 0, s>>>(in, out, cells, T); break;
        case 2: k_pow_blocks<2><<<g, 128, 0, s>>>(in, out, cells, T); break;
        case 3: k_pow_blocks<3><<<g, 128, 0, s>>>(in, out, cells, T); break;
        case 4: k_pow_blocks<4><<<g, 128, 0, s>>>(in, out, cells, T); break;
        case 5: k_pow_blocks<5><<<g, 128, 0, s>>>(in, out, cells, T); break;
        case 6: k_pow_blocks<6><<<g, 128, 0, s>>>(in, out, cells, T); break;
        case 7: k_pow_blocks<7><<<g, 128, 0, s>>>(in, out, cells, T); break;
        case 8: k_pow_blocks<8><<<g, 128, 0, s>>>(in, out, cells, T); break;
        default: return cudaErrorInvalidValue;
    }
    return cudaGetLastError();
}

cudaError_t launch_absmax(const double2* in, i64 n, double* out_max, cudaStream_t s) {
    k_absmax<<<grid_for(n, 256), 256, 0, s>>>(in, n, reinterpret_cast<unsigned long long*>(out_max));
    return cudaGetLastError();
}

cudaError_t launch_pinv(const double2* in, double2* out, i64 n, const double* maxabs, cudaStream_t s) {
    k_pinv<<<grid_for(n, 256), 256, 0, s>>>(in, out, n, maxabs);
    return cudaGetLastError();
}

cudaError_t launch_block_mul(const double2* a, const double2* b, double2* out, i64 cells, int m, cudaStream_t s) {
    const int g = grid_for(cells, 128);
    switch (m) {
        case 1: k_block_mul<1><<<g, 128, 0, s>>>(a, b, out, cells); break;
        case 2: k_block_mul<2><<<g, 128, 0, s>>>(a, b, out, cells); break;
        case 3: k_block_mul<3><<<g, 128, 0, s>>>(a, b, out, cells); break;
        case 4: k_block_mul<4><<<g, 128, 0, s>>>(a, b, out, cells); break;
        case 5: k_block_mul<5><<<g, 128, 0, s>>>(a, b, out, cells); break;
        case 6: k_block_mul<6><<<g, 128, 0, s>>>(a, b, out, cells); break;
        case 7: k_block_mul<7><<<g, 128, 0, s>>>(a, b, out, cells); break;
        case 8: k_block_mul<8><<<g, 128, 0, s>>>(a, b, out, cells); break;
        default: return cudaErrorInvalidValue;
    }
    return cudaGetLastError();
}

cudaError_t launch_block_matvec(const double2* lam, const double2* x, double2* y, i64 cells, int m, cudaStream_t s) {
    const int g = grid_for(cells, 128);
    switch (m) {
        case 1: k_block_matvec<1><<<g, 128, 0, s>>>(lam, x, y, cells); break;
        case 2: k_block_matvec<2><<<g, 128, 0, s>>>(lam, x, y, cells); break;
        case 3: k_block_matvec<3><<<g, 128, 0, s>>>(lam, x, y, cells); break;
        case 4: k_block_matvec<4><<<g, 128, 0, s>>>(lam, x, y, cells); break;
        case 5: k_block_matvec<5><<<g, 128, 0, s>>>(lam, x, y, cells); break;
        case 6: k_block_matvec<6><<<g, 128, 0, s>>>(lam, x, y, cells); break;
        case 7: k_block_matvec<7><<<g, 128, 0, s>>>(lam, x, y, cells); break;
        case 8: k_block_matvec<8><<<g, 128, 0, s>>>(lam, x, y, cells); break;
        default: return cudaErrorInvalidValue;
    }
    return cudaGetLastError();
}

cudaError_t launch_transpose_split(const double2* in, double2* out, i64 outer, i64 n1, i64 n2, i64 inner,
                                   int to_natural, cudaStream_t s) {
    k_transpose_split<<<grid_for(outer * n1 * n2 * inner, 256), 256, 0, s>>>(in, out, outer, n1, n2, inner, to_natural);
    return cudaGetLastError();
}

}  // namespace fsx
