// Strided-axis passes with TMA (cp.async.bulk.tensor) column I/O.
//
// A column of the half spectrum is N complex values 16 B apart at a stride
// of a full row (P * 16 B).  Loaded with per-thread LDG/STG, every warp
// instruction touches 16-32 different rows, and the round-1 profile of the
// fused pass showed the LSU queue saturating (stall_lg + drain ~35 % of
// samples).  Here one elected thread moves the whole column with
// N / 256 TMA box copies ({2 doubles} x {256 rows}) into a linear
// shared-memory tile (mbarrier completion), the CTA transforms it, and the
// result leaves the same way (bulk store from shared memory).  The tile
// doubles as the FFT exchange buffer, so a CTA needs N * 16 B of shared
// memory and two CTAs share an SM (one loads while the other computes).
//
// Tensor map: the complex array viewed as fp64 [outer][n][2 * inner]
// (dims {2 * inner, n, outer}), box {2, min(n, 256), 1}; built on the host
// (fsx_api.cpp) with cuTensorMapEncodeTiled.
#include <cuda.h>

#include <algorithm>
#include <cstdlib>
#include <cstring>

#include "fsx_async.cuh"
#include "fsx_device.cuh"
#include "fsx_kernels.h"
#include "fsx_spectral.cuh"

namespace fsx {

template <int N, int WW = 0>
struct TCfg {
    static constexpr int R = N < 16 ? N : 16;
    static constexpr int TPL = N / R;
    static constexpr int W = WW ? WW : (N >= 4096 ? 1 : 4096 / N);   // adjacent columns per CTA (64 KB tile)
    static constexpr int BOX = N < 256 ? N : 256;        // rows per TMA box
    static constexpr int NBOX = N / BOX;
    static constexpr int GW = W < 8 ? W : 8;
    static constexpr int LSW = GW > 1 ? N + 8 / GW : N;  // exchange line stride (bank padding)
    static constexpr int NT = W * TPL;
    static constexpr int MINB = NT <= 256 ? 2 : 1;
    static constexpr bool PRE = N <= 4096;                // fused mode: real multipliers in smem
    static constexpr size_t smem(int mode) {
        return (size_t)W * LSW * 16 + ((mode == 2 || mode == 4) && PRE ? (size_t)NT * R * 8 : 0);
    }
};

// MODE 0: forward C2C, 1: inverse C2C, 2: fused R2C spectral pass, 4: the
// same with an implicit (pinv(lamQ) lamS) real symbol, 3: copy only.
// The TMA tile is [N rows][W columns] (row-major, as the boxes land); the
// FFT exchanges reuse the same buffer as W line-major rows of LSW.
template <int N, int MODE, int WW = 0>
__global__ void __launch_bounds__(TCfg<N, WW>::NT, TCfg<N, WW>::MINB)
k_cols_tma(const __grid_constant__ CUtensorMap map, AxisGeom g, FusedSymbol sym, const double2* __restrict__ tw_all) {
    using C = TCfg<N, WW>;
    constexpr bool FUSED = MODE == 2 || MODE == 4;  // 4: implicit symbol (pinv(lamQ) lamS)
    constexpr int W = C::W;
    // full twiddle tables for the multi-column tiles (N < 4096); the one-column
    // 4096 tiles measured faster with derived twiddles (cfg2 158 vs 165 us)
#ifndef FSX_FT4096
#define FSX_FT4096 0
#endif
    constexpr int FT = N < 4096 ? ~0 : FSX_FT4096;
#ifndef FSX_COLS_LPF
#define FSX_COLS_LPF 0
#endif
    using FF = LineFFT<N, -1, false, false, FT, 0, double2, FSX_COLS_LPF != 0>;
    using FI = LineFFT<N, +1, false, false, FT, 0, double2, FSX_COLS_LPF != 0>;
    extern __shared__ __align__(128) double2 tile[];
    __shared__ __align__(8) unsigned long long bar;
    __shared__ double2 acoef[kMaxGroups][W];
    __shared__ double2 tapterm[MODE >= 2 ? kMaxFusedTaps : 1][W];
    const int w = threadIdx.x % W, t = threadIdx.x / W;
    const i64 tiles = (g.ncols + W - 1) / W;
    const i64 o = (i64)blockIdx.x / tiles;
    const i64 c0 = ((i64)blockIdx.x - o * tiles) * W;
    const i64 c = c0 + w;
    i64 kx = c, ky = 0;
    if constexpr (FUSED) {
        fused_col_freqs(sym, c, kx, ky);
        // pitch-padding tiles of a 3D plane (W divides P, so a tile is all-padding or none)
        if (c0 - (c0 / sym.P) * sym.P > sym.M && sym.rank == 3) return;
    }
    if (threadIdx.x == 0) {
        mbar_init(&bar, 1);
        mbar_init_fence();
        pdl_wait();  // the tile is the predecessor's output (PDL: everything above overlaps its tail)
        mbar_expect_tx(&bar, (unsigned)(N * W * sizeof(double2)));
#pragma unroll 1
        for (int b = 0; b < C::NBOX; ++b)
            tma_load_3d(tile + b * C::BOX * W, &map, (int)(2 * c0), b * C::BOX, (int)o, &bar);
    }
    // MODE 2, real symbol: lam(k0)^T * scale for this thread's 16 frequencies is
    // data independent -- computed while the tile is in flight and parked in
    // shared memory (mult[q * NT + thread], thread-private) for after the FFT.
    // (Under PDL the first-wave CTAs wait for the producer thread's pdl_wait at
    // the first barrier; per-thread group sums without that barrier measured
    // slower on the rank-3 symbol: cfg4 7.25 -> 8.05 ms.)
    // Not for the 128 KB tiles (N = 8192): the extra 64 KB would squeeze the
    // L1 that serves the table reads (cfg3 measured 0.87 -> 1.04 ms); parking
    // them in tensor memory instead measured neutral.
    constexpr bool PRE = FUSED && C::PRE;
    double* mult = reinterpret_cast<double*>(tile + W * C::LSW);
    // every multiplier of this warp's columns is a host-proved 0 (FusedSymbol::kzero); warp-uniform,
    // because the power's short cut votes across the warp
    // (evaluated where it is used, so that no flag stays live across the FFTs)
    auto is_dead = [&]() -> bool {
        // one-column tiles only: in the multi-column kernels (N < 4096; cfg4's 1024-point columns,
        // where no column is provably 0 anyway) the extra branch costs spills (ptxas: 168 -> 448 B)
        if constexpr (MODE != 2 || W != 1) return false;
        i64 kx2 = c, ky2 = 0;
        fused_col_freqs(sym, c, kx2, ky2);
        return __all_sync(0xffffffffu, kx2 > sym.kzero);
    };
    if constexpr (FUSED) {
        for (int j = t; j < sym.ntaps; j += C::TPL) tapterm[j][w] = tap_term(sym, tw_all, j, kx, ky);
    }
    __syncthreads();  // barrier initialised before anyone waits on it; tap terms visible
    if constexpr (FUSED) {
        for (int gi = t; gi < sym.ngroups; gi += C::TPL) {
            double2 a = make_double2(0.0, 0.0);
            for (int j = 0; j < sym.ntaps; ++j)
                if (sym.tap_group[j] == gi) a = cadd(a, tapterm[j][w]);
            acoef[gi][w] = a;
        }
        __syncthreads();
        if (PRE && sym.real) {
            if (is_dead()) {
                const double z = 0.0 * sym.scale;
#pragma unroll
                for (int q = 0; q < C::R; ++q) mult[q * C::NT + threadIdx.x] = z;
            } else {
                double lam[C::R];
                symbol_real<N, C::R, C::TPL, MODE == 4>(lam, t, sym, tw_all, [&](int gi) { return acoef[gi][w]; });
                pow_real_vec_skip<C::R, 4>(lam, sym.T, sym.neg_mag2);
#pragma unroll
                for (int q = 0; q < C::R; ++q) mult[q * C::NT + threadIdx.x] = lam[q] * sym.scale;
            }
        }
    }
    mbar_wait(&bar, 0);
    pdl_trigger();  // the successor may start its own prologue
    double2 v[C::R];
#pragma unroll
    for (int q = 0; q < C::R; ++q) v[q] = tile[(t + q * C::TPL) * W + w];
    double2* line = tile + w * C::LSW;
    if constexpr (MODE == 3) {
        // copy-only (measurement of the TMA column I/O alone)
    } else if constexpr (MODE == 1) {
        FI::run(v, t, line, tw_all + N);
    } else {
        FF::run(v, t, line, tw_all + N);
    }
    if constexpr (FUSED) {
        if (PRE && sym.real) {
#pragma unroll
            for (int q = 0; q < C::R; ++q) v[q] = cscale(v[q], mult[q * C::NT + threadIdx.x]);
        } else if (is_dead()) {
            // lam = 0 for the whole column: the products spectral_regs would form with it
#pragma unroll
            for (int q = 0; q < C::R; ++q) v[q] = zero_products(v[q], sym.real != 0);
        } else {
            spectral_regs<N, C::R, C::TPL>(v, t, sym, tw_all, [&](int gi) { return acoef[gi][w]; });
        }
        FI::run(v, t, line, tw_all + N);
    }
    __syncthreads();  // last exchange reads done before the tile is overwritten
#pragma unroll
    for (int q = 0; q < C::R; ++q) tile[(t + q * C::TPL) * W + w] = v[q];
    fence_proxy_async();
    __syncthreads();
    if (threadIdx.x == 0) {
#pragma unroll 1
        for (int b = 0; b < C::NBOX; ++b) tma_store_3d(&map, tile + b * C::BOX * W, (int)(2 * c0), b * C::BOX, (int)o);
        bulk_commit();
        bulk_wait_read0();
    }
}

// fp32 arithmetic for the fp32 mode's fused pass (real symbols, N <= 4096).
// The tile arrives and leaves as fp64 (the row passes are unchanged); the two
// FFTs run on float2 with a float2 copy of the twiddle tables, exchanging
// through the same tile viewed as float2 lines; the multipliers lam^T / N are
// computed in fp64 as in MODE 2 (the symbol power is where fp32 would lose
// the accuracy) and rounded once.  This takes the pass off
// the FP64 pipe that bounds the fp64 version; what is left is the TMA row rate.
// MODE 2: the fused pass; 0 / 1: a forward / inverse C2C pass (the 3D y passes).
template <int N, int MODE>
__global__ void __launch_bounds__(TCfg<N>::NT, TCfg<N>::MINB)
k_cols_tma_f32(const __grid_constant__ CUtensorMap map, AxisGeom g, FusedSymbol sym, const double2* __restrict__ tw_all,
               const float2* __restrict__ twf_all) {
    using C = TCfg<N>;
    constexpr int W = C::W;
    constexpr int FT = N < 4096 ? ~0 : 0;
    using FF = LineFFT<N, -1, false, false, FT, 0, float2>;
    using FI = LineFFT<N, +1, false, false, FT, 0, float2>;
    extern __shared__ __align__(128) double2 tile[];
    __shared__ __align__(8) unsigned long long bar;
    __shared__ double2 acoef[kMaxGroups][W];
    __shared__ double2 tapterm[kMaxFusedTaps][W];
    const int w = threadIdx.x % W, t = threadIdx.x / W;
    const i64 tiles = (g.ncols + W - 1) / W;
    const i64 o = (i64)blockIdx.x / tiles;
    const i64 c0 = ((i64)blockIdx.x - o * tiles) * W;
    const i64 c = c0 + w;
    i64 kx = c, ky = 0;
    if constexpr (MODE == 2) {
        fused_col_freqs(sym, c, kx, ky);
        if (c0 - (c0 / sym.P) * sym.P > sym.M && sym.rank == 3) return;  // pitch-padding tiles of a 3D plane
    }
    if (threadIdx.x == 0) {
        mbar_init(&bar, 1);
        mbar_init_fence();
        pdl_wait();
        mbar_expect_tx(&bar, (unsigned)(N * W * sizeof(double2)));
#pragma unroll 1
        for (int b = 0; b < C::NBOX; ++b)
            tma_load_3d(tile + b * C::BOX * W, &map, (int)(2 * c0), b * C::BOX, (int)o, &bar);
    }
    float* mult = reinterpret_cast<float*>(tile + W * C::LSW);
    if constexpr (MODE == 2) {
        for (int j = t; j < sym.ntaps; j += C::TPL) tapterm[j][w] = tap_term(sym, tw_all, j, kx, ky);
    }
    __syncthreads();
    if constexpr (MODE == 2) {
        for (int gi = t; gi < sym.ngroups; gi += C::TPL) {
            double2 a = make_double2(0.0, 0.0);
            for (int j = 0; j < sym.ntaps; ++j)
                if (sym.tap_group[j] == gi) a = cadd(a, tapterm[j][w]);
            acoef[gi][w] = a;
        }
        __syncthreads();
        double lam[C::R];
        symbol_real<N, C::R, C::TPL, false>(lam, t, sym, tw_all, [&](int gi) { return acoef[gi][w]; });
        pow_real_vec_skip<C::R, 4>(lam, sym.T, sym.neg_mag2);
#pragma unroll
        for (int q = 0; q < C::R; ++q) mult[q * C::NT + threadIdx.x] = (float)(lam[q] * sym.scale);
    }
    mbar_wait(&bar, 0);
    pdl_trigger();
    float2 v[C::R];
#pragma unroll
    for (int q = 0; q < C::R; ++q) {
        const double2 d = tile[(t + q * C::TPL) * W + w];
        v[q] = make_float2((float)d.x, (float)d.y);
    }
    float2* line = reinterpret_cast<float2*>(tile) + w * C::LSW;  // the first exchange is behind a barrier
    if constexpr (MODE == 1) {
        FI::run(v, t, line, twf_all + N);
    } else {
        FF::run(v, t, line, twf_all + N);
    }
    if constexpr (MODE == 2) {
#pragma unroll
        for (int q = 0; q < C::R; ++q) v[q] = cscale(v[q], mult[q * C::NT + threadIdx.x]);
        FI::run(v, t, line, twf_all + N);
    }
    __syncthreads();  // last exchange reads done before the tile is overwritten
#pragma unroll
    for (int q = 0; q < C::R; ++q) tile[(t + q * C::TPL) * W + w] = make_double2(v[q].x, v[q].y);
    fence_proxy_async();
    __syncthreads();
    if (threadIdx.x == 0) {
#pragma unroll 1
        for (int b = 0; b < C::NBOX; ++b) tma_store_3d(&map, tile + b * C::BOX * W, (int)(2 * c0), b * C::BOX, (int)o);
        bulk_commit();
        bulk_wait_read0();
    }
}

template <int N, int MODE>
static cudaError_t cols_tma_f32_n(const CUtensorMap& map, const AxisGeom& g, const FusedSymbol& sym, const double2* tw,
                                  const float2* twf, cudaStream_t s) {
    using C = TCfg<N>;
    const size_t smem = (size_t)C::W * C::LSW * 16 + (MODE == 2 ? (size_t)C::NT * C::R * 4 : 0);
    const i64 tiles = (g.ncols + C::W - 1) / C::W;
    auto kf = k_cols_tma_f32<N, MODE>;
    kernel_prepare((const void*)kf, smem);
    return launch_pdl(kf, dim3((unsigned)(g.outer * tiles)), dim3(C::NT), smem, s, map, g, sym, tw, twf);
}

// FSX_F32_COMPUTE=0 keeps the fp32 mode's fused pass in fp64 arithmetic (A/B)
bool f32_compute_enabled() {
    static int v = -1;
    if (v < 0) {
        const char* e = getenv("FSX_F32_COMPUTE");
        v = e ? atoi(e) : 1;
    }
    return v != 0;
}

cudaError_t launch_cols_tma_f32(const void* tensor_map, const AxisGeom& g, int mode, const FusedSymbol& sym,
                                const double2* tw, const float2* twf, cudaStream_t s) {
    const CUtensorMap& map = *reinterpret_cast<const CUtensorMap*>(tensor_map);
#define FSX_TMAF(N)                                                                  \
    case N:                                                                          \
        return mode == 0 ? cols_tma_f32_n<N, 0>(map, g, sym, tw, twf, s)             \
             : mode == 1 ? cols_tma_f32_n<N, 1>(map, g, sym, tw, twf, s)             \
                         : cols_tma_f32_n<N, 2>(map, g, sym, tw, twf, s);
    switch (g.n) {
        FSX_TMAF(512)
        FSX_TMAF(1024)
        FSX_TMAF(2048)
        FSX_TMAF(4096)
        default: return cudaErrorInvalidValue;
    }
#undef FSX_TMAF
}

// C2C strided pass with TMA column I/O for the general axis launcher
// (launch_axis_pow2): optional four-step twiddle (TWM 1: post-multiply by
// W^(b k), 2: pre-multiply by its conjugate; b = column / col_div, exponent as
// StepTwiddle), out of place (separate load / store maps), and the solve's
// non-finite scan on its output when `flags` is set.  Used by the 1D plan's
// column FFTs (128-point columns for cfg5, 512 for cfg1).
// WW: columns per tile (0: the 64 KB default, 4096 / N; a narrower tile gives
// small problems more CTAs than SMs, see launch_axis_tma).
template <int N, int SIGN, int TWM, int WW = 0>
__global__ void __launch_bounds__(TCfg<N, WW>::NT, TCfg<N, WW>::MINB)
k_axis_tma(const __grid_constant__ CUtensorMap map_in, const __grid_constant__ CUtensorMap map_out, AxisGeom g,
           StepTwiddle st, const double2* __restrict__ tw_all, Flags* flags) {
    using C = TCfg<N, WW>;
    constexpr int W = C::W;
    using F = LineFFT<N, SIGN, false, false, (N < 4096 ? ~0 : 0)>;
    extern __shared__ __align__(128) double2 tile[];
    __shared__ __align__(8) unsigned long long bar;
    const int w = threadIdx.x % W, t = threadIdx.x / W;
    const i64 tiles = (g.ncols + W - 1) / W;
    const i64 o = (i64)blockIdx.x / tiles;
    const i64 c0 = ((i64)blockIdx.x - o * tiles) * W;
    const i64 c = c0 + w;
    if (threadIdx.x == 0) {
        mbar_init(&bar, 1);
        mbar_init_fence();
        pdl_wait();
        mbar_expect_tx(&bar, (unsigned)(N * W * sizeof(double2)));
#pragma unroll 1
        for (int b = 0; b < C::NBOX; ++b) tma_load_3d(tile + b * C::BOX * W, &map_in, (int)(2 * c0), b * C::BOX, (int)o, &bar);
    }
    __syncthreads();
    mbar_wait(&bar, 0);
    pdl_trigger();
    double2 v[C::R];
#pragma unroll
    for (int q = 0; q < C::R; ++q) v[q] = tile[(t + q * C::TPL) * W + w];
    // twiddles as an arithmetic progression of exponents: base and ratio reads
    // and a running product (see k_strided)
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
    F::run(v, t, tile + w * C::LSW, tw_all + N);
    if constexpr (TWM == 1) {
#pragma unroll
        for (int q = 0; q < C::R; ++q) {
            v[q] = cmul(v[q], tq);
            tq = cmul(tq, tr);
        }
    }
    if (flags) {
        bool bad = false;
#pragma unroll
        for (int q = 0; q < C::R; ++q) bad |= c < g.ncols && (!isfinite(v[q].x) || !isfinite(v[q].y));
        flag_nonfinite(bad, flags);
    }
    __syncthreads();  // last exchange reads done before the tile is overwritten
#pragma unroll
    for (int q = 0; q < C::R; ++q) tile[(t + q * C::TPL) * W + w] = v[q];
    fence_proxy_async();
    __syncthreads();
    if (threadIdx.x == 0) {
#pragma unroll 1
        for (int b = 0; b < C::NBOX; ++b) tma_store_3d(&map_out, tile + b * C::BOX * W, (int)(2 * c0), b * C::BOX, (int)o);
        bulk_commit();
        bulk_wait_read0();
    }
}

static int axis_tma_enabled() {
    static int v = -1;
    if (v < 0) {
        const char* e = getenv("FSX_TMA_AXIS");
        v = e ? atoi(e) : 512;
    }
    return v;
}

template <int N, int SIGN, int TWM, int WW>
static cudaError_t axis_tma_nst(const CUtensorMap& mi, const CUtensorMap& mo, const AxisGeom& g, const StepTwiddle& st,
                                const double2* tw, Flags* f, cudaStream_t s) {
    using C = TCfg<N, WW>;
    const size_t smem = (size_t)C::W * C::LSW * sizeof(double2);
    const i64 tiles = (g.ncols + C::W - 1) / C::W;
    auto kf = k_axis_tma<N, SIGN, TWM, WW>;
    kernel_prepare((const void*)kf, smem);
    return launch_pdl(kf, dim3((unsigned)(g.outer * tiles)), dim3(C::NT), smem, s, mi, mo, g, st, tw, f);
}

template <int N, int WW = 0>
static cudaError_t axis_tma_n(const CUtensorMap& mi, const CUtensorMap& mo, const AxisGeom& g, int sign,
                              const StepTwiddle& st, const double2* tw, Flags* f, cudaStream_t s) {
    if (sign < 0)
        return st.mode == 1 ? axis_tma_nst<N, -1, 1, WW>(mi, mo, g, st, tw, f, s)
             : st.mode == 2 ? axis_tma_nst<N, -1, 2, WW>(mi, mo, g, st, tw, f, s)
                            : axis_tma_nst<N, -1, 0, WW>(mi, mo, g, st, tw, f, s);
    return st.mode == 1 ? axis_tma_nst<N, +1, 1, WW>(mi, mo, g, st, tw, f, s)
         : st.mode == 2 ? axis_tma_nst<N, +1, 2, WW>(mi, mo, g, st, tw, f, s)
                        : axis_tma_nst<N, +1, 0, WW>(mi, mo, g, st, tw, f, s);
}

// FSX_AXIS_NARROW (default 2; 0 = off): with fewer than two default tiles per
// SM, 512- and 1024-point columns use this many columns per tile instead
static int axis_narrow() {
    static int v = -1;
    if (v < 0) {
        const char* e = getenv("FSX_AXIS_NARROW");
        v = e ? atoi(e) : 2;
    }
    return v;
}

// Returns cudaErrorNotSupported when the TMA path does not apply (the caller
// falls back to the per-thread strided kernel).
cudaError_t launch_axis_tma(const double2* in, double2* out, const AxisGeom& g, int sign, const StepTwiddle& st,
                            const double2* tw, cudaStream_t s, Flags* flags) {
    // FSX_TMA_AXIS (default 512): the shortest column length taken by this path
    const int nmin = axis_tma_enabled();
    if (!nmin || g.inner <= 1 || g.n < nmin || g.n > 4096) return cudaErrorNotSupported;
    int W = tma_cols_width(g.n);
    static int sms = 0;
    if (!sms) {
        int dev = 0;
        cudaGetDevice(&dev);
        cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
        if (sms <= 0) sms = 148;
    }
    const int nw = axis_narrow();
    const bool narrow = (g.n == 512 || g.n == 1024) && (nw == 2 || nw == 4) && nw < W &&
                        g.outer * (g.ncols / W) < 2 * (i64)sms && g.ncols % nw == 0;
    if (narrow) W = nw;
    if (g.ncols % W || (reinterpret_cast<uintptr_t>(in) | reinterpret_cast<uintptr_t>(out)) % 16) return cudaErrorNotSupported;
    alignas(64) unsigned char mi[128], mo[128];
    if (make_cols_tensor_map_w(mi, const_cast<double2*>(in), g, W) != 0) return cudaErrorNotSupported;
    if (out == in) std::memcpy(mo, mi, sizeof mo);
    else if (make_cols_tensor_map_w(mo, out, g, W) != 0) return cudaErrorNotSupported;
    const CUtensorMap& MI = *reinterpret_cast<const CUtensorMap*>(mi);
    const CUtensorMap& MO = *reinterpret_cast<const CUtensorMap*>(mo);
    if (narrow) {
        if (g.n == 512) return W == 2 ? axis_tma_n<512, 2>(MI, MO, g, sign, st, tw, flags, s)
                                      : axis_tma_n<512, 4>(MI, MO, g, sign, st, tw, flags, s);
        return axis_tma_n<1024, 2>(MI, MO, g, sign, st, tw, flags, s);
    }
    switch (g.n) {
        case 128: return axis_tma_n<128>(MI, MO, g, sign, st, tw, flags, s);
        case 256: return axis_tma_n<256>(MI, MO, g, sign, st, tw, flags, s);
        case 512: return axis_tma_n<512>(MI, MO, g, sign, st, tw, flags, s);
        case 1024: return axis_tma_n<1024>(MI, MO, g, sign, st, tw, flags, s);
        case 2048: return axis_tma_n<2048>(MI, MO, g, sign, st, tw, flags, s);
        case 4096: return axis_tma_n<4096>(MI, MO, g, sign, st, tw, flags, s);
        default: return cudaErrorNotSupported;
    }
}

// Spectral multiply of the 8192-point halves passes: v[q] = X[k0],
// k0 = th + 256 q + 4096 h = th + 256 b + 2048 (a + 2 h) for q = 8 a + b, so
// exp(2 pi i og k0 / 8192) = e_b i^(og (a + 2 h)): eight reads per group, all
// in the table's first 2048 entries, and exact quarter turns.
__device__ __forceinline__ void spectral_halves(double2 (&v)[16], int th, int h, const FusedSymbol& sym,
                                                const double2* __restrict__ tw_all, const double2* acoef) {
    constexpr int N = 8192, NH = 4096;
    if (sym.real) {
        double lam[16];
#pragma unroll
        for (int q = 0; q < 16; ++q) lam[q] = 0.0;
        for (int gi = 0; gi < sym.ngroups; ++gi) {
            const double2 a = acoef[gi];
            const i64 og = sym.group_off[gi];
            if (og == 0) {
#pragma unroll
                for (int q = 0; q < 16; ++q) lam[q] += a.x;
                continue;
            }
            double2 eb[8];
#pragma unroll
            for (int b = 0; b < 8; ++b) eb[b] = eplus_tab(tw_all, N, (i64)(th + 256 * b) * og);
            const int mo = (int)(og & 3);
#pragma unroll
            for (int q = 0; q < 16; ++q) {
                const double2 e = rot_quarter(eb[q & 7], (mo * ((q >> 3) + 2 * h)) & 3);
                lam[q] = fma(a.x, e.x, fma(-a.y, e.y, lam[q]));
            }
        }
        pow_real_vec_skip<16, 4>(lam, sym.T, sym.neg_mag2);
#pragma unroll
        for (int q = 0; q < 16; ++q) v[q] = cscale(v[q], lam[q] * sym.scale);
    } else {
        spectral_regs_at<N, 16>(v, th + NH * h, 256, sym, tw_all, [&](int gi) { return acoef[gi]; });
    }
}

// Fused spectral pass for 8192-point columns as two 4096-point halves.
// A 128 KB column tile fits one CTA per SM, whose CTA-wide barriers then
// serialize every FFT phase of the SM.  Here the CTA splits the column by
// sample parity (x[2n], x[2n+1]: a 4-D tensor map {2 inner, parity, n/2,
// outer} loads each half contiguously) and two 256-thread groups run
// independent 4096-point FFTs with named barriers, so one group's exchanges
// overlap the other's arithmetic.  The radix-2 step joins them through
// shared memory: X[k] = E[k] + W^k O[k], X[k + 4096] = E[k] - W^k O[k]
// (group h then owns frequencies k + 4096 h), spectral multiply, and the
// inverse split e = X[k] + X[k+4096], o = (X[k] - X[k+4096]) W^-k feeds the
// two inverse FFTs whose outputs are again the even / odd samples.
__global__ void __launch_bounds__(512, 1)
k_fused8192h(const __grid_constant__ CUtensorMap map2, AxisGeom g, FusedSymbol sym, const double2* __restrict__ tw_all) {
    constexpr int N = 8192, NH = 4096, TH = 256;
    using FF = LineFFT<NH, -1, false, false, false, TH>;
    using FI = LineFFT<NH, +1, false, false, false, TH>;
    extern __shared__ __align__(128) double2 tile[];
    __shared__ __align__(8) unsigned long long bar[2];  // one per parity half: a group starts on its own half
    __shared__ double2 acoef[kMaxGroups];
    __shared__ double2 tapterm[kMaxFusedTaps];
    const int h = threadIdx.x >> 8, th = threadIdx.x & (TH - 1);
    const i64 c = blockIdx.x;
    i64 kx, ky;
    fused_col_freqs(sym, c, kx, ky);
    if (sym.rank == 3 && c - (c / sym.P) * sym.P > sym.M) return;  // pitch padding of a 3D plane
    if (threadIdx.x == 0) {
        mbar_init(&bar[0], 1);
        mbar_init(&bar[1], 1);
        mbar_init_fence();
        pdl_wait();
#pragma unroll 1
        for (int p = 0; p < 2; ++p) {
            mbar_expect_tx(&bar[p], (unsigned)(NH * sizeof(double2)));
#pragma unroll 1
            for (int b = 0; b < NH / 256; ++b)
                tma_load_4d(tile + p * NH + b * 256, &map2, (int)(2 * c), p, b * 256, 0, &bar[p]);
        }
    }
    for (int j = threadIdx.x; j < sym.ntaps; j += 2 * TH) tapterm[j] = tap_term(sym, tw_all, j, kx, ky);
    __syncthreads();
    for (int gi = threadIdx.x; gi < sym.ngroups; gi += 2 * TH) {
        double2 a = make_double2(0.0, 0.0);
        for (int j = 0; j < sym.ntaps; ++j)
            if (sym.tap_group[j] == gi) a = cadd(a, tapterm[j]);
        acoef[gi] = a;
    }
    __syncthreads();
    mbar_wait(&bar[h], 0);
    pdl_trigger();
    double2* reg = tile + h * NH;
    const double2* other = tile + (h ^ 1) * NH;
    double2 v[16];
#pragma unroll
    for (int q = 0; q < 16; ++q) v[q] = reg[th + 256 * q];
    FF::run(v, th, reg, tw_all + NH);
    // forward radix-2 join; W_8192^(th + 256 q) = W_8192^th W_32^q
    const double2 wt = __ldg(tw_all + N + th);
    if (h == 1) {
        static_for<0, 16>([&](auto Q) {
            constexpr int q = decltype(Q)::value;
            v[q] = cmul(v[q], cmul_const<q, 32, -1>(wt));
        });
    }
    group_sync<TH>();  // this group's last exchange reads are done
#pragma unroll
    for (int q = 0; q < 16; ++q) reg[th + 256 * q] = v[q];
    __syncthreads();
#pragma unroll
    for (int q = 0; q < 16; ++q) {
        const double2 o = other[th + 256 * q];
        v[q] = h == 0 ? cadd(v[q], o) : csub(o, v[q]);
    }
    spectral_halves(v, th, h, sym, tw_all, acoef);
    __syncthreads();  // both groups done reading the other half
#pragma unroll
    for (int q = 0; q < 16; ++q) reg[th + 256 * q] = v[q];
    __syncthreads();
    if (h == 0) {
#pragma unroll
        for (int q = 0; q < 16; ++q) v[q] = cadd(v[q], other[th + 256 * q]);
    } else {
        static_for<0, 16>([&](auto Q) {
            constexpr int q = decltype(Q)::value;
            v[q] = cmulc(csub(other[th + 256 * q], v[q]), cmul_const<q, 32, -1>(wt));
        });
    }
    __syncthreads();  // the inverse FFTs' exchanges overwrite the halves just read
    FI::run(v, th, reg, tw_all + NH);
    group_sync<TH>();
#pragma unroll
    for (int q = 0; q < 16; ++q) reg[th + 256 * q] = v[q];
    fence_proxy_async();
    group_sync<TH>();  // each group stores its own parity as soon as it is done
    if (th == 0) {
#pragma unroll 1
        for (int b = 0; b < NH / 256; ++b) tma_store_4d(&map2, reg + b * 256, (int)(2 * c), h, b * 256, 0);
        bulk_commit();
        bulk_wait_read0();
    }
}

// ------------------------------------------------------------------ 8192-point columns on a CTA pair
// Spectral multiply of the CTA-pair layout: u[b + 8 s] = X[k0] with
// k0 = th + 256 b + 2048 (h + 2 s), h = the CTA's rank, so
// exp(2 pi i og k0 / 8192) = e_b i^(og (h + 2 s)): eight table reads per group
// (e_b, b < 8) and exact quarter turns.  Four elements at a time
// {b, b + 1} x {s = 0, 1}, so only four multipliers are live next to the 16
// data values (the 16-wide complex multiplier array spilled at 128 registers).
__device__ __forceinline__ void spectral_pair8192(double2 (&u)[16], int th, int h, const FusedSymbol& sym,
                                                  const double2* __restrict__ tw_all, const double2* acoef) {
    constexpr int N = 8192;
#pragma unroll
    for (int c = 0; c < 4; ++c) {
        const int b0 = 2 * c;
        // element i of the chunk: b = b0 + (i & 1), s = i >> 1 -> u[b + 8 s]
        if (sym.real) {
            double lam[4] = {0.0, 0.0, 0.0, 0.0};
            for (int gi = 0; gi < sym.ngroups; ++gi) {
                if (sym.group_partner[gi] < 0) continue;  // -og of a symmetric pair: with +og below
                double2 a = acoef[gi];
                const i64 og = sym.group_off[gi];
                if (og == 0) {
#pragma unroll
                    for (int i = 0; i < 4; ++i) lam[i] += a.x;
                    continue;
                }
                if (sym.group_partner[gi] > 0) a = make_double2(2.0 * a.x, 2.0 * a.y);  // 2 Re(A e)
                const double2 e0 = eplus_tab(tw_all, N, (i64)(th + 256 * b0) * og);
                const double2 e1 = eplus_tab(tw_all, N, (i64)(th + 256 * (b0 + 1)) * og);
                const int mo = (int)(og & 3);
#pragma unroll
                for (int i = 0; i < 4; ++i) {
                    const double2 e = rot_quarter((i & 1) ? e1 : e0, (mo * (h + 2 * (i >> 1))) & 3);
                    lam[i] = fma(a.x, e.x, fma(-a.y, e.y, lam[i]));
                }
            }
            pow_real_vec_skip<4, 4>(lam, sym.T, sym.neg_mag2);
#pragma unroll
            for (int i = 0; i < 4; ++i) {
                const int j = b0 + (i & 1) + 8 * (i >> 1);
                u[j] = cscale(u[j], lam[i] * sym.scale);
            }
        } else {
            double2 lam[4];
#pragma unroll
            for (int i = 0; i < 4; ++i) lam[i] = make_double2(0.0, 0.0);
            for (int gi = 0; gi < sym.ngroups; ++gi) {
                const int pg = sym.group_partner[gi] - 1;  // -1: none
                if (pg == -2) continue;                     // folded into its +og partner
                const double2 a = acoef[gi];
                const i64 og = sym.group_off[gi];
                if (og == 0) {
#pragma unroll
                    for (int i = 0; i < 4; ++i) lam[i] = cadd(lam[i], a);
                    continue;
                }
                const double2 am = pg >= 0 ? acoef[pg] : make_double2(0.0, 0.0);
                const double2 e0 = eplus_tab(tw_all, N, (i64)(th + 256 * b0) * og);
                const double2 e1 = eplus_tab(tw_all, N, (i64)(th + 256 * (b0 + 1)) * og);
                const int mo = (int)(og & 3);
#pragma unroll
                for (int i = 0; i < 4; ++i) {
                    const double2 e = rot_quarter((i & 1) ? e1 : e0, (mo * (h + 2 * (i >> 1))) & 3);
                    lam[i] = cadd(lam[i], cmul(a, e));
                    if (pg >= 0) lam[i] = cadd(lam[i], cmul(am, cconj(e)));
                }
            }
            pow_complex_vec_skip<4, 4>(lam, sym.T, sym.neg_mag2);
#pragma unroll
            for (int i = 0; i < 4; ++i) {
                const int j = b0 + (i & 1) + 8 * (i >> 1);
                u[j] = cscale(cmul(lam[i], u[j]), sym.scale);
            }
        }
    }
}

// Fused spectral pass for 8192-point columns on a 2-CTA cluster.  CTA h of
// the pair owns the samples of parity h (x[2n + h]: the 4-D tensor map view
// {2 inner, parity, n/2, outer}), i.e. a 4096-point half column of 64 KB, so
// two pairs share an SM and one CTA's TMA load / store overlaps another's
// arithmetic (the 128 KB one-CTA-per-column kernel could not overlap them).
//   1. forward 4096-point FFT of the own half: E (h = 0) or O (h = 1); CTA 1
//      applies W_8192^k;
//   2. exchange 1 over DSMEM, 32 KB each way: CTA 0 keeps k < 2048 and sends
//      E[k >= 2048]; CTA 1 keeps k >= 2048 and sends W O[k < 2048]; the
//      radix-2 join X[k] = E + W O, X[k + 4096] = E - W O then runs in
//      registers for the own k;
//   3. symbol^T / N (spectral_pair8192) and the inverse split
//      e[k] = X[k] + X[k + 4096], o[k] = (X[k] - X[k + 4096]) W^-k;
//   4. exchange 2 into the peer's tile (once the peer reports its forward
//      FFT done): CTA 0 collects e, CTA 1 o;
//   5. inverse 4096-point FFT = the output samples of parity h; TMA store.
// The exchanges are st.async stores that complete on the RECEIVER's mbarrier
// (complete_tx, 32 KB expected), and "my tile is free" is one remote mbarrier
// arrive: the only cluster-wide barrier is the start-up one that publishes the
// barrier initialisation (a release cluster barrier per exchange costs a
// GPU-scope fence and an L1 invalidation: ~20 % of the stall samples).
__global__ void __cluster_dims__(2, 1, 1) __launch_bounds__(256, 2)
k_fused8192c(const __grid_constant__ CUtensorMap map2, AxisGeom g, FusedSymbol sym, const double2* __restrict__ tw_all,
             const double2* __restrict__ pf_base, int pf_dist) {
    constexpr int N = 8192, NH = 4096, TH = 256;
#ifndef FSX_F8192_LPF
#define FSX_F8192_LPF 1  // cfg3: fused 0.5829 -> 0.5800 ms (r02v)
#endif
    using FF = LineFFT<NH, -1, false, false, 0, 0, double2, FSX_F8192_LPF != 0>;
    using FI = LineFFT<NH, +1, false, false, 0, 0, double2, FSX_F8192_LPF != 0>;
    extern __shared__ __align__(128) double2 tile[];  // [NH] tile + [NH / 2] exchange-1 landing
    double2* recv = tile + NH;
    // bar: TMA load; bx1 / bx2: the peer's exchange-1 / exchange-2 stores
    // landed here; bok: the peer's tile is free for exchange 2
    __shared__ __align__(8) unsigned long long bar, bx1, bx2, bok;
    __shared__ double2 acoef[kMaxGroups];
    __shared__ double2 tapterm[kMaxFusedTaps];
    const int th = threadIdx.x;
    const unsigned h = cluster_rank(), peer = h ^ 1u;
    const i64 c = blockIdx.x >> 1;
    i64 kx, ky;
    fused_col_freqs(sym, c, kx, ky);
    if (sym.rank == 3 && c - (c / sym.P) * sym.P > sym.M) return;  // pitch padding of a 3D plane (both CTAs)
    if (th == 0) {
        mbar_init(&bar, 1);
        mbar_init(&bx1, 1);
        mbar_init(&bx2, 1);
        mbar_init(&bok, 1);
        mbar_init_fence();
        mbar_expect_tx(&bx1, (unsigned)(NH / 2 * sizeof(double2)));  // (its own arrival; the peer's bytes complete it)
        mbar_expect_tx(&bx2, (unsigned)(NH / 2 * sizeof(double2)));
        pdl_wait();
        mbar_expect_tx(&bar, (unsigned)(NH * sizeof(double2)));
#pragma unroll 1
        for (int b = 0; b < NH / 256; ++b) tma_load_4d(tile + b * 256, &map2, (int)(2 * c), (int)h, b * 256, 0, &bar);
    }
    cluster_arrive_relaxed();  // publishes the barrier initialisation (fence above) to the peer
    // L2 prefetch in full 128-byte lines: every eighth pair pulls the strip of
    // eight columns pf_dist ahead (the rows of its parity) into L2, so the
    // 16-byte-row TMA loads of the pairs that follow are L2 hits and DRAM sees
    // whole lines instead of one 32-byte sector per row and column pair.
    if (pf_base != nullptr && (c & 7) == 0 && c + pf_dist < g.ncols) {
        const double2* a = pf_base + (i64)(2 * th + (int)h) * g.inner + (c + pf_dist);
#pragma unroll
        for (int q = 0; q < 16; ++q) l2_prefetch_bulk(a + (i64)(512 * q) * g.inner, 128u);
    }
    for (int j = th; j < sym.ntaps; j += TH) tapterm[j] = tap_term(sym, tw_all, j, kx, ky);
    __syncthreads();
    for (int gi = th; gi < sym.ngroups; gi += TH) {
        double2 a = make_double2(0.0, 0.0);
        for (int j = 0; j < sym.ntaps; ++j)
            if (sym.tap_group[j] == gi) a = cadd(a, tapterm[j]);
        acoef[gi] = a;
    }
    cluster_wait();  // the peer's barriers exist (and, CTA-wide, acoef is written)
    mbar_wait(&bar, 0);
    pdl_trigger();
    double2 v[16];
#pragma unroll
    for (int q = 0; q < 16; ++q) v[q] = tile[th + 256 * q];
    FF::run(v, th, tile, tw_all + NH);
    const double2 wt = __ldg(tw_all + N + th);  // W_8192^th; W_8192^(th + 256 q) = wt W_32^q
    // exchange 1: the half of the k range the peer keeps, into its recv -- O goes out raw and
    // each CTA forms W^k O for the k it joins (the same products CTA 1 alone used to form for
    // all 16 values before sending: the pair's critical path loses 64 FP64 instructions)
    {
        const unsigned dst = peer_smem(recv + th, peer), pbar = peer_smem(&bx1, peer);
#pragma unroll
        for (int b = 0; b < 8; ++b) st_async_peer(dst + 256u * 16u * b, h == 0 ? v[8 + b] : v[b], pbar);
    }
    __syncthreads();  // every thread is past the forward FFT's tile reads
    if (th == 0) mbar_arrive_peer(peer_smem(&bok, peer));  // the peer may write into this tile
    mbar_wait(&bx1, 0);
    double2 u[16];
    static_for<0, 8>([&](auto B) {
        constexpr int b = decltype(B)::value;
        const double2 r = recv[th + 256 * b];
        const double2 e = h == 0 ? v[b] : r;
        const double2 oraw = h == 0 ? r : v[8 + b];
        const double2 o = h == 0 ? cmul(oraw, cmul_const<b, 32, -1>(wt)) : cmul(oraw, cmul_const<b + 8, 32, -1>(wt));
        u[b] = cadd(e, o);
        u[b + 8] = csub(e, o);
    });
    if (kx > sym.kzero) {
        // a column of host-proved zero multipliers (FusedSymbol::kzero): the products with lam = 0,
        // i.e. zeros whose signs are those the multiplications would give (zero_products)
#pragma unroll
        for (int j = 0; j < 16; ++j) u[j] = zero_products(u[j], sym.real != 0);
    } else {
        spectral_pair8192(u, th, (int)h, sym, tw_all, acoef);
    }
    // inverse split for the own k = th + 256 b + 2048 h: CTA 0 keeps e and sends o, CTA 1 the reverse
    double2 keep[8], send[8];
    static_for<0, 8>([&](auto B) {
        constexpr int b = decltype(B)::value;
        const double2 e = cadd(u[b], u[b + 8]);
        const double2 d = csub(u[b], u[b + 8]);
        const double2 o = h == 0 ? cmulc(d, cmul_const<b, 32, -1>(wt)) : cmulc(d, cmul_const<b + 8, 32, -1>(wt));
        keep[b] = h == 0 ? e : o;
        send[b] = h == 0 ? o : e;
    });
    // exchange 2 into the peer's tile, once the peer's forward FFT is done with it
    mbar_wait_cluster(&bok, 0);
    {
        const unsigned dst = peer_smem(tile + th, peer), pbar = peer_smem(&bx2, peer);
#pragma unroll
        for (int b = 0; b < 8; ++b) st_async_peer(dst + 256u * 16u * b, send[b], pbar);
    }
    mbar_wait(&bx2, 0);  // the peer's half of this CTA's inverse input landed
#pragma unroll
    for (int b = 0; b < 8; ++b) {
        const double2 r = tile[th + 256 * b];
        v[b] = h == 0 ? keep[b] : r;
        v[8 + b] = h == 0 ? r : keep[b];
    }
    FI::run(v, th, tile, tw_all + NH);
    __syncthreads();  // the last exchange reads are done before the tile is overwritten
#pragma unroll
    for (int q = 0; q < 16; ++q) tile[th + 256 * q] = v[q];
    fence_proxy_async();
    __syncthreads();
    if (th == 0) {
#pragma unroll 1
        for (int b = 0; b < NH / 256; ++b) tma_store_4d(&map2, tile + b * 256, (int)(2 * c), (int)h, b * 256, 0);
        bulk_commit();
        bulk_wait_read0();
    }
}

// ------------------------------------------------------------------ persistent CTA pairs, TMEM-prefetched columns
// k_fused8192c loads its column half when the CTA starts and stores it when
// it ends, so each CTA's TMA load and store latency is exposed to the SM
// except for what the one other resident CTA happens to overlap (ncu: ~20 %
// of the stall samples wait for the tile).  Shared memory has no room for a
// second 64 KB tile per CTA, but tensor memory (256 KB per SM, unused by an
// FFT) does: here each CTA pair is persistent over columns c, c + G, ... and
// while it transforms column c its thread 0 streams the next column's half
// through a 12 KB shared-memory stage into TMEM (TMA box loads -> mbarrier ->
// tcgen05.cp 128x128b -> tcgen05.commit), a chunk per checkpoint between the
// compute phases.  The next iteration starts with one tcgen05.ld.32x32b.x64
// per thread (its 16 values: lane = thread mod 128, 64 contiguous columns).
// The per-column symbol tap terms are computed one column ahead (double
// buffered), and the TMA store of the result drains while the next column's
// data comes out of TMEM.  Arithmetic, exchanges and results are those of
// k_fused8192c (bitwise).
__device__ __forceinline__ unsigned long long tmem_cp_desc(const void* smem) {
    // no-swizzle K-major matrix of 128 rows x 16 B: 8-row core matrices 128 B apart
    const unsigned a = smem_u32(smem);
    return (unsigned long long)((a >> 4) & 0x3FFF) | (1ull << 16) | ((unsigned long long)(128 >> 4) << 32) | (1ull << 46);
}
__device__ __forceinline__ void tmem_cp_128x128b(unsigned taddr, const void* smem) {
    asm volatile("tcgen05.cp.cta_group::1.128x128b [%0], %1;\n" ::"r"(taddr), "l"(tmem_cp_desc(smem)) : "memory");
}
__device__ __forceinline__ void tmem_commit(unsigned long long* bar) {
    asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];\n" ::"r"(smem_u32(bar))
                 : "memory");
}
__device__ __forceinline__ void tc_fence_before() { asm volatile("tcgen05.fence::before_thread_sync;\n" ::: "memory"); }
__device__ __forceinline__ void tc_fence_after() { asm volatile("tcgen05.fence::after_thread_sync;\n" ::: "memory"); }
// 16 complex values (64 x 32-bit TMEM columns) of this thread's lane
__device__ __forceinline__ void tmem_ld16(unsigned taddr, double2 (&v)[16]) {
    unsigned r[64];
    asm volatile(
        "tcgen05.ld.sync.aligned.32x32b.x64.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,%16,%17,%18,%19,"
        "%20,%21,%22,%23,%24,%25,%26,%27,%28,%29,%30,%31,%32,%33,%34,%35,%36,%37,%38,%39,%40,%41,%42,%43,%44,%45,%46,"
        "%47,%48,%49,%50,%51,%52,%53,%54,%55,%56,%57,%58,%59,%60,%61,%62,%63}, [%64];\n"
        : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]), "=r"(r[7]), "=r"(r[8]),
          "=r"(r[9]), "=r"(r[10]), "=r"(r[11]), "=r"(r[12]), "=r"(r[13]), "=r"(r[14]), "=r"(r[15]), "=r"(r[16]),
          "=r"(r[17]), "=r"(r[18]), "=r"(r[19]), "=r"(r[20]), "=r"(r[21]), "=r"(r[22]), "=r"(r[23]), "=r"(r[24]),
          "=r"(r[25]), "=r"(r[26]), "=r"(r[27]), "=r"(r[28]), "=r"(r[29]), "=r"(r[30]), "=r"(r[31]), "=r"(r[32]),
          "=r"(r[33]), "=r"(r[34]), "=r"(r[35]), "=r"(r[36]), "=r"(r[37]), "=r"(r[38]), "=r"(r[39]), "=r"(r[40]),
          "=r"(r[41]), "=r"(r[42]), "=r"(r[43]), "=r"(r[44]), "=r"(r[45]), "=r"(r[46]), "=r"(r[47]), "=r"(r[48]),
          "=r"(r[49]), "=r"(r[50]), "=r"(r[51]), "=r"(r[52]), "=r"(r[53]), "=r"(r[54]), "=r"(r[55]), "=r"(r[56]),
          "=r"(r[57]), "=r"(r[58]), "=r"(r[59]), "=r"(r[60]), "=r"(r[61]), "=r"(r[62]), "=r"(r[63])
        : "r"(taddr));
    asm volatile("tcgen05.wait::ld.sync.aligned;\n" ::: "memory");
#pragma unroll
    for (int q = 0; q < 16; ++q) {
        v[q].x = __hiloint2double((int)r[4 * q + 1], (int)r[4 * q]);
        v[q].y = __hiloint2double((int)r[4 * q + 3], (int)r[4 * q + 2]);
    }
}

// Thread 0's column-half prefetch: chunks of PF_BOX TMA boxes (256 rows of
// 16 B) land in the stage, then tcgen05.cp moves each 128-element block b
// (half-column elements 128 b .. 128 b + 127) to lanes 0..127, columns
// 64 (b % 2) + 4 (b / 2): thread th then finds elements th + 256 q at lane
// th % 128, columns 64 (th / 128) + 4 q.
__device__ __forceinline__ bool mbar_test(unsigned long long* bar, unsigned parity) {
    unsigned ok;
    asm volatile(
        "{\n.reg .pred P1;\nmbarrier.test_wait.parity.shared::cta.b64 P1, [%1], %2;\nselp.u32 %0, 1, 0, P1;\n}\n"
        : "=r"(ok)
        : "r"(smem_u32(bar)), "r"(parity)
        : "memory");
    return ok != 0;
}

struct PrefetchPipe {
    static constexpr int PF_BOX = 3;                              // boxes per chunk (12 KB stage)
    static constexpr int NCH = (16 + PF_BOX - 1) / PF_BOX;        // chunks per 4096-element half
    int pend = NCH;      // chunk in flight (NCH: nothing pending)
    int state = 0;       // 0 idle, 1 TMA landing in the stage, 2 tcgen05.cp reading the stage
    i64 col = 0;         // column being prefetched
    unsigned lpar = 0, cpar = 0;
    __device__ __forceinline__ void issue(const CUtensorMap* map, double2* stage, unsigned long long* lbar, unsigned h,
                                          int k) {
        const int b0 = k * PF_BOX, b1 = b0 + PF_BOX < 16 ? b0 + PF_BOX : 16;
        mbar_expect_tx(lbar, (unsigned)((b1 - b0) * 256 * sizeof(double2)));
        for (int b = b0; b < b1; ++b) tma_load_4d(stage + (b - b0) * 256, map, (int)(2 * col), (int)h, b * 256, 0, lbar);
        state = 1;
    }
    __device__ __forceinline__ void start(const CUtensorMap* map, double2* stage, unsigned long long* lbar, unsigned h,
                                          i64 c) {
        col = c;
        pend = 0;
        issue(map, stage, lbar, h, 0);
    }
    // Advance as far as possible without waiting (block = true: to the end):
    // a landed chunk is copied into TMEM, a finished copy frees the stage for
    // the next chunk's TMA loads.
    __device__ __forceinline__ void poll(const CUtensorMap* map, double2* stage, unsigned long long* lbar,
                                         unsigned long long* cbar, unsigned h, unsigned tbase, bool block = false) {
        while (state != 0) {
            if (state == 1) {
                if (!block && !mbar_test(lbar, lpar)) return;
                mbar_wait(lbar, lpar);
                lpar ^= 1u;
                tc_fence_after();
                const int b0 = pend * PF_BOX, b1 = b0 + PF_BOX < 16 ? b0 + PF_BOX : 16;
                for (int blk = 2 * b0; blk < 2 * b1; ++blk)
                    tmem_cp_128x128b(tbase + 64u * (unsigned)(blk & 1) + 4u * (unsigned)(blk >> 1),
                                     stage + (blk - 2 * b0) * 128);
                tmem_commit(cbar);
                state = 2;
            } else {
                if (!block && !mbar_test(cbar, cpar)) return;
                mbar_wait(cbar, cpar);
                cpar ^= 1u;
                if (++pend < NCH) issue(map, stage, lbar, h, pend);
                else state = 0;
            }
        }
    }
};

// Symbol group coefficients of one column: tap terms (threads j < ntaps),
// then their per-group sums (threads gi < ngroups) after a barrier.
__device__ __forceinline__ i64 next_fused_col(const FusedSymbol& sym, i64 c, i64 step, i64 ncols) {
    for (c += step; c < ncols; c += step)
        if (sym.rank != 3 || c - (c / sym.P) * sym.P <= sym.M) return c;
    return -1;
}

__global__ void __cluster_dims__(2, 1, 1) __launch_bounds__(256, 2)
k_fused8192p(const __grid_constant__ CUtensorMap map2, AxisGeom g, FusedSymbol sym, const double2* __restrict__ tw_all) {
    constexpr int N = 8192, NH = 4096, TH = 256;
    using FF = LineFFT<NH, -1>;
    using FI = LineFFT<NH, +1>;
    extern __shared__ __align__(1024) double2 tile[];  // [NH] tile, [NH / 2] exchange-1 landing, prefetch stage
    double2* recv = tile + NH;
    double2* stage = recv + NH / 2;
    __shared__ __align__(8) unsigned long long lbar, cbar, bx1, bx2, bok;
    __shared__ double2 acoef[2][kMaxGroups];
    __shared__ double2 tapterm[2][kMaxFusedTaps];
    __shared__ unsigned tmem_base;
    const int th = threadIdx.x;
    const unsigned h = cluster_rank(), peer = h ^ 1u;
    const i64 ncl = (i64)gridDim.x >> 1;
    i64 c = next_fused_col(sym, (i64)(blockIdx.x >> 1) - ncl, ncl, g.ncols);
    if (c < 0) return;  // (both CTAs of the pair)
    PrefetchPipe pf;
    if (th < 32) {  // 128 TMEM columns: one 4096-element half (lanes x 64 B)
        asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 128;\n" ::"r"(smem_u32(&tmem_base)));
        asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;\n");
    }
    if (th == 0) {
        mbar_init(&lbar, 1);
        mbar_init(&cbar, 1);
        mbar_init(&bx1, 1);
        mbar_init(&bx2, 1);
        mbar_init(&bok, 1);
        mbar_init_fence();
        mbar_expect_tx(&bx1, (unsigned)(NH / 2 * sizeof(double2)));
        mbar_expect_tx(&bx2, (unsigned)(NH / 2 * sizeof(double2)));
    }
    tc_fence_before();
    cluster_arrive_relaxed();  // publishes the barrier initialisation to the peer
    // the first column's tap terms and group sums
    {
        i64 kx, ky;
        fused_col_freqs(sym, c, kx, ky);
        for (int j = th; j < sym.ntaps; j += TH) tapterm[0][j] = tap_term(sym, tw_all, j, kx, ky);
    }
    __syncthreads();
    tc_fence_after();
    const unsigned tbase = tmem_base;
    for (int gi = th; gi < sym.ngroups; gi += TH) {
        double2 a = make_double2(0.0, 0.0);
        for (int j = 0; j < sym.ntaps; ++j)
            if (sym.tap_group[j] == gi) a = cadd(a, tapterm[0][j]);
        acoef[0][gi] = a;
    }
    if (th == 0) {
        pdl_wait();  // H is the predecessor's output
        pf.start(&map2, stage, &lbar, h, c);
        pf.poll(&map2, stage, &lbar, &cbar, h, tbase, true);
    }
    tc_fence_before();
    cluster_wait();  // the peer's barriers exist
    __syncthreads();  // the first column is in TMEM; acoef[0] written
    tc_fence_after();
    const unsigned my_taddr = tbase + ((unsigned)(32 * ((th >> 5) & 3)) << 16) + 64u * (unsigned)(th >> 7);
    const double2 wt = __ldg(tw_all + N + th);  // W_8192^th; W_8192^(th + 256 q) = wt W_32^q
    for (unsigned it = 0; c >= 0; ++it) {
        const unsigned s = it & 1u, par = it & 1u;
        const i64 cn = next_fused_col(sym, c, ncl, g.ncols);
        double2 v[16];
        tmem_ld16(my_taddr, v);
        tc_fence_before();
        if (th == 0) bulk_wait_read0();  // the previous column's store has read the tile
        if (cn < 0) pdl_trigger();
        __syncthreads();  // TMEM read by every thread; tile free
        if (th == 0 && cn >= 0) {
            tc_fence_after();
            pf.start(&map2, stage, &lbar, h, cn);
        }
        FF::run(v, th, tile, tw_all + NH);
        if (th == 0) pf.poll(&map2, stage, &lbar, &cbar, h, tbase);
        if (h == 1) {
            static_for<0, 16>([&](auto Q) {
                constexpr int q = decltype(Q)::value;
                v[q] = cmul(v[q], cmul_const<q, 32, -1>(wt));
            });
        }
        // exchange 1: the half of the k range the peer keeps, into its recv
        {
            const unsigned dst = peer_smem(recv + th, peer), pbar = peer_smem(&bx1, peer);
#pragma unroll
            for (int b = 0; b < 8; ++b) st_async_peer(dst + 256u * 16u * b, h == 0 ? v[8 + b] : v[b], pbar);
        }
        if (th == 0) pf.poll(&map2, stage, &lbar, &cbar, h, tbase);
        // the next column's tap terms (their table reads overlap the wait below)
        if (cn >= 0) {
            i64 kx, ky;
            fused_col_freqs(sym, cn, kx, ky);
            for (int j = th; j < sym.ntaps; j += TH) tapterm[s ^ 1u][j] = tap_term(sym, tw_all, j, kx, ky);
        }
        __syncthreads();  // every thread is past the forward FFT's tile reads
        if (th == 0) mbar_arrive_peer(peer_smem(&bok, peer));  // the peer may write into this tile
        mbar_wait(&bx1, par);
        double2 u[16];
#pragma unroll
        for (int b = 0; b < 8; ++b) {
            const double2 r = recv[th + 256 * b];
            const double2 e = h == 0 ? v[b] : r;
            const double2 o = h == 0 ? r : v[8 + b];
            u[b] = cadd(e, o);
            u[b + 8] = csub(e, o);
        }
        if (th == 0) {
            mbar_expect_tx(&bx1, (unsigned)(NH / 2 * sizeof(double2)));  // next column's exchange 1
            pf.poll(&map2, stage, &lbar, &cbar, h, tbase);
        }
        spectral_pair8192(u, th, (int)h, sym, tw_all, acoef[s]);
        double2 keep[8], send[8];
        static_for<0, 8>([&](auto B) {
            constexpr int b = decltype(B)::value;
            const double2 e = cadd(u[b], u[b + 8]);
            const double2 d = csub(u[b], u[b + 8]);
            const double2 o = h == 0 ? cmulc(d, cmul_const<b, 32, -1>(wt)) : cmulc(d, cmul_const<b + 8, 32, -1>(wt));
            keep[b] = h == 0 ? e : o;
            send[b] = h == 0 ? o : e;
        });
        if (th == 0) pf.poll(&map2, stage, &lbar, &cbar, h, tbase);
        // exchange 2 into the peer's tile, once the peer's forward FFT is done with it
        mbar_wait_cluster(&bok, par);
        {
            const unsigned dst = peer_smem(tile + th, peer), pbar = peer_smem(&bx2, peer);
#pragma unroll
            for (int b = 0; b < 8; ++b) st_async_peer(dst + 256u * 16u * b, send[b], pbar);
        }
        if (th == 0) pf.poll(&map2, stage, &lbar, &cbar, h, tbase);
        mbar_wait(&bx2, par);
#pragma unroll
        for (int b = 0; b < 8; ++b) {
            const double2 r = tile[th + 256 * b];
            v[b] = h == 0 ? keep[b] : r;
            v[8 + b] = h == 0 ? r : keep[b];
        }
        if (th == 0) mbar_expect_tx(&bx2, (unsigned)(NH / 2 * sizeof(double2)));
        FI::run(v, th, tile, tw_all + NH);
        if (th == 0) pf.poll(&map2, stage, &lbar, &cbar, h, tbase);
        __syncthreads();  // the last exchange reads are done before the tile is overwritten
#pragma unroll
        for (int q = 0; q < 16; ++q) tile[th + 256 * q] = v[q];
        fence_proxy_async();
        // the next column's group sums (its tap terms were written before two barriers)
        if (cn >= 0)
            for (int gi = th; gi < sym.ngroups; gi += TH) {
                double2 a = make_double2(0.0, 0.0);
                for (int j = 0; j < sym.ntaps; ++j)
                    if (sym.tap_group[j] == gi) a = cadd(a, tapterm[s ^ 1u][j]);
                acoef[s ^ 1u][gi] = a;
            }
        __syncthreads();
        if (th == 0) {
#pragma unroll 1
            for (int b = 0; b < NH / 256; ++b) tma_store_4d(&map2, tile + b * 256, (int)(2 * c), (int)h, b * 256, 0);
            bulk_commit();
            pf.poll(&map2, stage, &lbar, &cbar, h, tbase, true);
        }
        tc_fence_before();
        __syncthreads();  // the next column is in TMEM
        tc_fence_after();
        c = cn;
    }
    if (th == 0) bulk_wait_read0();
    tc_fence_before();
    __syncthreads();
    if (th < 32) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 128;\n" ::"r"(tbase));
}

// FSX_F8192: "c" (default) the one-column-per-pair kernel, "p" the persistent
// TMEM-prefetched pairs (measured slower on cfg3: 0.672 ms with blocking
// chunk steps, 0.811 ms polled, against 0.584 -- a 12 KB stage keeps too few
// bytes in flight to hide the 16-byte-row TMA latency), "h" the one-CTA
// parity-halves kernel
static int f8192_kind() {
    static int v = -1;
    if (v < 0) {
        const char* e = getenv("FSX_F8192");
        v = (e && e[0] == 'h') ? 0 : (e && e[0] == 'p') ? 2 : 1;
    }
    return v;
}
static bool f8192_pair() { return f8192_kind() != 0; }

static int fused_halves() {
    static int v = -1;
    if (v < 0) {
        const char* e = getenv("FSX_HALVES");
        v = e ? atoi(e) : 1;
    }
    return v;
}

bool halves_ok(const AxisGeom& g) { return g.n == 8192 && g.outer == 1 && fused_halves(); }

// FSX_F8192_PFD: L2 prefetch distance of k_fused8192c in columns (a multiple of 8; 0: off)
static int f8192_pfd() {
    static int v = -1;
    if (v < 0) {
        const char* e = getenv("FSX_F8192_PFD");
        v = e ? atoi(e) & ~7 : 0;
    }
    return v;
}

cudaError_t launch_fused_halves(const void* tensor_map2, const AxisGeom& g, const FusedSymbol& sym,
                                const double2* tw, cudaStream_t s, const double2* base) {
    const CUtensorMap& map = *reinterpret_cast<const CUtensorMap*>(tensor_map2);
    if (f8192_kind() == 2) {
        // one persistent pair per SM (two CTAs of 256 threads per SM)
        const size_t smem = (4096 + 2048 + 256 * PrefetchPipe::PF_BOX) * sizeof(double2);
        kernel_prepare((const void*)k_fused8192p, smem);
        static int nsm = 0;
        if (!nsm) {
            int dev = 0;
            cudaGetDevice(&dev);
            cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, dev);
        }
        const i64 pairs = std::min<i64>(nsm, g.ncols);
        return launch_pdl(k_fused8192p, dim3((unsigned)(2 * pairs)), dim3(256), smem, s, map, g, sym, tw);
    }
    if (f8192_pair()) {
        const size_t smem2 = (4096 + 2048) * sizeof(double2);
        kernel_prepare((const void*)k_fused8192c, smem2);
        const int pfd = base != nullptr && g.inner % 8 == 0 ? f8192_pfd() : 0;
        return launch_pdl_cluster(k_fused8192c, dim3((unsigned)(2 * g.ncols)), dim3(256), smem2, s, map, g, sym, tw,
                          pfd > 0 ? base : (const double2*)nullptr, pfd);
    }
    const size_t smem = 8192 * sizeof(double2);
    kernel_prepare((const void*)k_fused8192h, smem);
    return launch_pdl(k_fused8192h, dim3((unsigned)g.ncols), dim3(512), smem, s, map, g, sym, tw);
}

template <int N, int MODE>
static cudaError_t cols_tma_n(const CUtensorMap& map, const AxisGeom& g, const FusedSymbol& sym, const double2* tw,
                              cudaStream_t s) {
    using C = TCfg<N>;
    // tile + (fused mode) the per-frequency real multipliers
    const size_t smem = C::smem(MODE);
    const i64 tiles = (g.ncols + C::W - 1) / C::W;
    kernel_prepare((const void*)k_cols_tma<N, MODE>, smem);
    return launch_pdl(k_cols_tma<N, MODE>, dim3((unsigned)(g.outer * tiles)), dim3(C::NT), smem, s, map, g, sym, tw);
}

// columns per TMA tile for a line length (the host builds the box to match)
int tma_cols_width(i64 N) { return N >= 4096 ? 1 : (int)(4096 / N); }

bool tma_cols_ok(i64 N) { return N >= 512 && N <= 8192; }

cudaError_t launch_cols_tma(const void* tensor_map, const AxisGeom& g, int mode, const FusedSymbol& sym,
                            const double2* tw, cudaStream_t s) {
    const CUtensorMap& map = *reinterpret_cast<const CUtensorMap*>(tensor_map);
    if (getenv("FSX_TMA_COPYONLY") && g.n == 4096) return cols_tma_n<4096, 3>(map, g, sym, tw, s);  // measurement
#define FSX_TMA(N)                                                    \
    case N:                                                            \
        return mode == 0 ? cols_tma_n<N, 0>(map, g, sym, tw, s)        \
             : mode == 1 ? cols_tma_n<N, 1>(map, g, sym, tw, s)        \
             : sym.implicit ? cols_tma_n<N, 4>(map, g, sym, tw, s)     \
                            : cols_tma_n<N, 2>(map, g, sym, tw, s);
    switch (g.n) {
        FSX_TMA(512)
        FSX_TMA(1024)
        FSX_TMA(2048)
        FSX_TMA(4096)
        FSX_TMA(8192)
        default: return cudaErrorInvalidValue;
    }
#undef FSX_TMA
}

// Host: tensor map over a complex array viewed as fp64 [outer][n][2*inner].
typedef CUresult (*EncodeTiledFn)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*, const cuuint64_t*,
                                  const cuuint64_t*, const cuuint32_t*, const cuuint32_t*, CUtensorMapInterleave,
                                  CUtensorMapSwizzle, CUtensorMapL2promotion, CUtensorMapFloatOOBfill);

// Parity-split view for k_fused8192h: dims {2 inner, 2 (row parity), n/2, outer},
// box {2, 1, 256, 1}: one box = 256 rows of one parity of one column.
int make_cols_tensor_map_par(void* out_map, void* base, const AxisGeom& g) {
    static EncodeTiledFn encode = nullptr;
    if (!encode) {
        cudaDriverEntryPointQueryResult q;
        void* fn = nullptr;
        if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &fn, cudaEnableDefault, &q) != cudaSuccess ||
            q != cudaDriverEntryPointSuccess || !fn)
            return -1;
        encode = reinterpret_cast<EncodeTiledFn>(fn);
    }
    if (g.n % 2 || g.n / 2 < 256) return -2;
    const cuuint64_t dims[4] = {(cuuint64_t)(2 * g.inner), 2, (cuuint64_t)(g.n / 2), (cuuint64_t)g.outer};
    const cuuint64_t strides[3] = {(cuuint64_t)(g.inner * 16), (cuuint64_t)(2 * g.inner * 16), (cuuint64_t)(g.block * 16)};
    const cuuint32_t box[4] = {2, 1, 256, 1};
    const cuuint32_t estr[4] = {1, 1, 1, 1};
    CUresult r = encode(reinterpret_cast<CUtensorMap*>(out_map), CU_TENSOR_MAP_DATA_TYPE_FLOAT64, 4, base, dims, strides,
                        box, estr, CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE,
                        CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    return r == CUDA_SUCCESS ? 0 : (int)r;
}

int make_cols_tensor_map(void* out_map, void* base, const AxisGeom& g) {
    return make_cols_tensor_map_w(out_map, base, g, tma_cols_width(g.n));
}

int make_cols_tensor_map_w(void* out_map, void* base, const AxisGeom& g, int W) {
    static EncodeTiledFn encode = nullptr;
    if (!encode) {
        cudaDriverEntryPointQueryResult q;
        void* fn = nullptr;
        if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &fn, cudaEnableDefault, &q) != cudaSuccess ||
            q != cudaDriverEntryPointSuccess || !fn)
            return -1;
        encode = reinterpret_cast<EncodeTiledFn>(fn);
    }
    if (g.outer > 1 && g.block != g.n * g.inner) return -2;  // contiguous outer blocks only
    const cuuint64_t dims[3] = {(cuuint64_t)(2 * g.inner), (cuuint64_t)g.n, (cuuint64_t)g.outer};
    const cuuint64_t strides[2] = {(cuuint64_t)(g.inner * 16), (cuuint64_t)(g.block * 16)};
    const cuuint32_t box[3] = {(cuuint32_t)(2 * W), (cuuint32_t)(g.n < 256 ? g.n : 256), 1};
    const cuuint32_t estr[3] = {1, 1, 1};
    CUresult r = encode(reinterpret_cast<CUtensorMap*>(out_map), CU_TENSOR_MAP_DATA_TYPE_FLOAT64, 3, base, dims, strides,
                        box, estr, CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE,
                        CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    return r == CUDA_SUCCESS ? 0 : (int)r;
}

}  // namespace fsx
