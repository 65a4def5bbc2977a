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

#include <cstdlib>

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
    // ... or in tensor memory (16 warps x 32 columns): correct (tests cover it) but
    // measured neutral on cfg3 (0.834 vs 0.824 ms), so off; FSX_TMEM_MULT=1 at build
#ifdef FSX_TMEM_MULT
    static constexpr bool TMEM = N == 8192;
#else
    static constexpr bool TMEM = false;
#endif
    static constexpr size_t smem(int mode) {
        return (size_t)W * LSW * 16 + (mode == 2 && PRE ? (size_t)NT * R * 8 : 0);
    }
};

static int tma_w2();

// MODE 0: forward C2C, 1: inverse C2C, 2: fused R2C spectral pass.
// The TMA tile is [N rows][W columns] (row-major, as the boxes land); the
// FFT exchanges reuse the same buffer as W line-major rows of LSW.
template <int N, int MODE, int WW = 0>
__global__ void __launch_bounds__(TCfg<N, WW>::NT, TCfg<N, WW>::MINB)
k_cols_tma(const __grid_constant__ CUtensorMap map, AxisGeom g, FusedSymbol sym, const double2* __restrict__ tw_all) {
    using C = TCfg<N, WW>;
    constexpr int W = C::W;
    // full twiddle tables for the multi-column tiles (N < 4096); the one-column
    // 4096 tiles measured faster with derived twiddles (cfg2 158 vs 165 us)
    constexpr bool FT = N < 4096;
    using FF = LineFFT<N, -1, false, false, FT>;
    using FI = LineFFT<N, +1, false, false, FT>;
    extern __shared__ __align__(128) double2 tile[];
    __shared__ __align__(8) unsigned long long bar;
    __shared__ double2 acoef[kMaxGroups][W];
    __shared__ double2 tapterm[MODE == 2 ? kMaxFusedTaps : 1][W];
    const int w = threadIdx.x % W, t = threadIdx.x / W;
    const i64 tiles = (g.ncols + W - 1) / W;
    const i64 o = (i64)blockIdx.x / tiles;
    const i64 c0 = ((i64)blockIdx.x - o * tiles) * W;
    const i64 c = c0 + w;
    i64 kx = c, ky = 0;
    if constexpr (MODE == 2) {
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
    // L1 that serves the table reads (cfg3 measured 0.87 -> 1.04 ms).
    // The 128 KB tiles (N = 8192, 16 warps, one CTA per SM) park the
    // multipliers in tensor memory instead (128 columns; see fsx_async.cuh).
    constexpr bool PRE = MODE == 2 && C::PRE;
    constexpr bool TM = MODE == 2 && C::TMEM;
    double* mult = reinterpret_cast<double*>(tile + W * C::LSW);
    __shared__ unsigned tmem_base;
    const int warp = threadIdx.x >> 5;
    if constexpr (TM) {
        if (warp == 0) tmem_alloc<128>(&tmem_base);
        tmem_fence_before();
    }
    if constexpr (MODE == 2) {
        for (int j = t; j < sym.ntaps; j += C::TPL) tapterm[j][w] = tap_term(sym, tw_all, j, kx, ky);
    }
    __syncthreads();  // barrier initialised before anyone waits on it; tap terms visible
    if constexpr (TM) tmem_fence_after();
    if constexpr (MODE == 2) {
        for (int gi = t; gi < sym.ngroups; gi += C::TPL) {
            double2 a = make_double2(0.0, 0.0);
            for (int j = 0; j < sym.ntaps; ++j)
                if (sym.tap_group[j] == gi) a = cadd(a, tapterm[j][w]);
            acoef[gi][w] = a;
        }
        __syncthreads();
        if ((PRE || TM) && sym.real) {
            double lam[C::R];
            symbol_real<N, C::R, C::TPL>(lam, t, sym, tw_all, [&](int gi) { return acoef[gi][w]; });
            pow_real_vec_skip<C::R, 4>(lam, sym.T, sym.neg_mag2);
            if constexpr (TM) {
                static_assert(C::R == 16, "TMEM parking holds 16 doubles per thread");
                double h[8];
                const unsigned ta = tmem_warp_addr(tmem_base, warp);
#pragma unroll
                for (int half = 0; half < 2; ++half) {
#pragma unroll
                    for (int i = 0; i < 8; ++i) h[i] = lam[8 * half + i] * sym.scale;
                    tmem_st8(ta + 16 * half, h);
                }
                tmem_wait_st();
            } else {
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
    if constexpr (MODE == 2) {
        if (PRE && sym.real) {
#pragma unroll
            for (int q = 0; q < C::R; ++q) v[q] = cscale(v[q], mult[q * C::NT + threadIdx.x]);
        } else if (TM && sym.real) {
            const unsigned ta = tmem_warp_addr(tmem_base, warp);
#pragma unroll
            for (int half = 0; half < 2; ++half) {
                double h[8];
                tmem_ld8(ta + 16 * half, h);
#pragma unroll
                for (int i = 0; i < 8; ++i) v[8 * half + i] = cscale(v[8 * half + i], h[i]);
            }
        } else {
            spectral_regs<N, C::R, C::TPL>(v, t, sym, tw_all, [&](int gi) { return acoef[gi][w]; });
        }
        FI::run(v, t, line, tw_all + N);
    }
    if constexpr (TM) tmem_fence_before();
    __syncthreads();  // last exchange reads done before the tile is overwritten
#pragma unroll
    for (int q = 0; q < C::R; ++q) tile[(t + q * C::TPL) * W + w] = v[q];
    fence_proxy_async();
    __syncthreads();
    if constexpr (TM) {
        if (warp == 0) {
            tmem_fence_after();
            tmem_dealloc<128>(tmem_base);
        }
    }
    if (threadIdx.x == 0) {
#pragma unroll 1
        for (int b = 0; b < C::NBOX; ++b) tma_store_3d(&map, tile + b * C::BOX * W, (int)(2 * c0), b * C::BOX, (int)o);
        bulk_commit();
        bulk_wait_read0();
    }
}

// Fused spectral pass for 4096-point columns on the transposed four-step FFT
// (Fft4096T): forward leaves the column in digit-transposed frequency order,
// the symbol is evaluated in that order, and the inverse returns to natural
// order -- one CTA-wide exchange per direction instead of two.
__global__ void __launch_bounds__(256, 2)
k_fused_tma4(const __grid_constant__ CUtensorMap map, AxisGeom g, FusedSymbol sym, const double2* __restrict__ tw_all) {
    constexpr int N = 4096;
    extern __shared__ __align__(128) double2 tile[];
    __shared__ __align__(8) unsigned long long bar;
    __shared__ double2 acoef[kMaxGroups];
    __shared__ double2 tapterm[kMaxFusedTaps];
    const int t = threadIdx.x;
    const i64 c = blockIdx.x;
    i64 kx, ky;
    fused_col_freqs(sym, c, kx, ky);
    if (sym.rank == 3 && c - (c / sym.P) * sym.P > sym.M) return;
    if (t == 0) {
        mbar_init(&bar, 1);
        asm volatile("fence.mbarrier_init.release.cluster;\n" ::: "memory");
        mbar_expect_tx(&bar, (unsigned)(N * sizeof(double2)));
#pragma unroll 1
        for (int b = 0; b < N / 256; ++b) tma_load_3d(tile + b * 256, &map, (int)(2 * c), b * 256, 0, &bar);
    }
    for (int j = t; j < sym.ntaps; j += 256) tapterm[j] = tap_term(sym, tw_all, j, kx, ky);
    __syncthreads();
    mbar_wait(&bar, 0);
    double2 v[16];
#pragma unroll
    for (int q = 0; q < 16; ++q) v[q] = tile[t + 256 * q];
    __syncthreads();  // tile consumed before the exchange overwrites it
    Fft4096T::forward(v, t, tile, tw_all);
    for (int gi = t; gi < sym.ngroups; gi += 256) {
        double2 a = make_double2(0.0, 0.0);
        for (int j = 0; j < sym.ntaps; ++j)
            if (sym.tap_group[j] == gi) a = cadd(a, tapterm[j]);
        acoef[gi] = a;
    }
    __syncthreads();
    spectral_regs_at<N, 16>(v, (t >> 4) + 16 * (t & 15), 256, sym, tw_all, [&](int gi) { return acoef[gi]; });
    Fft4096T::inverse(v, t, tile, tw_all);
    __syncthreads();
#pragma unroll
    for (int q = 0; q < 16; ++q) tile[t + 256 * q] = v[q];
    fence_proxy_async();
    __syncthreads();
    if (t == 0) {
#pragma unroll 1
        for (int b = 0; b < N / 256; ++b) tma_store_3d(&map, tile + b * 256, (int)(2 * c), b * 256, 0);
        bulk_commit();
        bulk_wait_read0();
    }
}

// FSX_4STEP=1 selects k_fused_tma4 (measured slower on cfg2: 189 vs 165 us;
// the transposed order scatters the symbol-table reads), default off.
static int fused_4step() {
    static int v = -1;
    if (v < 0) {
        const char* e = getenv("FSX_4STEP");
        v = e ? atoi(e) : 0;
    }
    return v;
}

// Persistent variant: one CTA per SM walks the tiles with two shared-memory
// stages; the TMA load of tile i+1 is in flight while tile i is transformed,
// and a stage is refilled only after the bulk store that drained it has
// finished reading shared memory (cp.async.bulk.wait_group.read).
template <int N, int MODE>
__global__ void __launch_bounds__(TCfg<N>::NT, 1)
k_cols_tma_pers(const __grid_constant__ CUtensorMap map, AxisGeom g, FusedSymbol sym,
                const double2* __restrict__ tw_all) {
    using C = TCfg<N>;
    constexpr int W = C::W;
    constexpr int STAGE = W * C::LSW;
    using FF = LineFFT<N, -1, true>;
    using FI = LineFFT<N, +1, true>;
    extern __shared__ __align__(128) double2 tile[];
    constexpr int NST = 3;  // stages: refilled stage's store was issued a full iteration earlier
    __shared__ __align__(8) unsigned long long bar[NST];
    __shared__ double2 acoef[kMaxGroups][W];
    __shared__ double2 tapterm[MODE == 2 ? kMaxFusedTaps : 1][W];
    const int w = threadIdx.x % W, t = threadIdx.x / W;
    const i64 tiles = (g.ncols + W - 1) / W;
    const i64 ntiles = g.outer * tiles;
    auto pos = [&](i64 tl, i64& o, i64& c0) {
        o = tl / tiles;
        c0 = (tl - o * tiles) * W;
    };
    auto live = [&](i64 c0) {
        if constexpr (MODE == 2) {
            if (sym.rank == 3) return c0 - (c0 / sym.P) * sym.P <= sym.M;
        }
        return true;
    };
    auto issue = [&](i64 tl, int s) {  // thread 0 only
        i64 o, c0;
        pos(tl, o, c0);
        if (!live(c0)) {
            asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];\n" ::"r"(smem_u32(&bar[s])) : "memory");
            return;
        }
        mbar_expect_tx(&bar[s], (unsigned)(N * W * sizeof(double2)));
#pragma unroll 1
        for (int b = 0; b < C::NBOX; ++b)
            tma_load_3d(tile + s * STAGE + b * C::BOX * W, &map, (int)(2 * c0), b * C::BOX, (int)o, &bar[s]);
    };
    if (threadIdx.x == 0) {
#pragma unroll
        for (int i = 0; i < NST; ++i) mbar_init(&bar[i], 1);
        asm volatile("fence.mbarrier_init.release.cluster;\n" ::: "memory");
        if ((i64)blockIdx.x < ntiles) issue(blockIdx.x, 0);
    }
    __syncthreads();
    unsigned phase[NST] = {0u, 0u, 0u};
    int s = 0;
    for (i64 tl = blockIdx.x; tl < ntiles; tl += gridDim.x, s = (s + 1) % NST) {
        const i64 nxt = tl + gridDim.x;
        const int ns = (s + 1) % NST;
        if (threadIdx.x == 0 && nxt < ntiles) {
            // stage ns was last drained by the store issued two iterations ago;
            // only the newest store group may still be reading shared memory
            asm volatile("cp.async.bulk.wait_group.read 1;\n" ::: "memory");
            issue(nxt, ns);
        }
        i64 o, c0;
        pos(tl, o, c0);
        const i64 c = c0 + w;
        double2* stg = tile + s * STAGE;
        if (live(c0)) {
            i64 kx = c, ky = 0;
            if constexpr (MODE == 2) {
                fused_col_freqs(sym, c, kx, ky);
                for (int j = t; j < sym.ntaps; j += C::TPL) tapterm[j][w] = tap_term(sym, tw_all, j, kx, ky);
            }
            mbar_wait(&bar[s], phase[s]);
            double2 v[C::R];
#pragma unroll
            for (int q = 0; q < C::R; ++q) v[q] = stg[(t + q * C::TPL) * W + w];
            double2* line = stg + w * C::LSW;
            if constexpr (MODE == 3) {
                // copy-only (measurement of the TMA column I/O alone)
            } else if constexpr (MODE == 1) {
                FI::run(v, t, line, tw_all + N);
            } else {
                FF::run(v, t, line, tw_all + N);
            }
            if constexpr (MODE == 2) {
                __syncthreads();
                for (int gi = t; gi < sym.ngroups; gi += C::TPL) {
                    double2 a = make_double2(0.0, 0.0);
                    for (int j = 0; j < sym.ntaps; ++j)
                        if (sym.tap_group[j] == gi) a = cadd(a, tapterm[j][w]);
                    acoef[gi][w] = a;
                }
                __syncthreads();
                spectral_regs<N, C::R, C::TPL>(v, t, sym, tw_all, [&](int gi) { return acoef[gi][w]; });
                FI::run(v, t, line, tw_all + N);
            }
            __syncthreads();
#pragma unroll
            for (int q = 0; q < C::R; ++q) stg[(t + q * C::TPL) * W + w] = v[q];
            fence_proxy_async();
            __syncthreads();
            if (threadIdx.x == 0) {
#pragma unroll 1
                for (int b = 0; b < C::NBOX; ++b)
                    tma_store_3d(&map, stg + b * C::BOX * W, (int)(2 * c0), b * C::BOX, (int)o);
                bulk_commit();
            }
        } else {
            mbar_wait(&bar[s], phase[s]);
        }
        phase[s] ^= 1u;
        __syncthreads();
    }
    if (threadIdx.x == 0) bulk_wait_read0();
}

static int tma_persistent() {
    static int v = -1;
    if (v < 0) {
        const char* e = getenv("FSX_TMA_PERSIST");
        v = e ? atoi(e) : 0;
    }
    return v;
}

template <int N, int MODE>
static cudaError_t cols_tma_n(const CUtensorMap& map, const AxisGeom& g, const FusedSymbol& sym, const double2* tw,
                              cudaStream_t s) {
    if (tma_persistent() && 3 * TCfg<N>::W * TCfg<N>::LSW * 16 <= 220 * 1024) {
        using C = TCfg<N>;
        const size_t smem = (size_t)3 * C::W * C::LSW * sizeof(double2);
        const i64 ntiles = g.outer * ((g.ncols + C::W - 1) / C::W);
        int dev = 0, sms = 148;
        cudaGetDevice(&dev);
        cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
        kernel_prepare((const void*)k_cols_tma_pers<N, MODE>, smem);
        const int grid = (int)(ntiles < sms ? ntiles : sms);
        k_cols_tma_pers<N, MODE><<<grid, C::NT, smem, s>>>(map, g, sym, tw);
        return cudaGetLastError();
    }
    if constexpr (N == 4096) {
        if (tma_w2()) {
            using C2 = TCfg<N, 2>;
            const size_t smem = C2::smem(MODE);
            const i64 tiles = (g.ncols + C2::W - 1) / C2::W;
            kernel_prepare((const void*)k_cols_tma<N, MODE, 2>, smem);
            k_cols_tma<N, MODE, 2><<<(unsigned)(g.outer * tiles), C2::NT, smem, s>>>(map, g, sym, tw);
            return cudaGetLastError();
        }
    }
    using C = TCfg<N>;
    // tile + (fused mode) the per-frequency real multipliers
    const size_t smem = C::smem(MODE);
    const i64 tiles = (g.ncols + C::W - 1) / C::W;
    kernel_prepare((const void*)k_cols_tma<N, MODE>, smem);
    return launch_pdl(k_cols_tma<N, MODE>, dim3((unsigned)(g.outer * tiles)), dim3(C::NT), smem, s, map, g, sym, tw);
}

// FSX_TMA_W2=1: 2 columns (32 B rows) per 4096-point tile, 1 CTA/SM (measurement)
static int tma_w2() {
    static int v = -1;
    if (v < 0) {
        const char* e = getenv("FSX_TMA_W2");
        v = e ? atoi(e) : 0;
    }
    return v;
}

// columns per TMA tile for a line length (the host builds the box to match)
int tma_cols_width(i64 N) { return N == 4096 && tma_w2() ? 2 : (N >= 4096 ? 1 : (int)(4096 / N)); }

bool tma_cols_ok(i64 N) { return N >= 512 && N <= 8192; }

cudaError_t launch_cols_tma(const void* tensor_map, const AxisGeom& g, int mode, const FusedSymbol& sym,
                            const double2* tw, cudaStream_t s) {
    const CUtensorMap& map = *reinterpret_cast<const CUtensorMap*>(tensor_map);
    if (getenv("FSX_TMA_COPYONLY") && g.n == 4096) return cols_tma_n<4096, 3>(map, g, sym, tw, s);  // measurement
    if (mode == 2 && g.n == 4096 && g.outer == 1 && fused_4step()) {
        const size_t smem = 4096 * sizeof(double2);
        kernel_prepare((const void*)k_fused_tma4, smem);
        k_fused_tma4<<<(unsigned)g.ncols, 256, smem, s>>>(map, g, sym, tw);
        return cudaGetLastError();
    }
#define FSX_TMA(N)                                                    \
    case N:                                                            \
        return mode == 0 ? cols_tma_n<N, 0>(map, g, sym, tw, s)        \
             : mode == 1 ? cols_tma_n<N, 1>(map, g, sym, tw, s)        \
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

int make_cols_tensor_map(void* out_map, void* base, const AxisGeom& g) {
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
    const cuuint32_t box[3] = {(cuuint32_t)(2 * tma_cols_width(g.n)), (cuuint32_t)(g.n < 256 ? g.n : 256), 1};
    const cuuint32_t estr[3] = {1, 1, 1};
    CUresult r = encode(reinterpret_cast<CUtensorMap*>(out_map), CU_TENSOR_MAP_DATA_TYPE_FLOAT64, 3, base, dims, strides,
                        box, estr, CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE,
                        CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    return r == CUDA_SUCCESS ? 0 : (int)r;
}

}  // namespace fsx
