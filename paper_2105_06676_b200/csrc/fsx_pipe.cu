// Persistent, software-pipelined versions of the hot-path passes.
//
// One CTA per (SM x occupancy slot) walks the tiles of its pass with a
// two-stage cp.async pipeline: while tile i is transformed, tile i+1 is
// already streaming into the other shared-memory stage, so HBM reads
// overlap the FFT arithmetic instead of alternating with it (the round-1
// ncu capture of the one-tile-per-CTA kernels showed long-scoreboard stalls
// on the tile loads as the dominant stall at 8-16 warps/SM).
// The stage that holds tile i doubles as that tile's FFT exchange buffer,
// so a CTA needs 2 x tile bytes of shared memory.  Stores are plain
// st.global from registers (fire-and-forget).
//
// Tiles: rows = one line of the contiguous axis (32 / 64 KB); columns =
// W adjacent columns x N of a strided axis (64 KB).  Lines longer than 4096
// complex (128 KB tiles) stay on the one-tile kernels in fsx_kernels.cu.
#include <cstdlib>

#include "fsx_async.cuh"
#include "fsx_device.cuh"
#include "fsx_kernels.h"
#include "fsx_spectral.cuh"

namespace fsx {

__device__ __forceinline__ void cp_async16(void* smem, const void* gmem) {
    const unsigned s = (unsigned)__cvta_generic_to_shared(smem);
    asm volatile("cp.async.cg.shared.global [%0], [%1], 16;\n" ::"r"(s), "l"(gmem) : "memory");
}
__device__ __forceinline__ void cp_commit() { asm volatile("cp.async.commit_group;\n" ::: "memory"); }
template <int NPEND>
__device__ __forceinline__ void cp_wait() {
    asm volatile("cp.async.wait_group %0;\n" ::"n"(NPEND) : "memory");
}

template <int N>
struct PCfg {
    static constexpr int R = 16;
    static constexpr int TPL = N / R;
    static constexpr int W = N >= 4096 ? 1 : 4096 / N;   // columns per strided tile (64 KB)
    static constexpr int GW = W < 8 ? W : 8;
    static constexpr int LSW = GW > 1 ? N + 8 / GW : N;
    static constexpr int TILE_W = W * LSW;               // strided tile, elements
    static constexpr int NT_W = W * TPL;                 // strided threads
    static constexpr int MINB_ROW = (N * 32 <= 64 * 1024) ? 3 : 1;  // rows: 2 x 32 KB stages -> 3 CTAs/SM
};

// ------------------------------------------------------------------ rows: R2C
template <int M, bool BLK>
__global__ void __launch_bounds__(PCfg<M>::TPL, PCfg<M>::MINB_ROW)
k_r2c_pipe(const double* __restrict__ x, double2* __restrict__ H, i64 nrows, i64 L, RowLayout lay,
           const double2* __restrict__ tw_all) {
    using C = PCfg<M>;
    using F = LineFFT<M, -1, true>;
    extern __shared__ double2 sm[];
    const int t = threadIdx.x;
    auto issue = [&](i64 row, int s) {
        const double2* src = reinterpret_cast<const double2*>(x + row * L);
        double2* dst = sm + s * M;
#pragma unroll
        for (int q = 0; q < C::R; ++q) cp_async16(dst + swz(t + q * C::TPL), src + t + q * C::TPL);
    };
    i64 row = blockIdx.x;
    if (row < nrows) issue(row, 0);
    cp_commit();
    for (int s = 0; row < nrows; row += gridDim.x, s ^= 1) {
        const i64 nxt = row + gridDim.x;
        if (nxt < nrows) issue(nxt, s ^ 1);
        cp_commit();
        cp_wait<1>();
        double2* line = sm + s * M;
        double2 v[C::R];
#pragma unroll
        for (int q = 0; q < C::R; ++q) v[q] = line[swz(t + q * C::TPL)];
        F::run(v, t, line, tw_all + M);
        __syncthreads();
#pragma unroll
        for (int q = 0; q < C::R; ++q) line[swz(t + q * C::TPL)] = v[q];
        __syncthreads();
#pragma unroll
        for (int q = 0; q < C::R; ++q) {
            const int k = t + q * C::TPL;
            const double2 zk = v[q];
            const double2 zm = cconj(line[swz((M - k) & (M - 1))]);
            const double2 e = cscale(cadd(zk, zm), 0.5);
            const double2 od = cscale(cmul_si<-1>(csub(zk, zm)), 0.5);
            const double2 w = __ldg(tw_all + 2 * M + k);
            *row_ptr<BLK>(H, lay, row, k) = cadd(e, cmul(w, od));
            if (k == 0) *row_ptr<BLK>(H, lay, row, M) = make_double2(zk.x - zk.y, 0.0);
        }
        __syncthreads();
    }
    cp_wait<0>();
    if (BLK && lay.peers) __threadfence_system();  // remote (NVLink) stores ordered before the rank barrier
}

// ------------------------------------------------------------------ rows: C2R
template <int M, bool BLK>
__global__ void __launch_bounds__(PCfg<M>::TPL, PCfg<M>::MINB_ROW)
k_c2r_pipe(const double2* __restrict__ H, double* __restrict__ x, i64 nrows, i64 L, RowLayout lay,
           const double2* __restrict__ tw_all, Flags* flags) {
    using C = PCfg<M>;
    using F = LineFFT<M, +1, true>;
    extern __shared__ double2 sm[];
    __shared__ double2 nyq[2];
    const int t = threadIdx.x;
    auto issue = [&](i64 row, int s) {
        double2* dst = sm + s * M;
#pragma unroll
        for (int q = 0; q < C::R; ++q) cp_async16(dst + swz(t + q * C::TPL), row_ptr<BLK>(H, lay, row, t + q * C::TPL));
        if (t == 0) cp_async16(&nyq[s], row_ptr<BLK>(H, lay, row, M));
    };
    bool bad = false;
    i64 row = blockIdx.x;
    if (row < nrows) issue(row, 0);
    cp_commit();
    for (int s = 0; row < nrows; row += gridDim.x, s ^= 1) {
        const i64 nxt = row + gridDim.x;
        if (nxt < nrows) issue(nxt, s ^ 1);
        cp_commit();
        cp_wait<1>();
        __syncthreads();
        double2* line = sm + s * M;
        double2 v[C::R];
#pragma unroll
        for (int q = 0; q < C::R; ++q) {
            const int k = t + q * C::TPL;
            const double2 xk = line[swz(k)];
            const double2 xm = cconj(k == 0 ? nyq[s] : line[swz(M - k)]);
            const double2 e = cadd(xk, xm);
            const double2 od = cmulc(csub(xk, xm), __ldg(tw_all + 2 * M + k));
            v[q] = cadd(e, cmul_si<+1>(od));
        }
        F::run(v, t, line, tw_all + M);
        double2* dst = reinterpret_cast<double2*>(x + row * L);
#pragma unroll
        for (int q = 0; q < C::R; ++q) {
            dst[t + q * C::TPL] = v[q];
            bad |= !isfinite(v[q].x) || !isfinite(v[q].y);
        }
        __syncthreads();
    }
    cp_wait<0>();
    const unsigned any = __ballot_sync(0xffffffffu, bad);
    if (any && (threadIdx.x & 31) == 0) atomicOr(&flags->nonfinite, 1u);
}

// ------------------------------------------------------------------ rows, bulk-copy staged
// Same persistent two-stage structure, but the next row lands in shared
// memory through ONE cp.async.bulk (the TMA engine moves it: no per-thread
// cp.async, so neither the global read nor the shared-memory fill goes
// through the LSU/L1 data pipe that bounds the row passes), and the R2C
// split pairs k with M - k in registers where the FFT's last pass allows it
// (LineFFT PAIRED: M = 2^(4a+3)), dropping the split exchange.  Pitch
// layout only (element (row, k) at row * P + k).
// ST stages: 2 = the next row streams in while this one is transformed
// (one CTA's own pipeline); 1 = one 64 KB stage per CTA for the 4096-point
// rows so two CTAs share an SM and overlap each other instead (the two-stage
// version fits one 128 KB CTA per SM: 8 warps, 250 registers).
template <int M, int ST>
struct BulkCfg {
    static constexpr int MINB = ST == 2 ? PCfg<M>::MINB_ROW : ST == 1 ? 2 : 1;
};

// BLK: the output goes to the slab exchange layout (blocked, or straight
// into the peers' buffers over NVLink, RowLayout::ptr); otherwise pitch rows.
// TI = float: fp32 mode (the row lands as floats, half the bytes).  CT is
// the arithmetic: double2, or float2 for the fp32 mode's fp32 row FFT (with
// the float twiddle copy); the half spectrum H is fp64 either way.
template <int M, int ST, bool BLK, class TI = double, class CT = double2>
__global__ void __launch_bounds__(PCfg<M>::TPL, BulkCfg<M, ST>::MINB)
k_r2c_bulk(const TI* __restrict__ x, double2* __restrict__ H, i64 nrows, i64 L, RowLayout lay,
           const CT* __restrict__ tw_all) {
    using F = LineFFT<M, -1, true, true, 0, 0, CT>;
    constexpr int TPL = PCfg<M>::TPL, R = 16;
    constexpr unsigned BYTES = 2 * M * sizeof(TI);
    extern __shared__ __align__(128) double2 sm[];
    __shared__ __align__(8) unsigned long long bar[ST];
    const int t = threadIdx.x;
    const i64 G = gridDim.x;
    i64 row = blockIdx.x;
    if (t == 0) {
#pragma unroll
        for (int b = 0; b < ST; ++b) mbar_init(&bar[b], 1);
        mbar_init_fence();
        pdl_wait();  // x may be the predecessor's output
#pragma unroll
        for (int b = 0; b < (ST > 1 ? ST - 1 : 1); ++b)  // ST > 1: the first ST - 1 rows in flight
            if (row + b * G < nrows) {
                mbar_expect_tx(&bar[b], BYTES);
                bulk_load(sm + b * M, x + (row + b * G) * L, BYTES, &bar[b]);
            }
    }
    __syncthreads();
    unsigned par = 0;  // bit s: parity of the next completion of stage s
    for (int s = 0; row < nrows; row += G, s = (ST > 1 ? (s + 1) % ST : 0)) {
        const i64 nxt = row + G;
        const i64 pre = row + (ST - 1) * G;  // ST > 1: the row that now enters the stage the last one freed
        const int sp = (s + ST - 1) % ST;
        if (ST > 1 && t == 0 && pre < nrows) {
            mbar_expect_tx(&bar[sp], BYTES);
            bulk_load(sm + sp * M, x + pre * L, BYTES, &bar[sp]);
        }
        if (nxt >= nrows) pdl_trigger();  // last row of this CTA: let the successor launch
        mbar_wait(&bar[s], (par >> s) & 1u);
        par ^= 1u << s;
        CT* line = reinterpret_cast<CT*>(sm + s * M);
        CT v[R];
        if constexpr (sizeof(TI) == 8) {
#pragma unroll
            for (int q = 0; q < R; ++q) v[q] = from_d2<CT>(sm[s * M + t + q * TPL]);
        } else {
            const float2* lf = reinterpret_cast<const float2*>(sm + s * M);
#pragma unroll
            for (int q = 0; q < R; ++q) {
                const float2 f = lf[t + q * TPL];
                if constexpr (sizeof(CT) == 8) v[q] = f;
                else v[q] = make_double2(f.x, f.y);
            }
        }
        F::run(v, t, line, tw_all + M);
        auto h = [&](int k) -> double2& { return *row_ptr<BLK>(H, lay, row, k); };
        if constexpr (F::PAIRED) {
            // v[i + 2u] = Z[item(i) + u M/8]; the mirror M - k lives in this thread.
            // Split twiddle W_L^(j + u M/8) = W_L^j * W_16^u: one load per item.
            const int j1 = t == 0 ? TPL : 2 * TPL - t;
#pragma unroll
            for (int i = 0; i < 2; ++i) {
                const int j = i == 0 ? t : j1;
                const CT wj = __ldg(tw_all + 2 * M + j);
                static_for<0, 8>([&](auto U) {
                    constexpr int u = decltype(U)::value;
                    const int qp = (1 - i) + 2 * (7 - u);                        // partner slot, t != 0
                    const int qz = i == 0 ? 2 * ((8 - u) & 7) : 1 + 2 * (7 - u);  // partner slot, t == 0
                    const CT zk = v[i + 2 * u];
                    const CT zm = cconj(t == 0 ? v[qz] : v[qp]);
                    const CT e = cscale(cadd(zk, zm), 0.5);
                    const CT od = cscale(cmul_si<-1>(csub(zk, zm)), 0.5);
                    if (lay.kcut < 0 || j + u * (M / 8) <= lay.kcut)
                        h(j + u * (M / 8)) = to_d2(cadd(e, cmul(cmul_const<u, 16, -1>(wj), od)));
                    if (i == 0 && u == 0 && t == 0 && (lay.kcut < 0 || lay.kcut >= M))
                        h(M) = make_double2((double)zk.x - (double)zk.y, 0.0);
                });
            }
        } else {
            __syncthreads();
#pragma unroll
            for (int q = 0; q < R; ++q) line[swz(t + q * TPL)] = v[q];
            __syncthreads();
            const CT wt = __ldg(tw_all + 2 * M + t);  // W_L^(t + q M/16) = W_L^t * W_32^q
            static_for<0, R>([&](auto Q) {
                constexpr int q = decltype(Q)::value;
                const int k = t + q * TPL;
                const CT zk = v[q];
                const CT zm = cconj(line[swz((M - k) & (M - 1))]);
                const CT e = cscale(cadd(zk, zm), 0.5);
                const CT od = cscale(cmul_si<-1>(csub(zk, zm)), 0.5);
                if (lay.kcut < 0 || k <= lay.kcut) h(k) = to_d2(cadd(e, cmul(cmul_const<q, 32, -1>(wt), od)));
                if (k == 0 && (lay.kcut < 0 || lay.kcut >= M)) h(M) = make_double2((double)zk.x - (double)zk.y, 0.0);
            });
        }
        fence_proxy_async();  // generic writes of this stage before its next bulk fill
        __syncthreads();
        if (ST == 1 && t == 0 && nxt < nrows) {
            mbar_expect_tx(&bar[0], BYTES);
            bulk_load(sm, x + nxt * L, BYTES, &bar[0]);
        }
    }
    if (BLK && lay.peers) __threadfence_system();  // remote (NVLink) stores ordered before the rank barrier
}

// One half-spectrum row (M + 1 complex) into shared memory: one bulk copy
// from a pitch row, or one per column block of the slab exchange layout
// (local blocked buffer or the owning ranks' buffers over NVLink).
template <int M, bool BLK>
__device__ __forceinline__ void load_hrow(double2* dst, const double2* H, const RowLayout& lay, i64 row,
                                          unsigned long long* bar) {
    const unsigned nk = (unsigned)(BLK || lay.kcut < 0 || lay.kcut >= M ? M + 1 : lay.kcut + 1);
    mbar_expect_tx(bar, nk * (unsigned)sizeof(double2));
    if constexpr (!BLK) {
        bulk_load(dst, H + row * lay.P, nk * (unsigned)sizeof(double2), bar);
    } else {
        for (i64 k0 = 0; k0 <= M; k0 += lay.blk) {
            const i64 len = (M + 1 - k0) < lay.blk ? (M + 1 - k0) : lay.blk;
            bulk_load(dst + k0, lay.ptr(H, row, k0), (unsigned)(len * sizeof(double2)), bar);
        }
    }
}

// TO = float: fp32 mode (rounded to nearest on the store; a value outside the
// float range becomes inf and raises the non-finite flag).  CT: the
// arithmetic, as in k_r2c_bulk.
template <int M, int ST, bool BLK, class TO = double, class CT = double2>
__global__ void __launch_bounds__(PCfg<M>::TPL, BulkCfg<M, ST>::MINB)
k_c2r_bulk(const double2* __restrict__ H, TO* __restrict__ x, i64 nrows, i64 L, RowLayout lay,
           const CT* __restrict__ tw_all, Flags* flags) {
    using F = LineFFT<M, +1, true, false, 0, 0, CT>;
    constexpr int TPL = PCfg<M>::TPL, R = 16;
    constexpr int SS = M + 8;  // stage stride: M + 1 elements, 128 B aligned
    extern __shared__ __align__(128) double2 sm[];
    __shared__ __align__(8) unsigned long long bar[ST];
    const int t = threadIdx.x;
    const i64 G = gridDim.x;
    bool bad = false;
    i64 row = blockIdx.x;
    if (t == 0) {
#pragma unroll
        for (int b = 0; b < ST; ++b) mbar_init(&bar[b], 1);
        mbar_init_fence();
        pdl_wait();  // H is the predecessor's output
#pragma unroll
        for (int b = 0; b < (ST > 1 ? ST - 1 : 1); ++b)
            if (row + b * G < nrows) load_hrow<M, BLK>(sm + b * SS, H, lay, row + b * G, &bar[b]);
    }
    __syncthreads();
    unsigned par = 0;
    for (int s = 0; row < nrows; row += G, s = (ST > 1 ? (s + 1) % ST : 0)) {
        const i64 nxt = row + G;
        const i64 pre = row + (ST - 1) * G;
        const int sp = (s + ST - 1) % ST;
        if (ST > 1 && t == 0 && pre < nrows) load_hrow<M, BLK>(sm + sp * SS, H, lay, pre, &bar[sp]);
        if (nxt >= nrows) pdl_trigger();
        mbar_wait(&bar[s], (par >> s) & 1u);
        par ^= 1u << s;
        double2* line = sm + s * SS;
        if (!BLK && lay.kcut >= 0 && lay.kcut < M) {  // exact spectral cut: the dropped columns are 0
            for (i64 k = lay.kcut + 1 + t; k <= M; k += TPL) line[k] = make_double2(0.0, 0.0);
            __syncthreads();
        }
        CT v[R];
        // split twiddle W_L^(t + q M/16) = W_L^t * W_32^q: one load per thread
        const CT wt = __ldg(tw_all + 2 * M + t);
        static_for<0, R>([&](auto Q) {
            constexpr int q = decltype(Q)::value;
            const int k = t + q * TPL;
            const CT xk = from_d2<CT>(line[k]);
            const CT xm = cconj(from_d2<CT>(line[M - k]));
            const CT e = cadd(xk, xm);
            const CT od = cmulc(csub(xk, xm), cmul_const<q, 32, -1>(wt));
            v[q] = cadd(e, cmul_si<+1>(od));
        });
        F::run(v, t, reinterpret_cast<CT*>(line), tw_all + M);
        if constexpr (sizeof(TO) == 8) {
            double2* dst = reinterpret_cast<double2*>(x + row * L);
#pragma unroll
            for (int q = 0; q < R; ++q) {
                const double2 d = to_d2(v[q]);
                dst[t + q * TPL] = d;
                bad |= !isfinite(d.x) || !isfinite(d.y);
            }
        } else {
            float2* dst = reinterpret_cast<float2*>(x + row * L);
#pragma unroll
            for (int q = 0; q < R; ++q) {
                const float2 f = make_float2((float)v[q].x, (float)v[q].y);
                dst[t + q * TPL] = f;
                bad |= !isfinite(f.x) || !isfinite(f.y);
            }
        }
        fence_proxy_async();
        __syncthreads();
        if (ST == 1 && t == 0 && nxt < nrows) load_hrow<M, BLK>(sm, H, lay, nxt, &bar[0]);
    }
    const unsigned any = __ballot_sync(0xffffffffu, bad);
    if (any && (threadIdx.x & 31) == 0) atomicOr(&flags->nonfinite, 1u);
}

// ------------------------------------------------------------------ rows, two groups per CTA
// The bulk-staged row kernels at M = 4096 (cfg3's 8192-real rows) run one
// 256-thread CTA per SM (three 64 KB stages fill shared memory): 8 warps,
// ncu 12 % warps active, latency-bound at ~4.5 TB/s.  Here the same three
// stages feed TWO 256-thread groups of one CTA (16 warps per SM): row j of
// the CTA (global row blockIdx + j G) lands in stage j % 3 and is transformed
// by group j % 2 with named-barrier exchanges; the group that frees a stage
// refills it with row j + 3 at once.  A stage's row tag (written when its
// refill is issued) tells the consumer which load the stage's mbarrier phase
// belongs to, so a group never mistakes an older phase for its row's.
template <int NG>
__device__ __forceinline__ void grp_wait_stage(volatile int* tag, int s, int j, unsigned long long* bar, int ST) {
    while (tag[s] != j) {
    }
    mbar_wait(bar, (unsigned)(j / ST) & 1u);
}

template <int M, int NG, int ST, int MINB = 1>
__global__ void __launch_bounds__(NG * PCfg<M>::TPL, MINB)
k_r2c_grp(const double* __restrict__ x, double2* __restrict__ H, i64 nrows, i64 L, RowLayout lay,
          const double2* __restrict__ tw_all) {
    constexpr int TPL = PCfg<M>::TPL, R = 16;
    #ifndef FSX_ROWS_LPF
#define FSX_ROWS_LPF 1  // cfg3 rows ~1 % (r02v)
#endif
    using F = LineFFT<M, -1, false, false, 0, TPL, double2, FSX_ROWS_LPF != 0>;  // named barriers per group
    static_assert(!F::PAIRED, "k_r2c_grp: split through the exchange line (M = 2^(4a))");
    constexpr unsigned BYTES = 2 * M * sizeof(double);
    extern __shared__ __align__(128) double2 sm[];
    __shared__ __align__(8) unsigned long long bar[ST];
    __shared__ int tag[ST];
    const int g = threadIdx.x / TPL, t = threadIdx.x % TPL;
    const i64 G = gridDim.x;
    if (threadIdx.x == 0) {
#pragma unroll
        for (int b = 0; b < ST; ++b) mbar_init(&bar[b], 1);
        mbar_init_fence();
        pdl_wait();  // x may be the predecessor's output
#pragma unroll
        for (int j = 0; j < ST; ++j) {
            tag[j] = j;
            const i64 row = blockIdx.x + (i64)j * G;
            if (row < nrows) {
                mbar_expect_tx(&bar[j], BYTES);
                bulk_load(sm + j * M, x + row * L, BYTES, &bar[j]);
            }
        }
    }
    __syncthreads();
    for (int j = g;; j += NG) {
        const i64 row = blockIdx.x + (i64)j * G;
        if (row >= nrows) break;
        const int s = j % ST;
        if (row + (i64)NG * G >= nrows) pdl_trigger();  // this group's last row
        grp_wait_stage<NG>(tag, s, j, &bar[s], ST);
        double2* line = sm + s * M;
        double2 v[R];
#pragma unroll
        for (int q = 0; q < R; ++q) v[q] = line[t + q * TPL];
        F::run(v, t, line, tw_all + M);
        group_sync<TPL>();
#pragma unroll
        for (int q = 0; q < R; ++q) line[swz(t + q * TPL)] = v[q];
        group_sync<TPL>();
        const double2 wt = __ldg(tw_all + 2 * M + t);  // W_L^(t + q M/16) = W_L^t * W_32^q
        static_for<0, R>([&](auto Q) {
            constexpr int q = decltype(Q)::value;
            const int k = t + q * TPL;
            const double2 zk = v[q];
            const double2 zm = cconj(line[swz((M - k) & (M - 1))]);
            const double2 e = cscale(cadd(zk, zm), 0.5);
            const double2 od = cscale(cmul_si<-1>(csub(zk, zm)), 0.5);
            if (lay.kcut < 0 || k <= lay.kcut) H[row * lay.P + k] = cadd(e, cmul(cmul_const<q, 32, -1>(wt), od));
            if (k == 0 && (lay.kcut < 0 || lay.kcut >= M)) H[row * lay.P + M] = make_double2(zk.x - zk.y, 0.0);
        });
        fence_proxy_async();  // generic writes of this stage before its next bulk fill
        group_sync<TPL>();
        const i64 nrow = blockIdx.x + (i64)(j + ST) * G;
        if (t == 0 && nrow < nrows) {
            mbar_expect_tx(&bar[s], BYTES);
            bulk_load(sm + s * M, x + nrow * L, BYTES, &bar[s]);
            __threadfence_block();
            tag[s] = j + ST;
        }
    }
}

template <int M, int NG, int ST, int MINB = 1>
__global__ void __launch_bounds__(NG * PCfg<M>::TPL, MINB)
k_c2r_grp(const double2* __restrict__ H, double* __restrict__ x, i64 nrows, i64 L, RowLayout lay,
          const double2* __restrict__ tw_all, Flags* flags) {
    constexpr int TPL = PCfg<M>::TPL, R = 16;
    using F = LineFFT<M, +1, false, false, 0, TPL, double2, FSX_ROWS_LPF != 0>;
    constexpr int SS = M + 8;  // stage stride: M + 1 elements, 128 B aligned
    extern __shared__ __align__(128) double2 sm[];
    __shared__ __align__(8) unsigned long long bar[ST];
    __shared__ int tag[ST];
    const int g = threadIdx.x / TPL, t = threadIdx.x % TPL;
    const i64 G = gridDim.x;
    bool bad = false;
    if (threadIdx.x == 0) {
#pragma unroll
        for (int b = 0; b < ST; ++b) mbar_init(&bar[b], 1);
        mbar_init_fence();
        pdl_wait();  // H is the predecessor's output
#pragma unroll
        for (int j = 0; j < ST; ++j) {
            tag[j] = j;
            const i64 row = blockIdx.x + (i64)j * G;
            if (row < nrows) load_hrow<M, false>(sm + j * SS, H, lay, row, &bar[j]);
        }
    }
    __syncthreads();
    for (int j = g;; j += NG) {
        const i64 row = blockIdx.x + (i64)j * G;
        if (row >= nrows) break;
        const int s = j % ST;
        if (row + (i64)NG * G >= nrows) pdl_trigger();
        grp_wait_stage<NG>(tag, s, j, &bar[s], ST);
        double2* line = sm + s * SS;
        if (lay.kcut >= 0 && lay.kcut < M) {  // exact spectral cut: the dropped columns are 0
            for (i64 k = lay.kcut + 1 + t; k <= M; k += TPL) line[k] = make_double2(0.0, 0.0);
            group_sync<TPL>();
        }
        double2 v[R];
        const double2 wt = __ldg(tw_all + 2 * M + t);  // W_L^(t + q M/16) = W_L^t * W_32^q
        static_for<0, R>([&](auto Q) {
            constexpr int q = decltype(Q)::value;
            const int k = t + q * TPL;
            const double2 xk = line[k];
            const double2 xm = cconj(line[M - k]);
            const double2 e = cadd(xk, xm);
            const double2 od = cmulc(csub(xk, xm), cmul_const<q, 32, -1>(wt));
            v[q] = cadd(e, cmul_si<+1>(od));
        });
        F::run(v, t, line, tw_all + M);
        double2* dst = reinterpret_cast<double2*>(x + row * L);
#pragma unroll
        for (int q = 0; q < R; ++q) {
            dst[t + q * TPL] = v[q];
            bad |= !isfinite(v[q].x) || !isfinite(v[q].y);
        }
        fence_proxy_async();
        group_sync<TPL>();
        const i64 nrow = blockIdx.x + (i64)(j + ST) * G;
        if (t == 0 && nrow < nrows) {
            load_hrow<M, false>(sm + s * SS, H, lay, nrow, &bar[s]);
            __threadfence_block();
            tag[s] = j + ST;
        }
    }
    const unsigned any = __ballot_sync(0xffffffffu, bad);
    if (any && (threadIdx.x & 31) == 0) atomicOr(&flags->nonfinite, 1u);
}

// FSX_ROWS: 0 = one-row-per-CTA kernels, 1 = cp.async staged (cfg2 r2c 70 us /
// c2r 64 us at the time), 3 = bulk-copy staged (default: 67 / 63 us then, 52 / 51 us
// with the later twiddle work).  A register double-buffered variant (86 / 109 us)
// was removed.
int rows_variant() {
    static int v = -1;
    if (v < 0) {
        const char* e = getenv("FSX_ROWS");
        v = e ? atoi(e) : 3;
    }
    return v;
}


// ------------------------------------------------------------------ columns
// Tile = W adjacent columns x N of a strided axis.  MODE 0: forward C2C,
// 1: inverse C2C, 2: fused R2C spectral pass (forward, lam^T x / N, inverse).
template <int N, int MODE>
__global__ void __launch_bounds__(PCfg<N>::NT_W, 1)
k_cols_pipe(double2* H, AxisGeom g, FusedSymbol sym, const double2* __restrict__ tw_all) {
    using C = PCfg<N>;
    using FF = LineFFT<N, -1, true>;
    using FI = LineFFT<N, +1, true>;
    extern __shared__ double2 sm[];
    __shared__ double2 acoef[kMaxGroups][C::W];
    __shared__ double2 tapterm[MODE == 2 ? kMaxFusedTaps : 1][C::W];
    const int w = threadIdx.x % C::W, t = threadIdx.x / C::W;
    const i64 tiles_per_outer = (g.ncols + C::W - 1) / C::W;
    const i64 ntiles = g.outer * tiles_per_outer;
    auto colof = [&](i64 tile, i64& base, i64& c) {
        const i64 o = tile / tiles_per_outer;
        c = (tile - o * tiles_per_outer) * C::W + w;
        base = o * g.block + c;
    };
    auto valid = [&](i64 c) {
        if (c >= g.ncols) return false;
        if (MODE == 2) {
            i64 kx, ky;
            fused_col_freqs(sym, c, kx, ky);
            return kx <= sym.M;
        }
        return true;
    };
    auto issue = [&](i64 tile, int s) {
        i64 base, c;
        colof(tile, base, c);
        if (!valid(c)) return;
        double2* dst = sm + s * C::TILE_W + w * C::LSW;
#pragma unroll
        for (int q = 0; q < C::R; ++q) cp_async16(dst + swz(t + q * C::TPL), H + base + (i64)(t + q * C::TPL) * g.inner);
    };
    i64 tile = blockIdx.x;
    if (tile < ntiles) issue(tile, 0);
    cp_commit();
    for (int s = 0; tile < ntiles; tile += gridDim.x, s ^= 1) {
        const i64 nxt = tile + gridDim.x;
        if (nxt < ntiles) issue(nxt, s ^ 1);
        cp_commit();
        i64 base, c;
        colof(tile, base, c);
        const bool ok = valid(c);
        if constexpr (MODE == 2) {
            i64 kx, ky;
            fused_col_freqs(sym, c, kx, ky);
            for (int j = t; j < sym.ntaps; j += C::TPL) tapterm[j][w] = tap_term(sym, tw_all, j, kx, ky);
        }
        cp_wait<1>();
        double2* line = sm + s * C::TILE_W + w * C::LSW;
        double2 v[C::R];
#pragma unroll
        for (int q = 0; q < C::R; ++q) v[q] = line[swz(t + q * C::TPL)];
        if constexpr (MODE == 1) {
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
        if (ok) {
#pragma unroll
            for (int q = 0; q < C::R; ++q) H[base + (i64)(t + q * C::TPL) * g.inner] = v[q];
        }
        __syncthreads();
    }
    cp_wait<0>();
}

// ================================================================== launchers
static int sm_count() {
    static int n = 0;
    if (!n) {
        int dev = 0;
        cudaGetDevice(&dev);
        cudaDeviceGetAttribute(&n, cudaDevAttrMultiProcessorCount, dev);
        if (n <= 0) n = 148;
    }
    return n;
}

template <class K>
static int persistent_grid(K kernel, int threads, size_t smem, i64 ntiles) {
    int per_sm = 0;
    per_sm = kernel_prepare((const void*)kernel, smem, threads);
    if (per_sm < 1) per_sm = 1;
    const i64 g = (i64)per_sm * sm_count();
    return (int)(ntiles < g ? ntiles : g);
}

template <int M>
static cudaError_t r2c_pipe_m(const double* x, double2* H, i64 nrows, i64 L, const RowLayout& P, const double2* tw, cudaStream_t s) {
    const size_t smem = (size_t)2 * M * sizeof(double2);
    auto kf = P.blk ? k_r2c_pipe<M, true> : k_r2c_pipe<M, false>;
    kernel_prepare((const void*)kf, smem);
    const int grid = persistent_grid(kf, PCfg<M>::TPL, smem, nrows);
    kf<<<grid, PCfg<M>::TPL, smem, s>>>(x, H, nrows, L, P, tw);
    return cudaGetLastError();
}

template <int M>
static cudaError_t c2r_pipe_m(const double2* H, double* x, i64 nrows, i64 L, const RowLayout& P, const double2* tw, Flags* f,
                              cudaStream_t s) {
    const size_t smem = (size_t)2 * M * sizeof(double2);
    auto kf = P.blk ? k_c2r_pipe<M, true> : k_c2r_pipe<M, false>;
    kernel_prepare((const void*)kf, smem);
    const int grid = persistent_grid(kf, PCfg<M>::TPL, smem, nrows);
    kf<<<grid, PCfg<M>::TPL, smem, s>>>(H, x, nrows, L, P, tw, f);
    return cudaGetLastError();
}

// FSX_ROW_STAGES=1/2/3 selects the stage count (A/B); default 3 at M = 4096, else 2
static int row_stages(int M) {
    static int v = -1;
    if (v < 0) {
        const char* e = getenv("FSX_ROW_STAGES");
        v = e ? atoi(e) : 0;
    }
    // 1 stage x 2 CTAs measured slower at M = 4096 (269 vs 254 us); 3 stages (two rows in flight,
    // one 192 KB CTA per SM) measured 243 -> 238 us for the M = 4096 R2C rows (default there)
    if (v == 1 || v == 2 || v == 3) return v;
    return M == 4096 ? 3 : 2;
}

template <int M, int ST, bool BLK>
static cudaError_t r2c_bulk_ms(const double* x, double2* H, i64 nrows, i64 L, const RowLayout& lay, const double2* tw,
                               cudaStream_t s) {
    const size_t smem = (size_t)ST * M * sizeof(double2);
    auto kf = k_r2c_bulk<M, ST, BLK>;
    kernel_prepare((const void*)kf, smem);
    const int grid = persistent_grid(kf, PCfg<M>::TPL, smem, nrows);
    return launch_pdl(kf, dim3(grid), dim3(PCfg<M>::TPL), smem, s, x, H, nrows, L, lay, tw);
}

// FSX_ROW_GROUPS=0 keeps the one-group kernels at M = 4096 (A/B)
static bool row_groups() {
    static int v = -1;
    if (v < 0) {
        const char* e = getenv("FSX_ROW_GROUPS");
        v = e ? atoi(e) : 1;
    }
    return v != 0;
}

// FSX_ROW_GROUPS=2 also runs the M = 2048 rows as groups (A/B)
static bool row_groups_m2048() {
    static int v = -1;
    if (v < 0) {
        const char* e = getenv("FSX_ROW_GROUPS");
        v = e ? atoi(e) : 1;
    }
    return v == 2;
}

template <int M>
static cudaError_t r2c_bulk_m(const double* x, double2* H, i64 nrows, i64 L, const RowLayout& lay, const double2* tw,
                              cudaStream_t s) {
    if (lay.blk) return r2c_bulk_ms<M, 2, true>(x, H, nrows, L, lay, tw, s);
    if constexpr (M == 2048)
        if (row_groups_m2048()) {  // two 128-thread groups on three 32 KB stages, two CTAs per SM
            const size_t smem = (size_t)3 * M * sizeof(double2);
            auto kf = k_r2c_grp<M, 2, 3, 2>;
            kernel_prepare((const void*)kf, smem);
            const int grid = persistent_grid(kf, 2 * PCfg<M>::TPL, smem, (nrows + 1) / 2);
            return launch_pdl(kf, dim3(grid), dim3(2 * PCfg<M>::TPL), smem, s, x, H, nrows, L, lay, tw);
        }
    if constexpr (M == 4096)
        if (row_groups()) {  // two 256-thread groups on three 64 KB stages
            const size_t smem = (size_t)3 * M * sizeof(double2);
            auto kf = k_r2c_grp<M, 2, 3>;
            kernel_prepare((const void*)kf, smem);
            const int grid = persistent_grid(kf, 2 * PCfg<M>::TPL, smem, (nrows + 1) / 2);
            return launch_pdl(kf, dim3(grid), dim3(2 * PCfg<M>::TPL), smem, s, x, H, nrows, L, lay, tw);
        }
    if constexpr (M == 4096)  // FSX_ROW_STAGES=3: three 64 KB stages (two rows in flight)
        if (row_stages(M) == 3) return r2c_bulk_ms<M, 3, false>(x, H, nrows, L, lay, tw, s);
    return row_stages(M) == 1 ? r2c_bulk_ms<M, 1, false>(x, H, nrows, L, lay, tw, s)
                              : r2c_bulk_ms<M, 2, false>(x, H, nrows, L, lay, tw, s);
}

template <int M, int ST, bool BLK>
static cudaError_t c2r_bulk_ms(const double2* H, double* x, i64 nrows, i64 L, const RowLayout& lay, const double2* tw,
                               Flags* f, cudaStream_t s) {
    const size_t smem = (size_t)ST * (M + 8) * sizeof(double2);
    auto kf = k_c2r_bulk<M, ST, BLK>;
    kernel_prepare((const void*)kf, smem);
    const int grid = persistent_grid(kf, PCfg<M>::TPL, smem, nrows);
    return launch_pdl(kf, dim3(grid), dim3(PCfg<M>::TPL), smem, s, H, x, nrows, L, lay, tw, f);
}

template <int M>
static cudaError_t c2r_bulk_m(const double2* H, double* x, i64 nrows, i64 L, const RowLayout& lay, const double2* tw,
                              Flags* f, cudaStream_t s) {
    if (lay.blk) return c2r_bulk_ms<M, 2, true>(H, x, nrows, L, lay, tw, f, s);
    if constexpr (M == 2048)
        if (row_groups_m2048()) {
            const size_t smem = (size_t)3 * (M + 8) * sizeof(double2);
            auto kf = k_c2r_grp<M, 2, 3, 2>;
            kernel_prepare((const void*)kf, smem);
            const int grid = persistent_grid(kf, 2 * PCfg<M>::TPL, smem, (nrows + 1) / 2);
            return launch_pdl(kf, dim3(grid), dim3(2 * PCfg<M>::TPL), smem, s, H, x, nrows, L, lay, tw, f);
        }
    if constexpr (M == 4096)
        if (row_groups()) {
            const size_t smem = (size_t)3 * (M + 8) * sizeof(double2);
            auto kf = k_c2r_grp<M, 2, 3>;
            kernel_prepare((const void*)kf, smem);
            const int grid = persistent_grid(kf, 2 * PCfg<M>::TPL, smem, (nrows + 1) / 2);
            return launch_pdl(kf, dim3(grid), dim3(2 * PCfg<M>::TPL), smem, s, H, x, nrows, L, lay, tw, f);
        }
    if constexpr (M == 4096)
        if (row_stages(M) == 3) return c2r_bulk_ms<M, 3, false>(H, x, nrows, L, lay, tw, f, s);
    return row_stages(M) == 1 ? c2r_bulk_ms<M, 1, false>(H, x, nrows, L, lay, tw, f, s)
                              : c2r_bulk_ms<M, 2, false>(H, x, nrows, L, lay, tw, f, s);
}

template <int N, int MODE>
static cudaError_t cols_pipe_n(double2* H, const AxisGeom& g, const FusedSymbol& sym, const double2* tw, cudaStream_t s) {
    using C = PCfg<N>;
    const size_t smem = (size_t)2 * C::TILE_W * sizeof(double2);
    kernel_prepare((const void*)k_cols_pipe<N, MODE>, smem);
    const i64 ntiles = g.outer * ((g.ncols + C::W - 1) / C::W);
    const int grid = persistent_grid(k_cols_pipe<N, MODE>, C::NT_W, smem, ntiles);
    k_cols_pipe<N, MODE><<<grid, C::NT_W, smem, s>>>(H, g, sym, tw);
    return cudaGetLastError();
}

// FSX_PIPE=0 selects the one-tile-per-CTA kernels (A/B measurements).
bool pipe_enabled() {
    static int on = -1;
    if (on < 0) {
        const char* e = getenv("FSX_PIPE");
        on = (e && e[0] == '0') ? 0 : 1;
    }
    return on == 1;
}

bool pipe_rows_ok(i64 M) { return M >= 512 && M <= 4096; }
bool pipe_cols_ok(i64 N) { return N >= 1024 && N <= 4096; }

cudaError_t launch_r2c_pipe(const double* x, double2* H, i64 nrows, i64 L, const RowLayout& P, const double2* tw, cudaStream_t s) {
    switch (L / 2) {
        case 512: return r2c_pipe_m<512>(x, H, nrows, L, P, tw, s);
        case 1024: return r2c_pipe_m<1024>(x, H, nrows, L, P, tw, s);
        case 2048: return r2c_pipe_m<2048>(x, H, nrows, L, P, tw, s);
        case 4096: return r2c_pipe_m<4096>(x, H, nrows, L, P, tw, s);
        default: return cudaErrorInvalidValue;
    }
}

cudaError_t launch_c2r_pipe(const double2* H, double* x, i64 nrows, i64 L, const RowLayout& P, const double2* tw, Flags* f,
                            cudaStream_t s) {
    switch (L / 2) {
        case 512: return c2r_pipe_m<512>(H, x, nrows, L, P, tw, f, s);
        case 1024: return c2r_pipe_m<1024>(H, x, nrows, L, P, tw, f, s);
        case 2048: return c2r_pipe_m<2048>(H, x, nrows, L, P, tw, f, s);
        case 4096: return c2r_pipe_m<4096>(H, x, nrows, L, P, tw, f, s);
        default: return cudaErrorInvalidValue;
    }
}

cudaError_t launch_r2c_bulk(const double* x, double2* H, i64 nrows, i64 L, const RowLayout& lay, const double2* tw,
                            cudaStream_t s) {
    switch (L / 2) {
        case 512: return r2c_bulk_m<512>(x, H, nrows, L, lay, tw, s);
        case 1024: return r2c_bulk_m<1024>(x, H, nrows, L, lay, tw, s);
        case 2048: return r2c_bulk_m<2048>(x, H, nrows, L, lay, tw, s);
        case 4096: return r2c_bulk_m<4096>(x, H, nrows, L, lay, tw, s);
        default: return cudaErrorInvalidValue;
    }
}

cudaError_t launch_c2r_bulk(const double2* H, double* x, i64 nrows, i64 L, const RowLayout& lay, const double2* tw,
                            Flags* f, cudaStream_t s) {
    switch (L / 2) {
        case 512: return c2r_bulk_m<512>(H, x, nrows, L, lay, tw, f, s);
        case 1024: return c2r_bulk_m<1024>(H, x, nrows, L, lay, tw, f, s);
        case 2048: return c2r_bulk_m<2048>(H, x, nrows, L, lay, tw, f, s);
        case 4096: return c2r_bulk_m<4096>(H, x, nrows, L, lay, tw, f, s);
        default: return cudaErrorInvalidValue;
    }
}

// fp32 storage mode rows (pitch layout, two stages as the fp64 default)
// (twf: the float twiddle copy -> fp32 row FFTs; nullptr -> fp64 arithmetic)
template <int M>
static cudaError_t r2c_bulk_f32_m(const float* x, double2* H, i64 nrows, i64 L, const RowLayout& lay, const double2* tw,
                                  const float2* twf, cudaStream_t s) {
    const size_t smem = (size_t)2 * M * sizeof(double2);
    if (twf) {
        auto kf = k_r2c_bulk<M, 2, false, float, float2>;
        kernel_prepare((const void*)kf, smem);
        const int grid = persistent_grid(kf, PCfg<M>::TPL, smem, nrows);
        return launch_pdl(kf, dim3(grid), dim3(PCfg<M>::TPL), smem, s, x, H, nrows, L, lay, twf);
    }
    auto kf = k_r2c_bulk<M, 2, false, float>;
    kernel_prepare((const void*)kf, smem);
    const int grid = persistent_grid(kf, PCfg<M>::TPL, smem, nrows);
    return launch_pdl(kf, dim3(grid), dim3(PCfg<M>::TPL), smem, s, x, H, nrows, L, lay, tw);
}

template <int M>
static cudaError_t c2r_bulk_f32_m(const double2* H, float* x, i64 nrows, i64 L, const RowLayout& lay, const double2* tw,
                                  const float2* twf, Flags* f, cudaStream_t s) {
    const size_t smem = (size_t)2 * (M + 8) * sizeof(double2);
    if (twf) {
        auto kf = k_c2r_bulk<M, 2, false, float, float2>;
        kernel_prepare((const void*)kf, smem);
        const int grid = persistent_grid(kf, PCfg<M>::TPL, smem, nrows);
        return launch_pdl(kf, dim3(grid), dim3(PCfg<M>::TPL), smem, s, H, x, nrows, L, lay, twf, f);
    }
    auto kf = k_c2r_bulk<M, 2, false, float>;
    kernel_prepare((const void*)kf, smem);
    const int grid = persistent_grid(kf, PCfg<M>::TPL, smem, nrows);
    return launch_pdl(kf, dim3(grid), dim3(PCfg<M>::TPL), smem, s, H, x, nrows, L, lay, tw, f);
}

bool rows_f32_ok(i64 L) { return pipe_enabled() && pipe_rows_ok(L / 2) && rows_variant() == 3; }

cudaError_t launch_r2c_rows_f32(const float* x, double2* H, i64 nrows, i64 L, const RowLayout& lay, const double2* tw,
                                const float2* twf, cudaStream_t s) {
    if (lay.blk) return cudaErrorInvalidValue;
    switch (L / 2) {
        case 512: return r2c_bulk_f32_m<512>(x, H, nrows, L, lay, tw, twf, s);
        case 1024: return r2c_bulk_f32_m<1024>(x, H, nrows, L, lay, tw, twf, s);
        case 2048: return r2c_bulk_f32_m<2048>(x, H, nrows, L, lay, tw, twf, s);
        case 4096: return r2c_bulk_f32_m<4096>(x, H, nrows, L, lay, tw, twf, s);
        default: return cudaErrorInvalidValue;
    }
}

cudaError_t launch_c2r_rows_f32(const double2* H, float* x, i64 nrows, i64 L, const RowLayout& lay, const double2* tw,
                                const float2* twf, Flags* f, cudaStream_t s) {
    if (lay.blk) return cudaErrorInvalidValue;
    switch (L / 2) {
        case 512: return c2r_bulk_f32_m<512>(H, x, nrows, L, lay, tw, twf, f, s);
        case 1024: return c2r_bulk_f32_m<1024>(H, x, nrows, L, lay, tw, twf, f, s);
        case 2048: return c2r_bulk_f32_m<2048>(H, x, nrows, L, lay, tw, twf, f, s);
        case 4096: return c2r_bulk_f32_m<4096>(H, x, nrows, L, lay, tw, twf, f, s);
        default: return cudaErrorInvalidValue;
    }
}

cudaError_t launch_cols_pipe(double2* H, const AxisGeom& g, int mode, const FusedSymbol& sym, const double2* tw,
                             cudaStream_t s) {
#define FSX_COLS(N)                                                          \
    case N:                                                                  \
        return mode == 0 ? cols_pipe_n<N, 0>(H, g, sym, tw, s)               \
             : mode == 1 ? cols_pipe_n<N, 1>(H, g, sym, tw, s)               \
                         : cols_pipe_n<N, 2>(H, g, sym, tw, s);
    switch (g.n) {
        FSX_COLS(1024)
        FSX_COLS(2048)
        FSX_COLS(4096)
        default: return cudaErrorInvalidValue;
    }
#undef FSX_COLS
}

}  // namespace fsx
