// Micro-benchmark: the I/O skeleton of the 8192-point fused column pass on a
// cfg3-shaped half spectrum [8192][4104] complex fp64 (load a column tile by
// TMA, touch it, store it back), comparing
//   A  one column per CTA pair, 16-byte box rows (the shipped k_fused8192c
//      layout: 64 KB parity half per CTA, 2 CTAs/SM);
//   B  two adjacent columns per 4-CTA cluster, 32-byte box rows: CTA (j, h)
//      loads half of the rows of BOTH columns (64 KB), then swaps 32 KB with
//      CTA (1 - j, h) over DSMEM (st.async, receiver-side mbarrier) so it holds
//      one column's rows, and the reverse before its 32-byte-row store;
//   A2 as A with half the rows read by the threads (LDG.128) instead of TMA;
//   C  two adjacent columns per CTA, 32-byte rows, 128 KB tile (1 CTA/SM).
// Measured (B200): A 304 us (3.5 TB/s), A2 354 us, B 336 us, C 236 us (4.6 TB/s).
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -I../../paper_2105_06676_b200/csrc tma_cluster.cu -o tma_cluster
#include <cuda.h>
#include <cuda_runtime.h>

#include <cstdio>

#include "fsx_async.cuh"

namespace fsx {
bool pdl_enabled() { return false; }
}
using namespace fsx;

__device__ __forceinline__ unsigned cl_rank() {
    unsigned r;
    asm volatile("mov.u32 %0, %%cluster_ctarank;\n" : "=r"(r));
    return r;
}
__device__ __forceinline__ unsigned peer_addr(const void* local, unsigned rank) {
    unsigned out;
    asm volatile("mapa.shared::cluster.u32 %0, %1, %2;\n" : "=r"(out) : "r"(smem_u32(local)), "r"(rank));
    return out;
}
__device__ __forceinline__ void st_async(unsigned addr, double2 v, unsigned bar) {
    asm volatile("st.async.shared::cluster.mbarrier::complete_tx::bytes.v2.f64 [%0], {%1, %2}, [%3];\n" ::"r"(addr),
                 "d"(v.x), "d"(v.y), "r"(bar)
                 : "memory");
}
__device__ __forceinline__ void cl_arrive() { asm volatile("barrier.cluster.arrive.relaxed.aligned;\n" ::: "memory"); }
__device__ __forceinline__ void cl_wait() { asm volatile("barrier.cluster.wait.acquire.aligned;\n" ::: "memory"); }

// A: CTA = (column, row half); box {2 doubles, 256 rows}
__global__ void __launch_bounds__(256, 2) k_a(const __grid_constant__ CUtensorMap map, int ncols) {
    extern __shared__ __align__(128) double2 tile[];
    __shared__ __align__(8) unsigned long long bar;
    const int c = blockIdx.x % ncols, h = blockIdx.x / ncols;
    if (threadIdx.x == 0) {
        mbar_init(&bar, 1);
        mbar_init_fence();
        mbar_expect_tx(&bar, 4096 * 16);
        for (int b = 0; b < 16; ++b) tma_load_3d(tile + b * 256, &map, 2 * c, h * 4096 + b * 256, 0, &bar);
    }
    __syncthreads();
    mbar_wait(&bar, 0);
    for (int i = threadIdx.x; i < 4096; i += 256) {
        double2 v = tile[i];
        v.x += 1.0;
        tile[i] = v;
    }
    fence_proxy_async();
    __syncthreads();
    if (threadIdx.x == 0) {
        for (int b = 0; b < 16; ++b) tma_store_3d(&map, tile + b * 256, 2 * c, h * 4096 + b * 256, 0);
        bulk_commit();
        bulk_wait_read0();
    }
}

// B: cluster of 4 = (row half h) x (quarter j); CTA (h, j) loads rows
// [h 4096 + j 2048, +2048) of columns c, c+1 as 32-byte rows (64 KB), keeps
// column c+j, sends column c+1-j's 32 KB to CTA (h, 1-j), receives the other
// 2048 rows of column c+j; touches its 4096 rows; reverse; 32-byte-row store.
__global__ void __cluster_dims__(4, 1, 1) __launch_bounds__(256, 2) k_b(const __grid_constant__ CUtensorMap map2) {
    extern __shared__ __align__(128) double2 sm[];
    double2* tile = sm;          // [2048 rows][2 cols] as loaded
    double2* land = sm + 4096;   // [2048] the partner's rows of my column
    __shared__ __align__(8) unsigned long long bar, bx, bx2, bok;
    const unsigned r = cl_rank(), h = r >> 1, j = r & 1, partner = r ^ 1u;
    const int c = (blockIdx.x >> 2) * 2;
    const int row0 = (int)(h * 4096 + j * 2048);
    const int t = threadIdx.x;
    if (t == 0) {
        mbar_init(&bar, 1);
        mbar_init(&bx, 1);
        mbar_init(&bx2, 1);
        mbar_init(&bok, 1);
        mbar_init_fence();
        mbar_expect_tx(&bx, 2048 * 16);
        mbar_expect_tx(&bx2, 2048 * 16);
        mbar_expect_tx(&bar, 4096 * 16);
        for (int b = 0; b < 8; ++b) tma_load_3d(tile + b * 512, &map2, 2 * c, row0 + b * 256, 0, &bar);
    }
    cl_arrive();
    cl_wait();
    mbar_wait(&bar, 0);
    // send the other column's 2048 rows to the partner's landing zone
    {
        const unsigned dst = peer_addr(land, partner), pb = peer_addr(&bx, partner);
        for (int i = t; i < 2048; i += 256) st_async(dst + 16u * i, tile[2 * i + (1 - j)], pb);
    }
    double2 v[16];
    for (int q = 0; q < 8; ++q) v[q] = tile[2 * (t + 256 * q) + j];
    mbar_wait(&bx, 0);
    for (int q = 0; q < 8; ++q) v[8 + q] = land[t + 256 * q];
    for (int q = 0; q < 16; ++q) v[q].x += 1.0;
    __syncthreads();  // tile and land reads done
    if (t == 0) asm volatile("mbarrier.arrive.release.cluster.shared::cluster.b64 _, [%0];\n" ::"r"(peer_addr(&bok, partner)) : "memory");
    // reverse: my column's rows of the partner's range go back into the partner's tile
    {
        asm volatile(
            "{\n.reg .pred P1;\nW_%=:\nmbarrier.try_wait.parity.acquire.cluster.shared::cta.b64 P1, [%0], 0;\n@!P1 bra W_%=;\n}\n" ::"r"(
                smem_u32(&bok))
            : "memory");
        const unsigned dst = peer_addr(tile, partner), pb = peer_addr(&bx2, partner);
        for (int q = 0; q < 8; ++q) st_async(dst + 16u * (2 * (t + 256 * q) + j), v[8 + q], pb);
    }
    for (int q = 0; q < 8; ++q) tile[2 * (t + 256 * q) + j] = v[q];
    mbar_wait(&bx2, 0);
    fence_proxy_async();
    __syncthreads();
    if (t == 0) {
        for (int b = 0; b < 8; ++b) tma_store_3d(&map2, tile + b * 512, 2 * c, row0 + b * 256, 0);
        bulk_commit();
        bulk_wait_read0();
    }
}

// A2: as A, but only the first half of the rows by TMA; the second half is
// read by the threads themselves (LDG.128, one 16-byte element each, the
// values a thread would own in registers): does a second path raise the
// 16-byte-row request rate?
__global__ void __launch_bounds__(256, 2) k_a2(const __grid_constant__ CUtensorMap map, const double2* __restrict__ H,
                                               int ncols, long long P) {
    extern __shared__ __align__(128) double2 tile[];
    __shared__ __align__(8) unsigned long long bar;
    const int c = blockIdx.x % ncols, h = blockIdx.x / ncols;
    if (threadIdx.x == 0) {
        mbar_init(&bar, 1);
        mbar_init_fence();
        mbar_expect_tx(&bar, 2048 * 16);
        for (int b = 0; b < 8; ++b) tma_load_3d(tile + b * 256, &map, 2 * c, h * 4096 + b * 256, 0, &bar);
    }
    double2 v[8];
#pragma unroll
    for (int q = 0; q < 8; ++q) v[q] = __ldg(H + (long long)(h * 4096 + 2048 + threadIdx.x + 256 * q) * P + c);
    __syncthreads();
    mbar_wait(&bar, 0);
#pragma unroll
    for (int q = 0; q < 8; ++q) {
        v[q].x += 1.0;
        tile[2048 + threadIdx.x + 256 * q] = v[q];
    }
    for (int i = threadIdx.x; i < 2048; i += 256) {
        double2 u = tile[i];
        u.x += 1.0;
        tile[i] = u;
    }
    fence_proxy_async();
    __syncthreads();
    if (threadIdx.x == 0) {
        for (int b = 0; b < 16; ++b) tma_store_3d(&map, tile + b * 256, 2 * c, h * 4096 + b * 256, 0);
        bulk_commit();
        bulk_wait_read0();
    }
}

// C: two columns x 4096 rows per CTA (128 KB), 32-byte rows
__global__ void __launch_bounds__(512, 1) k_c(const __grid_constant__ CUtensorMap map2, int npair) {
    extern __shared__ __align__(128) double2 tile[];
    __shared__ __align__(8) unsigned long long bar;
    const int c = (blockIdx.x % npair) * 2, h = blockIdx.x / npair;
    if (threadIdx.x == 0) {
        mbar_init(&bar, 1);
        mbar_init_fence();
        mbar_expect_tx(&bar, 8192 * 16);
        for (int b = 0; b < 16; ++b) tma_load_3d(tile + b * 512, &map2, 2 * c, h * 4096 + b * 256, 0, &bar);
    }
    __syncthreads();
    mbar_wait(&bar, 0);
    for (int i = threadIdx.x; i < 8192; i += 512) {
        double2 v = tile[i];
        v.x += 1.0;
        tile[i] = v;
    }
    fence_proxy_async();
    __syncthreads();
    if (threadIdx.x == 0) {
        for (int b = 0; b < 16; ++b) tma_store_3d(&map2, tile + b * 512, 2 * c, h * 4096 + b * 256, 0);
        bulk_commit();
        bulk_wait_read0();
    }
}

typedef CUresult (*EncodeTiledFn)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*, const cuuint64_t*,
                                  const cuuint64_t*, const cuuint32_t*, const cuuint32_t*, CUtensorMapInterleave,
                                  CUtensorMapSwizzle, CUtensorMapL2promotion, CUtensorMapFloatOOBfill);

static EncodeTiledFn enc() {
    void* fn = nullptr;
    cudaDriverEntryPointQueryResult q;
    cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &fn, cudaEnableDefault, &q);
    return (EncodeTiledFn)fn;
}

static CUtensorMap make(double2* H, int rows, int P, int W) {
    CUtensorMap map;
    const cuuint64_t dims[3] = {(cuuint64_t)(2 * P), (cuuint64_t)rows, 1};
    const cuuint64_t strides[2] = {(cuuint64_t)(P * 16), (cuuint64_t)((size_t)rows * P * 16)};
    const cuuint32_t box[3] = {(cuuint32_t)(2 * W), 256, 1};
    const cuuint32_t estr[3] = {1, 1, 1};
    CUresult r = enc()(&map, CU_TENSOR_MAP_DATA_TYPE_FLOAT64, 3, H, dims, strides, box, estr, CU_TENSOR_MAP_INTERLEAVE_NONE,
                       CU_TENSOR_MAP_SWIZZLE_NONE, CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    if (r != CUDA_SUCCESS) printf("encode failed %d\n", (int)r);
    return map;
}

template <class F>
static void timeit(const char* name, F&& launch, double bytes) {
    cudaEvent_t a, b;
    cudaEventCreate(&a);
    cudaEventCreate(&b);
    for (int i = 0; i < 3; ++i) launch();
    cudaEventRecord(a);
    const int it = 10;
    for (int i = 0; i < it; ++i) launch();
    cudaEventRecord(b);
    cudaEventSynchronize(b);
    float ms = 0;
    cudaEventElapsedTime(&ms, a, b);
    ms /= it;
    printf("%-52s %8.1f us  %6.0f GB/s  %s\n", name, ms * 1e3, bytes / (ms * 1e-3) / 1e9,
           cudaGetErrorString(cudaGetLastError()));
}

int main() {
    const int rows = 8192, P = 4104, ncols = 4096;  // cfg3: 4097 columns used, pitch 4104
    double2* H;
    cudaMalloc(&H, (size_t)rows * P * 16);
    cudaMemset(H, 0, (size_t)rows * P * 16);
    const double bytes = 2.0 * rows * (double)ncols * 16;
    const CUtensorMap m1 = make(H, rows, P, 1), m2 = make(H, rows, P, 2);
    const size_t sa = 96 * 1024;  // the shipped kernel's 64 KB tile + 32 KB exchange landing (2 CTAs/SM)
    cudaFuncSetAttribute(k_a, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sa);
    timeit("A  16 B rows, 64 KB tile/CTA, 2 CTAs/SM", [&] { k_a<<<2 * ncols, 256, sa>>>(m1, ncols); }, bytes);
    cudaFuncSetAttribute(k_a2, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sa);
    timeit("A2 16 B rows, half TMA / half per-thread LDG", [&] { k_a2<<<2 * ncols, 256, sa>>>(m1, H, ncols, P); }, bytes);
    const size_t sb = 96 * 1024;
    cudaFuncSetAttribute(k_b, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sb);
    timeit("B  32 B rows, 4-CTA cluster + 2 DSMEM swaps", [&] { k_b<<<2 * ncols, 256, sb>>>(m2); }, bytes);
    const size_t sc = 128 * 1024;
    cudaFuncSetAttribute(k_c, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sc);
    timeit("C  32 B rows, 128 KB tile/CTA, 1 CTA/SM", [&] { k_c<<<ncols, 512, sc>>>(m2, ncols / 2); }, bytes);
    return 0;
}
