// Micro-benchmark: TMA column-tile copy (load box -> smem -> store box, in
// place) over a cfg2-shaped half spectrum [4096][2056] complex fp64, as a
// function of the bytes per box row (16 B * W adjacent columns) and the
// tile size.  Measures whether the column passes are bound by TMA row
// requests rather than HBM bytes.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -I../../paper_2105_06676_b200/csrc tma_rows.cu -lcuda -o tma_rows
#include <cuda.h>
#include <cuda_runtime.h>

#include <cstdio>
#include <vector>

#include "fsx_async.cuh"

namespace fsx {
bool pdl_enabled() { return false; }
}
using namespace fsx;

template <int W, int ROWS>
__global__ void k_copy(const __grid_constant__ CUtensorMap map, int ctiles) {
    extern __shared__ __align__(128) double2 tile[];
    __shared__ __align__(8) unsigned long long bar;
    constexpr int BOX = 256;
    const int c0 = (blockIdx.x % ctiles) * W;
    const int r0 = (blockIdx.x / ctiles) * ROWS;
    if (threadIdx.x == 0) {
        mbar_init(&bar, 1);
        mbar_init_fence();
        mbar_expect_tx(&bar, ROWS * W * 16);
        for (int b = 0; b < ROWS / BOX; ++b) tma_load_3d(tile + b * BOX * W, &map, 2 * c0, r0 + b * BOX, 0, &bar);
    }
    __syncthreads();
    mbar_wait(&bar, 0);
    // touch the tile (one pass of smem reads/writes like the FFT's first load)
    for (int i = threadIdx.x; i < ROWS * W; i += blockDim.x) {
        double2 v = tile[i];
        v.x += 1.0;
        tile[i] = v;
    }
    fence_proxy_async();
    __syncthreads();
    if (threadIdx.x == 0) {
        for (int b = 0; b < ROWS / BOX; ++b) tma_store_3d(&map, tile + b * BOX * W, 2 * c0, r0 + b * BOX, 0);
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

template <int W, int ROWS>
static void run(double2* H, int rows, int P, int ncols, int threads) {
    CUtensorMap map;
    const cuuint64_t dims[3] = {(cuuint64_t)(2 * P), (cuuint64_t)rows, 1};
    const cuuint64_t strides[2] = {(cuuint64_t)(P * 16), (cuuint64_t)((size_t)rows * P * 16)};
    const cuuint32_t box[3] = {(cuuint32_t)(2 * W), 256, 1};
    const cuuint32_t estr[3] = {1, 1, 1};
    CUresult r = enc()(&map, CU_TENSOR_MAP_DATA_TYPE_FLOAT64, 3, H, dims, strides, box, estr, CU_TENSOR_MAP_INTERLEAVE_NONE,
                       CU_TENSOR_MAP_SWIZZLE_NONE, CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    if (r != CUDA_SUCCESS) {
        printf("encode failed %d\n", (int)r);
        return;
    }
    const int ctiles = ncols / W;
    const int grid = ctiles * (rows / ROWS);
    const size_t smem = (size_t)ROWS * W * 16;
    cudaFuncSetAttribute(k_copy<W, ROWS>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    int occ = 0;
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, k_copy<W, ROWS>, threads, smem);
    cudaEvent_t a, b;
    cudaEventCreate(&a);
    cudaEventCreate(&b);
    for (int i = 0; i < 3; ++i) k_copy<W, ROWS><<<grid, threads, smem>>>(map, ctiles);
    cudaEventRecord(a);
    const int it = 10;
    for (int i = 0; i < it; ++i) k_copy<W, ROWS><<<grid, threads, smem>>>(map, ctiles);
    cudaEventRecord(b);
    cudaEventSynchronize(b);
    float ms = 0;
    cudaEventElapsedTime(&ms, a, b);
    ms /= it;
    const double bytes = 2.0 * rows * (double)ncols * 16;
    printf("W=%d (%3d B rows) ROWS=%4d tile=%6zu B CTAs/SM=%d  %.1f us  %.0f GB/s  err=%s\n", W, W * 16, ROWS, smem, occ,
           ms * 1e3, bytes / (ms * 1e-3) / 1e9, cudaGetErrorString(cudaGetLastError()));
}

int main() {
    const int rows = 4096, P = 2056, ncols = 2048;
    double2* H;
    cudaMalloc(&H, (size_t)rows * P * 16);
    cudaMemset(H, 0, (size_t)rows * P * 16);
    run<1, 4096>(H, rows, P, ncols, 256);
    run<1, 2048>(H, rows, P, ncols, 256);
    run<1, 1024>(H, rows, P, ncols, 128);
    run<2, 2048>(H, rows, P, ncols, 256);
    run<2, 1024>(H, rows, P, ncols, 256);
    run<4, 1024>(H, rows, P, ncols, 256);
    run<4, 512>(H, rows, P, ncols, 256);
    run<8, 512>(H, rows, P, ncols, 256);
    run<8, 256>(H, rows, P, ncols, 256);
    run<16, 256>(H, rows, P, ncols, 256);
    run<32, 256>(H, rows, P, ncols, 256);
    return 0;
}
