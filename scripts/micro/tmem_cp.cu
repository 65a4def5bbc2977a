// Self-test of the tensor-memory staging used by the persistent fused column
// pass: a 2 KB shared-memory block of 128 x 16-byte elements is copied into
// TMEM with tcgen05.cp.128x128b (no-swizzle K-major descriptor, 8-row core
// matrices 128 B apart) and read back with tcgen05.ld.32x32b; element i must
// land in lane i, columns [c, c + 4).  Also times a 64 KB fill + read.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -I../../paper_2105_06676_b200/csrc tmem_cp.cu -o tmem_cp
#include <cuda_runtime.h>

#include <cstdio>

#include "fsx_async.cuh"

namespace fsx {
bool pdl_enabled() { return false; }
}
using namespace fsx;

__device__ __forceinline__ unsigned long long cp_desc(const void* smem) {
    const unsigned a = smem_u32(smem);
    unsigned long long d = 0;
    d |= (unsigned long long)((a >> 4) & 0x3FFF);          // start address
    d |= (unsigned long long)(1) << 16;                     // leading byte offset (unused: one 16-B column)
    d |= (unsigned long long)(128 >> 4) << 32;              // stride byte offset: 8-row core matrices 128 B apart
    d |= (unsigned long long)1 << 46;                       // version (sm_100)
    return d;                                               // base offset 0, lbo mode 0, layout SWIZZLE_NONE (0)
}

__global__ void k_test(double2* out, int* ok) {
    extern __shared__ __align__(1024) double2 buf[];  // 64 KB (128 x 32 elements)
    __shared__ unsigned tbase;
    __shared__ __align__(8) unsigned long long cbar;
    const int t = threadIdx.x;  // 128 threads
    for (int i = t; i < 128 * 32; i += 128) buf[i] = make_double2(1000.0 * i + 0.25, -(double)i - 0.5);
    if (t < 32) {
        asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 128;\n" ::"r"(smem_u32(&tbase)));
        asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;\n");
    }
    if (t == 0) {
        mbar_init(&cbar, 1);
        mbar_init_fence();
    }
    asm volatile("fence.proxy.async.shared::cta;\n" ::: "memory");  // generic smem writes visible to the async proxy
    asm volatile("tcgen05.fence::before_thread_sync;\n" ::: "memory");
    __syncthreads();
    asm volatile("tcgen05.fence::after_thread_sync;\n" ::: "memory");
    const unsigned tb = tbase;
    long long t0 = clock64();
    if (t == 0) {
        // block b (elements 128 b .. 128 b + 127) -> columns 4 b .. 4 b + 3
        for (int b = 0; b < 32; ++b) {
            const unsigned long long d = cp_desc(buf + 128 * b);
            asm volatile("tcgen05.cp.cta_group::1.128x128b [%0], %1;\n" ::"r"(tb + 4u * b), "l"(d) : "memory");
        }
        asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];\n" ::"r"(smem_u32(&cbar))
                     : "memory");
    }
    mbar_wait(&cbar, 0);
    asm volatile("tcgen05.fence::after_thread_sync;\n" ::: "memory");
    long long t1 = clock64();
    // warp w reads lanes 32 w .. 32 w + 31: thread t = lane t, all 128 columns (32 elements)
    unsigned r[64];
    for (int half = 0; half < 2; ++half) {
        const unsigned addr = tb + ((unsigned)(32 * (t / 32)) << 16) + 64u * half;
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
            : "r"(addr));
        asm volatile("tcgen05.wait::ld.sync.aligned;\n" ::: "memory");
        for (int j = 0; j < 16; ++j) {
            const int b = 16 * half + j;
            double2 v;
            v.x = __hiloint2double((int)r[4 * j + 1], (int)r[4 * j]);
            v.y = __hiloint2double((int)r[4 * j + 3], (int)r[4 * j + 2]);
            out[t * 32 + b] = v;
            const double2 want = buf[128 * b + t];
            if (v.x != want.x || v.y != want.y) atomicAdd(ok, 1);
        }
    }
    long long t2 = clock64();
    if (t == 0) printf("cp 64 KB: %lld clk, ld 64 KB (2 x x64 per thread): %lld clk\n", t1 - t0, t2 - t1);
    asm volatile("tcgen05.fence::before_thread_sync;\n" ::: "memory");
    __syncthreads();
    if (t < 32) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 128;\n" ::"r"(tb));
}

int main() {
    double2* out;
    int* bad;
    cudaMalloc(&out, 128 * 32 * sizeof(double2));
    cudaMalloc(&bad, 4);
    cudaMemset(bad, 0, 4);
    cudaFuncSetAttribute(k_test, cudaFuncAttributeMaxDynamicSharedMemorySize, 65536);
    k_test<<<1, 128, 65536>>>(out, bad);
    cudaError_t e = cudaDeviceSynchronize();
    int h = -1;
    cudaMemcpy(&h, bad, 4, cudaMemcpyDeviceToHost);
    printf("tmem_cp: %s, mismatches %d\n", cudaGetErrorString(e), h);
    return (e == cudaSuccess && h == 0) ? 0 : 1;
}
