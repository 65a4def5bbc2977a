// Where do the two CTAs of a 2-CTA cluster land?  Launches the cfg3 fused
// pass's geometry (8194 CTAs of 256 threads, 98 KB of shared memory each, two
// per SM by occupancy) and records each CTA's SM: the fraction of pairs that
// share an SM tells whether an SM's two CTAs are the two (lock-stepped)
// halves of one column or halves of two different columns.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 cluster_place.cu -o cluster_place
#include <cuda_runtime.h>

#include <cstdio>
#include <vector>

__global__ void __cluster_dims__(2, 1, 1) __launch_bounds__(256, 2) k_place(int* smid, long long* t0) {
    extern __shared__ double sm[];
    unsigned s;
    asm volatile("mov.u32 %0, %%smid;" : "=r"(s));
    long long c = clock64();
    // hold the SM a while (like a column's FFT work)
    double x = threadIdx.x;
    for (int i = 0; i < 20000; ++i) x = x * 1.0000001 + 1e-9;
    sm[threadIdx.x] = x;
    __syncthreads();
    if (threadIdx.x == 0) {
        smid[blockIdx.x] = (int)s + (sm[0] > 1e300 ? 1 : 0);
        t0[blockIdx.x] = c;
    }
}

static void run(int policy, const char* name) {
    const int n = 8194;
    int* d;
    long long* t;
    cudaMalloc(&d, n * sizeof(int));
    cudaMalloc(&t, n * sizeof(long long));
    const size_t smem = (4096 + 2048) * 16;
    cudaFuncSetAttribute(k_place, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = dim3(n);
    cfg.blockDim = dim3(256);
    cfg.dynamicSmemBytes = smem;
    cudaLaunchAttribute attr[1];
    attr[0].id = cudaLaunchAttributeClusterSchedulingPolicyPreference;
    attr[0].val.clusterSchedulingPolicyPreference =
        policy == 1 ? cudaClusterSchedulingPolicySpread : cudaClusterSchedulingPolicyLoadBalancing;
    cfg.attrs = attr;
    cfg.numAttrs = policy ? 1 : 0;
    cudaLaunchKernelEx(&cfg, k_place, d, t);
    cudaError_t e = cudaDeviceSynchronize();
    std::vector<int> h(n);
    cudaMemcpy(h.data(), d, n * sizeof(int), cudaMemcpyDeviceToHost);
    int same = 0;
    for (int i = 0; i < n; i += 2) same += h[i] == h[i + 1];
    printf("%-16s %s: %d of %d pairs on one SM (%.1f %%)\n", name, cudaGetErrorString(e), same, n / 2,
           100.0 * same / (n / 2));
    cudaFree(d);
    cudaFree(t);
}

int main() {
    run(0, "default");
    run(1, "spread");
    run(2, "load balancing");
    return 0;
}
