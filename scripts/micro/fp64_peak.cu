// FP64 FMA throughput of this B200 (the denominator of the fused passes'
// fp64 roofline): every thread runs 8 independent DFMA chains.
// nvcc -O3 -gencode arch=compute_100a,code=sm_100a fp64_peak.cu -o fp64_peak
#include <cstdio>
#include <cuda_runtime.h>

__global__ void k_dfma(double* out, int iters, double a, double b) {
    double x[8];
#pragma unroll
    for (int i = 0; i < 8; ++i) x[i] = threadIdx.x * 1e-9 + i;
    for (int it = 0; it < iters; ++it) {
#pragma unroll
        for (int i = 0; i < 8; ++i) x[i] = fma(x[i], a, b);
    }
    double s = 0;
#pragma unroll
    for (int i = 0; i < 8; ++i) s += x[i];
    if (s == 12345.678) out[threadIdx.x] = s;  // keep the chains alive
}

int main() {
    int dev = 0, sms = 0;
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    double* out;
    cudaMalloc(&out, 1024 * sizeof(double));
    const int blocks = sms * 8, threads = 256, iters = 4096;
    k_dfma<<<blocks, threads>>>(out, iters, 0.999999, 1e-7);
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0);
    cudaEventCreate(&e1);
    float best = 1e30f;
    for (int r = 0; r < 10; ++r) {
        cudaEventRecord(e0);
        k_dfma<<<blocks, threads>>>(out, iters, 0.999999, 1e-7);
        cudaEventRecord(e1);
        cudaEventSynchronize(e1);
        float ms;
        cudaEventElapsedTime(&ms, e0, e1);
        if (ms < best) best = ms;
    }
    const double flops = 2.0 * 8 * (double)iters * blocks * threads;
    printf("{\"fp64_fma_tflops\": %.2f, \"ms\": %.4f, \"sms\": %d, \"how\": \"8 independent DFMA chains per thread, %d blocks x %d threads x %d iters, best of 10, CUDA events\"}\n",
           flops / (best * 1e-3) / 1e12, best, sms, blocks, threads, iters);
    return 0;
}
