// Microbenchmark (scratch, not product): compute-only throughput of the
// LineFFT<4096> engine -- forward + inverse on a register tile, no global
// memory traffic in the loop -- to separate FFT arithmetic efficiency from
// memory overlap in the fused pass.
#include <cstdio>
#include <vector>
#include "../../paper_2105_06676_b200/csrc/fsx_device.cuh"
using namespace fsx;

template <int MINB>
__global__ void __launch_bounds__(256, MINB) k_fft_loop(double2* out, const double2* tw_all, int iters) {
    extern __shared__ double2 sm[];
    const int t = threadIdx.x;
    double2 v[16];
#pragma unroll
    for (int q = 0; q < 16; ++q) v[q] = make_double2(t * 1e-3 + q, blockIdx.x * 1e-4 - q);
    for (int it = 0; it < iters; ++it) {
        LineFFT<4096, -1>::run(v, t, sm, tw_all + 4096);
#pragma unroll
        for (int q = 0; q < 16; ++q) v[q] = cscale(v[q], 1.0 / 4096);
        LineFFT<4096, +1>::run(v, t, sm, tw_all + 4096);
    }
    double2 acc = make_double2(0, 0);
#pragma unroll
    for (int q = 0; q < 16; ++q) acc = cadd(acc, v[q]);
    out[blockIdx.x * 256 + t] = acc;
}

int main() {
    std::vector<double2> tw(2 * 32768);
    for (long N = 1; N <= 32768; N <<= 1)
        for (long x = 0; x < N; ++x) tw[N + x] = make_double2(cos(-2 * M_PI * x / N), sin(-2 * M_PI * x / N));
    double2 *dtw, *dout;
    cudaMalloc(&dtw, tw.size() * 16);
    cudaMemcpy(dtw, tw.data(), tw.size() * 16, cudaMemcpyHostToDevice);
    const int ctas = 2049, iters = 8;
    cudaMalloc(&dout, (size_t)ctas * 256 * 16);
    cudaEvent_t a, b;
    cudaEventCreate(&a);
    cudaEventCreate(&b);
    for (int minb = 1; minb <= 2; ++minb) {
        auto k = minb == 1 ? k_fft_loop<1> : k_fft_loop<2>;
        cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, 65536);
        k<<<ctas, 256, 65536>>>(dout, dtw, iters);
        cudaEventRecord(a);
        k<<<ctas, 256, 65536>>>(dout, dtw, iters);
        cudaEventRecord(b);
        cudaEventSynchronize(b);
        float ms;
        cudaEventElapsedTime(&ms, a, b);
        const double per = ms * 1e3 / iters;  // us per (2049 columns x fwd+inv)
        printf("MINB=%d: %.1f us per 2049-column fwd+inv pair (fused pass compute share), err=%s\n", minb, per,
               cudaGetErrorString(cudaGetLastError()));
    }
    return 0;
}
