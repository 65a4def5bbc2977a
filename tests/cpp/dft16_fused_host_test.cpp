// Host-side check of the radix-16 butterfly with folded pass twiddles
// (fsx_device.cuh, dft16_tw_fused) against the direct sum
//   X[k] = sum_u a[u] w^u exp(SIGN 2 pi i u k / 16)
// in long double, and against the unfused path (twiddle products + Dft<16>).
// Compiled with plain g++: outside nvcc __device__ expands to nothing, and the
// few device intrinsics the header names are stubbed below (never called).
#include <cmath>
#include <complex>
#include <cstdio>
#include <cstdlib>
#include <cuda_runtime.h>

struct FakeIdx { unsigned x = 0, y = 0, z = 0; };
static FakeIdx threadIdx;
static inline void __syncthreads() {}
template <class T>
static inline T __ldg(const T* p) { return *p; }

#include "fsx_device.cuh"

using fsx::dft16_tw_fused;
typedef std::complex<long double> cld;

template <int SIGN, class CT>
static double run_case(unsigned seed, double* vs_unfused) {
    using T = typename fsx::CScalar<CT>::T;
    srand(seed);
    auto rnd = [] { return (double)rand() / RAND_MAX * 2.0 - 1.0; };
    CT a[16], b[16];
    cld x[16];
    for (int u = 0; u < 16; ++u) {
        a[u] = fsx::CScalar<CT>::make((T)rnd(), (T)rnd());
        b[u] = a[u];
        x[u] = cld(a[u].x, a[u].y);
    }
    const long double th = -2.0L * M_PIl * (long double)rnd();  // table value w = exp(i th)
    CT w[16];
    for (int u = 0; u < 16; ++u) w[u] = fsx::CScalar<CT>::make((T)cosl(u * th), (T)sinl(u * th));
    dft16_tw_fused<SIGN>(a, w[1], w[2], w[4], w[8]);
    for (int u = 1; u < 16; ++u) b[u] = fsx::ctw<SIGN>(b[u], w[u]);
    fsx::Dft<16, SIGN>::run(b);
    long double err = 0, nrm = 0, e2 = 0;
    for (int k = 0; k < 16; ++k) {
        cld s = 0;
        for (int u = 0; u < 16; ++u) {
            const long double ang = (SIGN < 0 ? 1.0L : -1.0L) * u * th + SIGN * 2.0L * M_PIl * u * k / 16.0L;
            s += x[u] * cld(cosl(ang), sinl(ang));
        }
        err += std::norm(s - cld(a[k].x, a[k].y));
        e2 += std::norm(cld(b[k].x, b[k].y) - cld(a[k].x, a[k].y));
        nrm += std::norm(s);
    }
    *vs_unfused = (double)sqrtl(e2 / nrm);
    return (double)sqrtl(err / nrm);
}

int main() {
    double worst64 = 0, worst32 = 0, wu64 = 0, wu32 = 0, u;
    for (unsigned s = 1; s <= 200; ++s) {
        worst64 = fmax(worst64, run_case<-1, double2>(s, &u)); wu64 = fmax(wu64, u);
        worst64 = fmax(worst64, run_case<+1, double2>(s + 1000, &u)); wu64 = fmax(wu64, u);
        worst32 = fmax(worst32, run_case<-1, float2>(s, &u)); wu32 = fmax(wu32, u);
        worst32 = fmax(worst32, run_case<+1, float2>(s + 1000, &u)); wu32 = fmax(wu32, u);
    }
    printf("dft16_tw_fused: worst rel L2 vs direct sum fp64 %.3e fp32 %.3e; vs unfused fp64 %.3e fp32 %.3e\n", worst64,
           worst32, wu64, wu32);
    const bool ok = worst64 < 2e-15 && worst32 < 1e-6 && wu64 < 2e-15 && wu32 < 1e-6;
    printf(ok ? "OK\n" : "FAIL\n");
    return ok ? 0 : 1;
}
