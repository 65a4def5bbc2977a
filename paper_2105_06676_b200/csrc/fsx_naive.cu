// Direct periodic stencil stepping on the GPU: the reference's naive oracle
// (proj/src/oracle.cpp:26-115, step_periodic / evolve_periodic_naive)
// restated as a verifier kernel.  It is NOT on the solve path; it gives an
// independent full-size check of the FFT solver
// where the CPU loop (N * T * taps) is infeasible.
//
// Arithmetic follows the reference loop exactly so results are bitwise
// identical to it: per output cell the taps are visited in sorted-offset
// order; scalar grids accumulate out = out + c * a[x + off] (oracle.cpp:52-53,
// starting from 0, no FMA contraction: the reference is built without
// -march, so x86-64 SSE2 rounds the product and the sum separately); vector
// grids form acc = sum_g B(f,g) a[g] per tap and add it (oracle.cpp:76-80).
//
// Layout: one thread per cell of the last axis (x), grid y / z over the two
// preceding axes (rank <= 3); ranks 4..8 decode the cell index with divisions.
#include "fsx_kernels.h"

namespace fsx {

template <int MFIX>
__global__ void k_step_naive(const double* __restrict__ a, double* __restrict__ out, NaiveGeom g,
                             const long long* __restrict__ off, const double* __restrict__ blk) {
    const int m = MFIX > 0 ? MFIX : g.m;
    i64 idx[kMaxRank];
    i64 cell;
    if (g.rank <= 3) {
        const i64 x = (i64)blockIdx.x * blockDim.x + threadIdx.x;
        if (x >= g.n[2]) return;
        idx[0] = blockIdx.z;
        idx[1] = blockIdx.y;
        idx[2] = x;
        cell = (idx[0] * g.n[1] + idx[1]) * g.n[2] + x;
    } else {
        cell = (i64)blockIdx.x * blockDim.x + threadIdx.x;
        if (cell >= g.cells) return;
        i64 r = cell;
        for (int ax = g.rank - 1; ax >= 0; --ax) {
            idx[ax] = r % g.n[ax];
            r /= g.n[ax];
        }
    }
    const int ra = g.rank <= 3 ? 3 : g.rank;  // axes of idx / n in use
    double acc_out[MFIX > 0 ? MFIX : kMaxNaiveFields];
    for (int f = 0; f < m; ++f) acc_out[f] = 0.0;
    for (int j = 0; j < g.ntaps; ++j) {
        i64 sc = 0;
        for (int ax = 0; ax < ra; ++ax) {
            // tap offsets are stored padded to 3 axes for rank <= 3 (leading zeros)
            i64 s = idx[ax] + off[j * ra + ax];
            if (s >= g.n[ax]) s -= g.n[ax];
            else if (s < 0) s += g.n[ax];
            sc = sc * g.n[ax] + s;
        }
        const double* b = blk + (i64)j * m * m;
        if (m == 1) {
            acc_out[0] = __dadd_rn(acc_out[0], __dmul_rn(b[0], a[sc]));
        } else {
            for (int f = 0; f < m; ++f) {
                double acc = 0.0;
                for (int q = 0; q < m; ++q) acc = __dadd_rn(acc, __dmul_rn(b[f * m + q], a[sc * m + q]));
                acc_out[f] = __dadd_rn(acc_out[f], acc);
            }
        }
    }
    for (int f = 0; f < m; ++f) out[cell * m + f] = acc_out[f];
}

cudaError_t launch_step_naive(const double* a, double* out, const NaiveGeom& g, const long long* off,
                              const double* blk, cudaStream_t s) {
    if (g.m < 1 || g.m > kMaxNaiveFields) return cudaErrorInvalidValue;
    const int threads = 256;
    dim3 grid;
    if (g.rank <= 3) {
        if (g.n[0] > 65535 || g.n[1] > 65535) return cudaErrorInvalidValue;
        grid = dim3((unsigned)((g.n[2] + threads - 1) / threads), (unsigned)g.n[1], (unsigned)g.n[0]);
    } else {
        grid = dim3((unsigned)((g.cells + threads - 1) / threads));
    }
    if (g.m == 1) k_step_naive<1><<<grid, threads, 0, s>>>(a, out, g, off, blk);
    else if (g.m == 2) k_step_naive<2><<<grid, threads, 0, s>>>(a, out, g, off, blk);
    else k_step_naive<0><<<grid, threads, 0, s>>>(a, out, g, off, blk);
    return cudaGetLastError();
}

}  // namespace fsx
