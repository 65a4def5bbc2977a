// C entry points over the REFERENCE's own periodic path -- TEST INFRASTRUCTURE.
//
// oracle/Makefile (target `ref`) compiles the reference's sources where they lie
// (/root/reference/proj/src/{fft,spectrum,periodic,parallel,grid,kernel,oracle,band}.cpp,
// unmodified, with the reference's flags) against oracle/eigen_shim (a stand-in
// for the absent Eigen3) together with this file into
// oracle/_ref/libfftstencil_ref.so.  The exported functions have the same
// names, arguments and status codes as oracle/fftstencil_oracle.cpp's, so
// oracle/oracle.py binds either library; tests/test_oracle_vs_ref_cpu.py uses
// this one to validate the restatement, and bench.py's CPU legs time it when it
// is present (`cpu_baseline.kind = "reference"`).  Nothing here is product code.
//
// Each function calls the reference API it names:
//   orc_solve_periodic            fftstencil::solve_periodic          periodic.hpp:43-44
//   orc_solve_periodic_vector     fftstencil::solve_periodic_vector   periodic.hpp:54-55
//   orc_solve_periodic_implicit   fftstencil::solve_periodic_implicit periodic.hpp:58-60
//   orc_multi_fft                 multi_fft / multi_ifft               fft.hpp:14-15
//   orc_spectrum_from_kernel ...  spectrum.hpp:41-49
//   orc_step_periodic, orc_evolve_periodic_naive, orc_dense_stencil_matrix   oracle.hpp:12-33
//   orc_set_threads / orc_thread_count   parallel.hpp:10-11
#include <complex>
#include <cstdint>
#include <cstring>
#include <string>
#include <vector>

#include "fftstencil/oracle.hpp"
#include "fftstencil/parallel.hpp"
#include "fftstencil/periodic.hpp"
#include "fftstencil/spectrum.hpp"

namespace fs = fftstencil;
using cd = std::complex<double>;

namespace {
thread_local std::string g_err;

template <class F>
int guard(F&& f) {
    try {
        f();
        g_err.clear();
        return 0;
    } catch (const fs::SpecError& e) {
        g_err = e.what();
        return 1;
    } catch (const fs::NumericError& e) {
        g_err = e.what();
        return 2;
    } catch (const std::exception& e) {
        g_err = e.what();
        return 9;
    }
}

fs::GridShape shape_of(int rank, const int64_t* dims, int fields) {
    return fs::GridShape(std::vector<fs::Index>(dims, dims + rank), fields);
}

fs::StencilKernel kernel_of(int rank, int fields, int64_t ntaps, const int64_t* offsets, const double* blocks) {
    fs::StencilKernel k(rank, fields);
    for (int64_t t = 0; t < ntaps; ++t) {
        fs::StencilKernel::Offset off(offsets + t * rank, offsets + (t + 1) * rank);
        Eigen::MatrixXd b(fields, fields);
        for (int r = 0; r < fields; ++r)
            for (int c = 0; c < fields; ++c) b(r, c) = blocks[(t * fields + r) * fields + c];
        k.add_tap(std::move(off), b);
    }
    return k;
}

fs::FieldGrid grid_of(const fs::GridShape& s, const double* a) {
    fs::FieldGrid g(s);
    std::memcpy(g.data.data(), a, sizeof(double) * static_cast<size_t>(s.values()));
    return g;
}

void put(const fs::FieldGrid& g, double* out) {
    std::memcpy(out, g.data.data(), sizeof(double) * static_cast<size_t>(g.shape.values()));
}

void put_timings(const fs::StageTimings& t, double* st) {
    if (!st) return;
    st[0] += t.forward_fft;
    st[1] += t.squaring;
    st[2] += t.hadamard;
    st[3] += t.inverse_fft;
    st[4] += t.boundary_recursion;
}

fs::DiagonalSpectrum spectrum_of(const fs::GridShape& s, const double* in) {
    fs::DiagonalSpectrum lam(s);
    std::memcpy(lam.blocks.data(), in, sizeof(cd) * static_cast<size_t>(lam.blocks.size()));
    return lam;
}
}  // namespace

extern "C" {

const char* orc_last_error(void) { return g_err.c_str(); }
void orc_set_threads(int n) { fs::set_thread_count(n); }
int orc_thread_count(void) { return fs::thread_count(); }
int orc_is_reference(void) { return 1; }

int orc_solve_periodic(int rank, const int64_t* dims, int fields, const double* a0, int64_t ntaps,
                       const int64_t* offsets, const double* blocks, uint64_t T, double* out, double* timings) {
    return guard([&] {
        const fs::GridShape s = shape_of(rank, dims, fields);
        const fs::StencilKernel k = kernel_of(rank, fields, ntaps, offsets, blocks);
        fs::StageTimings t;
        put(fs::solve_periodic(grid_of(s, a0), k, T, &t), out);
        put_timings(t, timings);
    });
}

int orc_solve_periodic_vector(int rank, const int64_t* dims, int fields, const double* a0, int64_t ntaps,
                              const int64_t* offsets, const double* blocks, uint64_t T, double* out,
                              double* timings) {
    return guard([&] {
        const fs::GridShape s = shape_of(rank, dims, fields);
        const fs::StencilKernel k = kernel_of(rank, fields, ntaps, offsets, blocks);
        fs::StageTimings t;
        put(fs::solve_periodic_vector(grid_of(s, a0), k, T, &t), out);
        put_timings(t, timings);
    });
}

int orc_solve_periodic_implicit(int rank, const int64_t* dims, const double* a0, int64_t nq, const int64_t* qoff,
                                const double* qval, int64_t ns, const int64_t* soff, const double* sval, uint64_t T,
                                double* out, double* timings) {
    return guard([&] {
        const fs::GridShape s = shape_of(rank, dims, 1);
        const fs::StencilKernel q = kernel_of(rank, 1, nq, qoff, qval);
        const fs::StencilKernel sk = kernel_of(rank, 1, ns, soff, sval);
        fs::StageTimings t;
        put(fs::solve_periodic_implicit(q, sk, grid_of(s, a0), T, &t), out);
        put_timings(t, timings);
    });
}

int orc_multi_fft(int rank, const int64_t* dims, int fields, const double* in, double* out, int inverse) {
    return guard([&] {
        fs::ComplexGrid g(shape_of(rank, dims, fields));
        std::memcpy(g.data.data(), in, sizeof(cd) * static_cast<size_t>(g.shape.values()));
        const fs::ComplexGrid r = inverse ? fs::multi_ifft(g) : fs::multi_fft(g);
        std::memcpy(out, r.data.data(), sizeof(cd) * static_cast<size_t>(r.shape.values()));
    });
}

int orc_spectrum_from_kernel(int rank, const int64_t* dims, int fields, int64_t ntaps, const int64_t* offsets,
                             const double* blocks, double* out) {
    return guard([&] {
        const fs::GridShape s = shape_of(rank, dims, fields);
        const fs::DiagonalSpectrum lam = fs::spectrum_from_kernel(kernel_of(rank, fields, ntaps, offsets, blocks), s);
        std::memcpy(out, lam.blocks.data(), sizeof(cd) * static_cast<size_t>(lam.blocks.size()));
    });
}

int orc_pow_spectrum(int rank, const int64_t* dims, int m, const double* in, uint64_t T, double* out) {
    return guard([&] {
        const fs::DiagonalSpectrum r = fs::pow_spectrum(spectrum_of(shape_of(rank, dims, m), in), T);
        std::memcpy(out, r.blocks.data(), sizeof(cd) * static_cast<size_t>(r.blocks.size()));
    });
}

int orc_pseudo_inverse_spectrum(int rank, const int64_t* dims, int m, const double* in, double* out) {
    return guard([&] {
        const fs::DiagonalSpectrum r = fs::pseudo_inverse_spectrum(spectrum_of(shape_of(rank, dims, m), in));
        std::memcpy(out, r.blocks.data(), sizeof(cd) * static_cast<size_t>(r.blocks.size()));
    });
}

int orc_multiply_spectra(int rank, const int64_t* dims, int m, const double* a, const double* b, double* out) {
    return guard([&] {
        const fs::GridShape s = shape_of(rank, dims, m);
        const fs::DiagonalSpectrum r = fs::multiply_spectra(spectrum_of(s, a), spectrum_of(s, b));
        std::memcpy(out, r.blocks.data(), sizeof(cd) * static_cast<size_t>(r.blocks.size()));
    });
}

int orc_hadamard(int rank, const int64_t* dims, int m, const double* lam_blocks, const double* x, double* out) {
    return guard([&] {
        const fs::GridShape s = shape_of(rank, dims, m);
        fs::ComplexGrid g(s);
        std::memcpy(g.data.data(), x, sizeof(cd) * static_cast<size_t>(s.values()));
        const fs::ComplexGrid y = fs::hadamard(spectrum_of(s, lam_blocks), g);
        std::memcpy(out, y.data.data(), sizeof(cd) * static_cast<size_t>(s.values()));
    });
}

int orc_step_periodic(int rank, const int64_t* dims, int fields, const double* a, int64_t ntaps,
                      const int64_t* offsets, const double* blocks, double* out) {
    return guard([&] {
        const fs::GridShape s = shape_of(rank, dims, fields);
        put(fs::step_periodic(grid_of(s, a), kernel_of(rank, fields, ntaps, offsets, blocks)), out);
    });
}

int orc_evolve_periodic_naive(int rank, const int64_t* dims, int fields, const double* a0, int64_t ntaps,
                              const int64_t* offsets, const double* blocks, uint64_t T, double* out) {
    return guard([&] {
        const fs::GridShape s = shape_of(rank, dims, fields);
        put(fs::evolve_periodic_naive(grid_of(s, a0), kernel_of(rank, fields, ntaps, offsets, blocks), T), out);
    });
}

int orc_dense_stencil_matrix(int rank, const int64_t* dims, int fields, int64_t ntaps, const int64_t* offsets,
                             const double* blocks, double* mat) {
    return guard([&] {
        const fs::GridShape s = shape_of(rank, dims, fields);
        const Eigen::MatrixXd m = fs::dense_stencil_matrix(kernel_of(rank, fields, ntaps, offsets, blocks), s);
        for (Eigen::Index r = 0; r < m.rows(); ++r)
            for (Eigen::Index c = 0; c < m.cols(); ++c) mat[r * m.cols() + c] = m(r, c);
    });
}

}  // extern "C"
