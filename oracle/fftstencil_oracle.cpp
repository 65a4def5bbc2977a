// ============================================================================
// fftstencil ORACLE — TEST INFRASTRUCTURE, NOT PRODUCT CODE.
//
// A CPU restatement of the reference library's StencilFFT-P hot path
// (/root/reference/proj, C++20 + Eigen; its own build needs Eigen3 and
// vendor/, both absent).  It follows the reference
// algorithm for algorithm so that it can stand in for the reference both as
// the parity checker and as the timed CPU baseline:
//
//   * radix-2 iterative FFT with bit-reverse + twiddle tables, Bluestein for
//     every other length, inverse by conjugation     (proj/src/fft.cpp:20-155)
//   * per-axis strided gather/transform/scatter       (proj/src/fft.cpp:159-192)
//   * generator scatter + multi-FFT spectrum          (proj/src/spectrum.cpp:21-45)
//   * binary-exponentiation spectrum power            (proj/src/spectrum.cpp:47-83)
//   * pseudo-inverse / multiply / hadamard            (proj/src/spectrum.cpp:85-134)
//   * pipeline, residue check, T == 0 short cut       (proj/src/periodic.cpp:27-124)
//   * std::thread chunked parallel_for, n < 2048 inline (proj/src/parallel.cpp:11-58)
//   * naive Theta(NT) stepping                        (proj/src/oracle.cpp:23-113)
//   * tap accumulation and require_fits               (proj/src/kernel.cpp:7-49)
//   * modal truth: three Fourier modes amplified by the double-double
//     lambda^T (accuracy-parity criterion)             (proj/src/modal.cpp:13-145)
//
// It is pinned against the reference's own known-answer and property tests
// (tests/golden/reference_known_answers.json, tests/test_oracle_cpu.py) and,
// bit for bit, against the reference's own sources compiled against a
// stand-in for Eigen (oracle/_ref, `make -C oracle ref`;
// tests/test_oracle_vs_ref_cpu.py, tests/golden/reference_outputs.npz).
//
// Only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline /
// `--impl reference` leg may load this library; the product path never does.
//
// The numerical core is templated on the real type so that the same
// algorithm instantiated with x87 long double serves as the higher-precision
// "truth" of the config-5 parity protocol.
// ============================================================================

#include <algorithm>
#include <atomic>
#include <bit>
#include <chrono>
#include <cmath>
#include <complex>
#include <cstdint>
#include <cstring>
#include <exception>
#include <functional>
#include <map>
#include <memory>
#include <mutex>
#include <numbers>
#include <stdexcept>
#include <string>
#include <thread>
#include <vector>

namespace orc {

using i64 = std::int64_t;
using u64 = std::uint64_t;

struct SpecError : std::runtime_error {
    using std::runtime_error::runtime_error;
};
struct NumericError : std::runtime_error {
    using std::runtime_error::runtime_error;
};

// ---------------------------------------------------------------- threading
// proj/src/parallel.cpp:11-58: a process-wide thread budget; ranges below
// 2048 items (or a budget of one) run inline; otherwise contiguous chunks,
// one std::thread each, joined, first exception rethrown.
static std::atomic<int> g_thread_budget{0};

static int threads_in_use() {
    int t = g_thread_budget.load(std::memory_order_relaxed);
    if (t > 0) return t;
    unsigned hw = std::thread::hardware_concurrency();
    return hw ? static_cast<int>(hw) : 1;
}

static void for_chunks(i64 count, const std::function<void(i64, i64)>& body) {
    if (count <= 0) return;
    const int budget = threads_in_use();
    if (budget <= 1 || count < 2048) {
        body(0, count);
        return;
    }
    const i64 workers = std::min<i64>(budget, count);
    const i64 span = (count + workers - 1) / workers;
    std::exception_ptr err;
    std::atomic<bool> failed{false};
    auto guarded = [&](i64 lo, i64 hi) {
        try {
            body(lo, hi);
        } catch (...) {
            if (!failed.exchange(true)) err = std::current_exception();
        }
    };
    std::vector<std::thread> crew;
    for (i64 w = 1; w < workers; ++w) {
        const i64 lo = w * span, hi = std::min(count, lo + span);
        if (lo >= hi) break;
        crew.emplace_back(guarded, lo, hi);
    }
    guarded(0, std::min(span, count));
    for (auto& t : crew) t.join();
    if (failed.load()) std::rethrow_exception(err);
}

// ---------------------------------------------------------------- shapes
struct Shape {
    std::vector<i64> dims;
    int fields = 1;
    i64 cells = 0;

    Shape() = default;
    Shape(const i64* d, int rank, int m) : dims(d, d + rank), fields(m) {
        if (rank < 1) throw SpecError("GridShape: need at least one dimension");
        if (fields < 1) throw SpecError("GridShape: fields must be >= 1");
        __int128 n = 1;
        for (i64 v : dims) {
            if (v < 1) throw SpecError("GridShape: every dimension must be >= 1");
            n *= v;
            if (n * fields > (__int128)INT64_MAX)
                throw SpecError("GridShape: total value count overflows");
        }
        cells = static_cast<i64>(n);
    }
    int rank() const { return static_cast<int>(dims.size()); }
    i64 values() const { return cells * fields; }
};

// ---------------------------------------------------------------- kernels
// Sorted map offset -> m*m row-major block; add accumulates and rejects
// non-finite coefficients (proj/src/kernel.cpp:7-22).
struct Kernel {
    int rank = 1, fields = 1;
    std::map<std::vector<i64>, std::vector<double>> taps;

    Kernel(int r, int m) : rank(r), fields(m) {
        if (rank < 1) throw SpecError("StencilKernel: rank must be >= 1");
        if (fields < 1) throw SpecError("StencilKernel: fields must be >= 1");
    }
    void add(const i64* off, const double* block) {
        const int mm = fields * fields;
        for (int i = 0; i < mm; ++i)
            if (!std::isfinite(block[i]))
                throw SpecError("StencilKernel: non-finite coefficient");
        std::vector<i64> key(off, off + rank);
        auto [it, fresh] = taps.try_emplace(key, std::vector<double>(block, block + mm));
        if (!fresh)
            for (int i = 0; i < mm; ++i) it->second[i] += block[i];
    }
    // proj/src/kernel.cpp:38-49
    void require_fits(const Shape& s) const {
        if (taps.empty()) throw SpecError("StencilKernel: at least one tap required");
        if (s.rank() != rank) throw SpecError("StencilKernel: grid rank mismatch");
        if (s.fields != fields) throw SpecError("StencilKernel: grid field count mismatch");
        for (int a = 0; a < rank; ++a) {
            i64 reach = 0;
            for (const auto& [off, blk] : taps) reach = std::max(reach, off[a] < 0 ? -off[a] : off[a]);
            if (reach >= s.dims[a])
                throw SpecError("StencilKernel: tap offset exceeds dimension " + std::to_string(a));
        }
    }
};

static Kernel kernel_from_arrays(int rank, int m, i64 ntaps, const i64* offsets,
                                 const double* blocks) {
    Kernel k(rank, m);
    for (i64 t = 0; t < ntaps; ++t) k.add(offsets + t * rank, blocks + t * m * m);
    return k;
}

// ---------------------------------------------------------------- FFT
template <class R>
using cx = std::complex<R>;

template <class R>
static R pi_v() {
    return std::numbers::pi_v<R>;
}

template <class R>
struct FftPlan {
    i64 n = 0;
    bool pow2 = false;
    std::vector<i64> rev;      // bit reversal permutation
    std::vector<cx<R>> roots;  // exp(-2 pi i j / n), j < n/2
    std::shared_ptr<const FftPlan<R>> inner;  // Bluestein: padded pow2 plan
    i64 padded = 0;
    std::vector<cx<R>> chirp;      // exp(-i pi k^2 / n)
    std::vector<cx<R>> chirp_hat;  // transform of the wrapped conjugate chirp
};

// exp(-i pi k^2 / n) with k^2 reduced mod 2n first (proj/src/fft.cpp:18-25)
template <class R>
static cx<R> chirp_at(i64 k, i64 n) {
    const i64 q = static_cast<i64>((static_cast<__int128>(k) * k) % (2 * n));
    const R ang = -pi_v<R>() * static_cast<R>(q) / static_cast<R>(n);
    return {std::cos(ang), std::sin(ang)};
}

// Iterative radix-2: bit-reverse permutation then log2 n butterfly sweeps
// reading the twiddle at stride n/len (proj/src/fft.cpp:40-59).
template <class R>
static void radix2(const FftPlan<R>& p, cx<R>* a) {
    const i64 n = p.n;
    for (i64 i = 0; i < n; ++i) {
        const i64 j = p.rev[i];
        if (i < j) std::swap(a[i], a[j]);
    }
    for (i64 len = 2; len <= n; len <<= 1) {
        const i64 half = len / 2, stride = n / len;
        for (i64 base = 0; base < n; base += len)
            for (i64 j = 0; j < half; ++j) {
                const cx<R> w = p.roots[j * stride];
                const cx<R> lo = a[base + j];
                const cx<R> hi = a[base + j + half] * w;
                a[base + j] = lo + hi;
                a[base + j + half] = lo - hi;
            }
    }
}

template <class R>
static std::shared_ptr<const FftPlan<R>> plan_for(i64 n);

template <class R>
static std::shared_ptr<const FftPlan<R>> build_plan(i64 n) {
    auto p = std::make_shared<FftPlan<R>>();
    p->n = n;
    p->pow2 = std::has_single_bit(static_cast<u64>(n));
    if (p->pow2) {
        const int bits = std::countr_zero(static_cast<u64>(n));
        p->rev.resize(n);
        for (i64 i = 0; i < n; ++i) {
            u64 v = static_cast<u64>(i), r = 0;
            for (int b = 0; b < bits; ++b) {
                r = (r << 1) | (v & 1);
                v >>= 1;
            }
            p->rev[i] = static_cast<i64>(r);
        }
        p->roots.resize(std::max<i64>(n / 2, 1));
        for (i64 j = 0; j < static_cast<i64>(p->roots.size()); ++j) {
            const R ang = -R(2) * pi_v<R>() * static_cast<R>(j) / static_cast<R>(n);
            p->roots[j] = {std::cos(ang), std::sin(ang)};
        }
        return p;
    }
    // Bluestein (proj/src/fft.cpp:103-119): padded power of two >= 2n-1.
    i64 m = 1;
    while (m < 2 * n - 1) m <<= 1;
    p->padded = m;
    p->inner = plan_for<R>(m);
    p->chirp.resize(n);
    for (i64 k = 0; k < n; ++k) p->chirp[k] = chirp_at<R>(k, n);
    std::vector<cx<R>> b(m, cx<R>(0, 0));
    b[0] = std::conj(p->chirp[0]);
    for (i64 k = 1; k < n; ++k) {
        b[k] = std::conj(p->chirp[k]);
        b[m - k] = b[k];
    }
    radix2(*p->inner, b.data());
    p->chirp_hat = std::move(b);
    return p;
}

template <class R>
struct PlanCache {
    std::mutex mu;
    std::map<i64, std::shared_ptr<const FftPlan<R>>> by_len;
};

template <class R>
static PlanCache<R>& plan_cache() {
    static PlanCache<R> c;
    return c;
}

// proj/src/fft.cpp:63-77: lookup under the lock, build outside it.
template <class R>
static std::shared_ptr<const FftPlan<R>> plan_for(i64 n) {
    auto& c = plan_cache<R>();
    {
        std::scoped_lock lk(c.mu);
        auto it = c.by_len.find(n);
        if (it != c.by_len.end()) return it->second;
    }
    auto fresh = build_plan<R>(n);
    std::scoped_lock lk(c.mu);
    return c.by_len.try_emplace(n, std::move(fresh)).first->second;
}

template <class R>
static void forward_any(const FftPlan<R>& p, cx<R>* a) {
    if (p.pow2) {
        radix2(p, a);
        return;
    }
    // Bluestein chirp-z (proj/src/fft.cpp:122-139)
    const i64 n = p.n, m = p.padded;
    std::vector<cx<R>> w(m, cx<R>(0, 0));
    for (i64 k = 0; k < n; ++k) w[k] = a[k] * p.chirp[k];
    radix2(*p.inner, w.data());
    for (i64 k = 0; k < m; ++k) w[k] *= p.chirp_hat[k];
    for (auto& v : w) v = std::conj(v);
    radix2(*p.inner, w.data());
    const R s = R(1) / static_cast<R>(m);
    for (i64 j = 0; j < n; ++j) a[j] = std::conj(w[j]) * s * p.chirp[j];
}

// proj/src/fft.cpp:143-155: forward unnormalized; inverse = conj, forward,
// conj * 1/n.
template <class R>
static void fft_line(cx<R>* buf, i64 n, bool inverse) {
    if (n <= 1) return;
    auto p = plan_for<R>(n);
    if (!inverse) {
        forward_any(*p, buf);
        return;
    }
    for (i64 i = 0; i < n; ++i) buf[i] = std::conj(buf[i]);
    forward_any(*p, buf);
    const R s = R(1) / static_cast<R>(n);
    for (i64 i = 0; i < n; ++i) buf[i] = std::conj(buf[i]) * s;
}

// proj/src/fft.cpp:159-186: copy, then per axis (length-1 axes skipped)
// every line (outer x inner, inner includes the field count) is gathered,
// transformed and scattered back, lines spread over parallel_for.
template <class R>
static std::vector<cx<R>> multi_transform(const std::vector<cx<R>>& g, const Shape& s,
                                          bool inverse) {
    std::vector<cx<R>> out = g;
    const int rank = s.rank();
    for (int axis = 0; axis < rank; ++axis) {
        const i64 len = s.dims[axis];
        if (len == 1) continue;
        i64 outer = 1, inner = s.fields;
        for (int b = 0; b < axis; ++b) outer *= s.dims[b];
        for (int b = axis + 1; b < rank; ++b) inner *= s.dims[b];
        const i64 block = len * inner;
        for_chunks(outer * inner, [&](i64 lo, i64 hi) {
            std::vector<cx<R>> line(len);
            for (i64 L = lo; L < hi; ++L) {
                cx<R>* base = out.data() + (L / inner) * block + (L % inner);
                for (i64 k = 0; k < len; ++k) line[k] = base[k * inner];
                fft_line<R>(line.data(), len, inverse);
                for (i64 k = 0; k < len; ++k) base[k * inner] = line[k];
            }
        });
    }
    return out;
}

// ---------------------------------------------------------------- spectra
// Frequency-major m*m complex blocks (proj/include/fftstencil/spectrum.hpp:16-38).
template <class R>
struct Spectrum {
    Shape shape;
    std::vector<cx<R>> blocks;
    int m() const { return shape.fields; }
};

// proj/src/spectrum.cpp:21-45: scatter block at (-off) mod dims into an
// m^2-field generator grid, one multi-FFT of it.
template <class R>
static Spectrum<R> spectrum_from_kernel(const Kernel& k, const Shape& s) {
    k.require_fits(s);
    const int rank = s.rank(), m = s.fields;
    Shape gs = s;
    gs.fields = m * m;
    std::vector<cx<R>> gen(static_cast<size_t>(s.cells) * m * m, cx<R>(0, 0));
    for (const auto& [off, blk] : k.taps) {
        i64 cell = 0;
        for (int a = 0; a < rank; ++a) {
            i64 j = (-off[a]) % s.dims[a];
            if (j < 0) j += s.dims[a];
            cell = cell * s.dims[a] + j;
        }
        for (int i = 0; i < m * m; ++i) gen[cell * m * m + i] += cx<R>(static_cast<R>(blk[i]), 0);
    }
    Spectrum<R> lam{s, {}};
    lam.blocks = multi_transform<R>(gen, gs, false);
    return lam;
}

template <class R>
static void matmul(int m, const cx<R>* a, const cx<R>* b, cx<R>* c) {
    for (int r = 0; r < m; ++r)
        for (int col = 0; col < m; ++col) {
            cx<R> acc(0, 0);
            for (int t = 0; t < m; ++t) acc += a[r * m + t] * b[t * m + col];
            c[r * m + col] = acc;
        }
}

// proj/src/spectrum.cpp:47-83: acc = 1, sq = lambda; while t {if t&1 acc *=
// sq; t >>= 1; if t sq *= sq}.  Blocks use m x m products.
template <class R>
static Spectrum<R> pow_spectrum(const Spectrum<R>& lam, u64 T) {
    const int m = lam.m();
    Spectrum<R> out{lam.shape, std::vector<cx<R>>(lam.blocks.size())};
    const i64 n = lam.shape.cells;
    if (m == 1) {
        for_chunks(n, [&](i64 lo, i64 hi) {
            for (i64 j = lo; j < hi; ++j) {
                cx<R> acc(1, 0), sq = lam.blocks[j];
                u64 t = T;
                while (t) {
                    if (t & 1) acc *= sq;
                    t >>= 1;
                    if (t) sq *= sq;
                }
                out.blocks[j] = acc;
            }
        });
        return out;
    }
    for_chunks(n, [&](i64 lo, i64 hi) {
        std::vector<cx<R>> acc(m * m), sq(m * m), tmp(m * m);
        for (i64 j = lo; j < hi; ++j) {
            for (int i = 0; i < m * m; ++i) acc[i] = (i % (m + 1) == 0) ? cx<R>(1, 0) : cx<R>(0, 0);
            std::copy_n(lam.blocks.begin() + j * m * m, m * m, sq.begin());
            u64 t = T;
            while (t) {
                if (t & 1) {
                    matmul<R>(m, acc.data(), sq.data(), tmp.data());
                    acc.swap(tmp);
                }
                t >>= 1;
                if (t) {
                    matmul<R>(m, sq.data(), sq.data(), tmp.data());
                    sq.swap(tmp);
                }
            }
            std::copy_n(acc.begin(), m * m, out.blocks.begin() + j * m * m);
        }
    });
    return out;
}

// proj/src/spectrum.cpp:85-96: |v| <= 1e-12 * max|v| -> 0, else 1/v.
template <class R>
static Spectrum<R> pseudo_inverse_spectrum(const Spectrum<R>& lam) {
    if (lam.m() != 1) throw SpecError("pseudo_inverse_spectrum: scalar spectra only");
    R maxmag = 0;
    for (const auto& v : lam.blocks) maxmag = std::max<R>(maxmag, std::abs(v));
    const R eps = R(1e-12) * maxmag;
    Spectrum<R> out{lam.shape, std::vector<cx<R>>(lam.blocks.size())};
    for (size_t j = 0; j < lam.blocks.size(); ++j) {
        const cx<R> v = lam.blocks[j];
        out.blocks[j] = std::abs(v) <= eps ? cx<R>(0, 0) : R(1) / v;
    }
    return out;
}

// proj/src/spectrum.cpp:98-109
template <class R>
static Spectrum<R> multiply_spectra(const Spectrum<R>& a, const Spectrum<R>& b) {
    if (a.shape.dims != b.shape.dims || a.shape.fields != b.shape.fields)
        throw SpecError("multiply_spectra: shape mismatch");
    const int m = a.m();
    Spectrum<R> out{a.shape, std::vector<cx<R>>(a.blocks.size())};
    if (m == 1) {
        for (size_t j = 0; j < a.blocks.size(); ++j) out.blocks[j] = a.blocks[j] * b.blocks[j];
        return out;
    }
    for (i64 j = 0; j < a.shape.cells; ++j)
        matmul<R>(m, &a.blocks[j * m * m], &b.blocks[j * m * m], &out.blocks[j * m * m]);
    return out;
}

// proj/src/spectrum.cpp:111-134: y[j] = lam[j] x[j] (block mat-vec for m>1).
template <class R>
static std::vector<cx<R>> hadamard(const Spectrum<R>& lam, const std::vector<cx<R>>& x,
                                   const Shape& xs) {
    if (lam.shape.dims != xs.dims || lam.shape.fields != xs.fields)
        throw SpecError("hadamard: shape mismatch");
    const int m = lam.m();
    const i64 n = xs.cells;
    std::vector<cx<R>> y(x.size());
    if (m == 1) {
        for_chunks(n, [&](i64 lo, i64 hi) {
            for (i64 j = lo; j < hi; ++j) y[j] = lam.blocks[j] * x[j];
        });
        return y;
    }
    for_chunks(n, [&](i64 lo, i64 hi) {
        for (i64 j = lo; j < hi; ++j)
            for (int r = 0; r < m; ++r) {
                cx<R> acc(0, 0);
                for (int c = 0; c < m; ++c) acc += lam.blocks[j * m * m + r * m + c] * x[j * m + c];
                y[j * m + r] = acc;
            }
    });
    return y;
}

// ---------------------------------------------------------------- solver
// StageTimings: seconds accumulated with += (proj/src/periodic.cpp:9-25).
struct Timings {
    double fwd = 0, sq = 0, had = 0, inv = 0, brec = 0;
};

struct Watch {
    double* sink;
    std::chrono::steady_clock::time_point t0 = std::chrono::steady_clock::now();
    explicit Watch(double* s) : sink(s) {}
    ~Watch() {
        if (sink)
            *sink += std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count();
    }
};

// proj/src/periodic.cpp:49-65: inverse multi-FFT, serial finite/residue
// scan, real part.
template <class R>
static void realize_checked(const std::vector<cx<R>>& y, const Shape& s, R* out, Timings* st) {
    Watch w(st ? &st->inv : nullptr);
    const std::vector<cx<R>> z = multi_transform<R>(y, s, true);
    R max_re = 0, max_im = 0;
    for (const auto& v : z) {
        if (!std::isfinite(v.real()) || !std::isfinite(v.imag()))
            throw NumericError("solve_periodic: non-finite value after inverse FFT");
        max_re = std::max<R>(max_re, std::abs(v.real()));
        max_im = std::max<R>(max_im, std::abs(v.imag()));
    }
    if (max_im > R(1e-6) * max_re)
        throw NumericError("solve_periodic: imaginary residue " + std::to_string((double)max_im) +
                           " exceeds 1e-6 * max |real| (" + std::to_string((double)max_re) +
                           "); spectrum likely blew up");
    for (size_t i = 0; i < z.size(); ++i) out[i] = z[i].real();
}

// proj/src/periodic.cpp:27-45
template <class R>
static void pipeline(const R* a0, const Shape& s, const Spectrum<R>& lam, u64 T, R* out,
                     Timings* st) {
    std::vector<cx<R>> x;
    {
        Watch w(st ? &st->fwd : nullptr);
        std::vector<cx<R>> c(s.values());
        for (i64 i = 0; i < s.values(); ++i) c[i] = cx<R>(a0[i], 0);
        x = multi_transform<R>(c, s, false);
    }
    Spectrum<R> lt;
    {
        Watch w(st ? &st->sq : nullptr);
        lt = pow_spectrum<R>(lam, T);
    }
    std::vector<cx<R>> y;
    {
        Watch w(st ? &st->had : nullptr);
        y = hadamard<R>(lt, x, s);
    }
    realize_checked<R>(y, s, out, st);
}

// proj/src/periodic.cpp:76-86
template <class R>
static void solve_periodic(const R* a0, const Shape& s, const Kernel& k, u64 T, R* out,
                           Timings* st) {
    k.require_fits(s);
    if (T == 0) {
        std::copy_n(a0, s.values(), out);
        return;
    }
    Spectrum<R> lam;
    {
        Watch w(st ? &st->fwd : nullptr);
        lam = spectrum_from_kernel<R>(k, s);
    }
    pipeline<R>(a0, s, lam, T, out, st);
}

// proj/src/periodic.cpp:108-124
template <class R>
static void solve_periodic_implicit(const Kernel& q, const Kernel& sk, const R* a0,
                                    const Shape& s, u64 T, R* out, Timings* st) {
    if (q.fields != 1 || sk.fields != 1)
        throw SpecError("solve_periodic_implicit: scalar kernels only");
    q.require_fits(s);
    sk.require_fits(s);
    if (T == 0) {
        std::copy_n(a0, s.values(), out);
        return;
    }
    Spectrum<R> lr;
    {
        Watch w(st ? &st->fwd : nullptr);
        const Spectrum<R> lq = spectrum_from_kernel<R>(q, s);
        const Spectrum<R> ls = spectrum_from_kernel<R>(sk, s);
        lr = multiply_spectra<R>(pseudo_inverse_spectrum<R>(lq), ls);
    }
    pipeline<R>(a0, s, lr, T, out, st);
}

// ---------------------------------------------------------------- naive
// proj/src/oracle.cpp:26-86: one periodic step, taps in sorted order; the
// scalar path accumulates c * shifted line per tap, the block path per cell.
static void step_scalar(const double* a, const Shape& s, const Kernel& k, double* out) {
    const int rank = s.rank();
    const i64 inner = s.dims[rank - 1];
    const i64 outer = s.cells / inner;
    std::fill_n(out, s.cells, 0.0);
    for (const auto& [off, blk] : k.taps) {
        const double c = blk[0];
        const i64 shift = ((off[rank - 1] % inner) + inner) % inner;
        std::vector<i64> idx(std::max(rank - 1, 0), 0);
        for (i64 o = 0; o < outer; ++o) {
            i64 src = 0;
            for (int ax = 0; ax + 1 < rank; ++ax) {
                i64 j = (idx[ax] + off[ax]) % s.dims[ax];
                if (j < 0) j += s.dims[ax];
                src = src * s.dims[ax] + j;
            }
            const double* in = a + src * inner;
            double* dst = out + o * inner;
            const i64 run = inner - shift;
            for (i64 i = 0; i < run; ++i) dst[i] += c * in[i + shift];
            for (i64 i = run; i < inner; ++i) dst[i] += c * in[i + shift - inner];
            for (int ax = rank - 2; ax >= 0; --ax) {
                if (++idx[ax] < s.dims[ax]) break;
                idx[ax] = 0;
            }
        }
    }
}

static void step_blocks(const double* a, const Shape& s, const Kernel& k, double* out) {
    const int rank = s.rank(), m = s.fields;
    std::fill_n(out, s.values(), 0.0);
    std::vector<i64> idx(rank, 0);
    for (i64 cell = 0; cell < s.cells; ++cell) {
        for (const auto& [off, blk] : k.taps) {
            i64 src = 0;
            for (int ax = 0; ax < rank; ++ax) {
                i64 j = (idx[ax] + off[ax]) % s.dims[ax];
                if (j < 0) j += s.dims[ax];
                src = src * s.dims[ax] + j;
            }
            for (int f = 0; f < m; ++f) {
                double acc = 0;
                for (int g = 0; g < m; ++g) acc += blk[f * m + g] * a[src * m + g];
                out[cell * m + f] += acc;
            }
        }
        for (int ax = rank - 1; ax >= 0; --ax) {
            if (++idx[ax] < s.dims[ax]) break;
            idx[ax] = 0;
        }
    }
}

static void step_periodic(const double* a, const Shape& s, const Kernel& k, double* out) {
    k.require_fits(s);
    if (s.fields == 1)
        step_scalar(a, s, k, out);
    else
        step_blocks(a, s, k, out);
}

// proj/src/oracle.cpp:100-113
static void evolve_naive(const double* a0, const Shape& s, const Kernel& k, u64 T, double* out) {
    k.require_fits(s);
    std::vector<double> cur(a0, a0 + s.values()), nxt(s.values());
    for (u64 t = 0; t < T; ++t) {
        if (s.fields == 1)
            step_scalar(cur.data(), s, k, nxt.data());
        else
            step_blocks(cur.data(), s, k, nxt.data());
        cur.swap(nxt);
    }
    std::copy(cur.begin(), cur.end(), out);
}

// proj/src/oracle.cpp:194-220 (dense step matrix, <= 2048 values).
static void dense_matrix(const Shape& s, const Kernel& k, double* mat) {
    k.require_fits(s);
    const i64 n = s.values();
    if (n > 2048)
        throw SpecError("dense_stencil_matrix: size " + std::to_string(n) +
                        " exceeds the dense-storage guard (2048)");
    const int rank = s.rank(), m = s.fields;
    std::fill_n(mat, n * n, 0.0);
    std::vector<i64> idx(rank, 0);
    for (i64 cell = 0; cell < s.cells; ++cell) {
        for (const auto& [off, blk] : k.taps) {
            i64 src = 0;
            for (int ax = 0; ax < rank; ++ax) {
                i64 j = (idx[ax] + off[ax]) % s.dims[ax];
                if (j < 0) j += s.dims[ax];
                src = src * s.dims[ax] + j;
            }
            for (int f = 0; f < m; ++f)
                for (int g = 0; g < m; ++g) mat[(cell * m + f) * n + src * m + g] += blk[f * m + g];
        }
        for (int ax = rank - 1; ax >= 0; --ax) {
            if (++idx[ax] < s.dims[ax]) break;
            idx[ax] = 0;
        }
    }
}

}  // namespace orc

// ============================================================================
// C ABI (mirrors include/fsx.h so parity tests can call both the same way).
// Status: 0 ok, 1 SpecError, 2 NumericError, 9 other.
// ============================================================================
namespace {
thread_local std::string g_err;

template <class F>
int guard(F&& f) {
    try {
        f();
        g_err.clear();
        return 0;
    } catch (const orc::SpecError& e) {
        g_err = e.what();
        return 1;
    } catch (const orc::NumericError& e) {
        g_err = e.what();
        return 2;
    } catch (const std::exception& e) {
        g_err = e.what();
        return 9;
    }
}

void put_timings(const orc::Timings& t, double* st) {
    if (!st) return;
    st[0] += t.fwd;
    st[1] += t.sq;
    st[2] += t.had;
    st[3] += t.inv;
    st[4] += t.brec;
}

using cd = std::complex<double>;
using cl = std::complex<long double>;

// ---------------------------------------------------------------- modal truth
// proj/src/modal.cpp:13-145: three periodic Fourier modes whose eigenvalues
// are raised to T in double-double complex arithmetic (relative error ~1e-32
// per multiply), so the reference grid Re(sum_q A_q lam_q^T e^{i(2 pi k_q.x/n + phi_q)})
// is exact far below either solver's error.  Used by the accuracy-parity
// acceptance criterion (proj/tests/acceptance.cpp:298-320).
namespace modal {
using orc::i64;
using orc::Kernel;
using orc::Shape;
using orc::SpecError;
using orc::u64;
struct DD {
    double hi = 0, lo = 0;
};
static DD two_sum(double a, double b) {
    const double s = a + b;
    const double bb = s - a;
    return {s, (a - (s - bb)) + (b - bb)};
}
static DD two_prod(double a, double b) {
    const double p = a * b;
    return {p, std::fma(a, b, -p)};
}
static DD dd_add(DD a, DD b) {
    const DD s = two_sum(a.hi, b.hi);
    return two_sum(s.hi, s.lo + a.lo + b.lo);
}
static DD dd_mul(DD a, DD b) {
    const DD p = two_prod(a.hi, b.hi);
    return two_sum(p.hi, p.lo + a.hi * b.lo + a.lo * b.hi);
}
static DD dd(double x) { return {x, 0.0}; }
struct DDC {
    DD re, im;
};
static DDC ddc_mul(const DDC& a, const DDC& b) {
    return {dd_add(dd_mul(a.re, b.re), dd_mul(dd_mul(a.im, b.im), dd(-1.0))),
            dd_add(dd_mul(a.re, b.im), dd_mul(a.im, b.re))};
}
static DDC ddc_pow(DDC base, u64 t) {
    DDC acc{dd(1.0), dd(0.0)};
    while (t) {
        if (t & 1) acc = ddc_mul(acc, base);
        t >>= 1;
        if (t) base = ddc_mul(base, base);
    }
    return acc;
}
struct Mode {
    std::vector<i64> k;
    double amplitude, phase;
};
static void problem_periodic(const Shape& s, const Kernel& k, u64 T, double* initial, double* reference) {
    k.require_fits(s);
    if (s.fields != 1) throw SpecError("accuracy mode: periodic reference needs a scalar field");
    const int d = s.rank();
    std::vector<Mode> modes(3);
    modes[0] = {std::vector<i64>(d, 0), 1.0, 0.0};
    modes[0].k[0] = 1;
    modes[1] = {std::vector<i64>(d, 0), 0.6, 0.7};
    if (d >= 2) modes[1].k[1] = 1;
    else modes[1].k[0] = 2;
    modes[2] = {std::vector<i64>(d, 1), 0.3, 1.3};
    if (d == 1) modes[2].k[0] = 3;
    std::vector<DDC> amp(modes.size());
    for (size_t q = 0; q < modes.size(); ++q) {
        std::complex<double> lam(0, 0);
        for (const auto& [off, block] : k.taps) {
            double frac = 0;
            for (int a = 0; a < d; ++a)
                frac += static_cast<double>(modes[q].k[a] * off[a]) / static_cast<double>(s.dims[a]);
            const double angle = 2.0 * std::numbers::pi * frac;
            lam += block[0] * std::complex<double>(std::cos(angle), std::sin(angle));
        }
        amp[q] = ddc_pow({dd(lam.real()), dd(lam.imag())}, T);
    }
    std::vector<i64> idx(d, 0);
    for (i64 cell = 0; cell < s.cells; ++cell) {
        double init = 0, ref = 0;
        for (size_t q = 0; q < modes.size(); ++q) {
            double frac = 0;
            for (int a = 0; a < d; ++a)
                frac += static_cast<double>((modes[q].k[a] * idx[a]) % s.dims[a]) / static_cast<double>(s.dims[a]);
            const double angle = 2.0 * std::numbers::pi * frac + modes[q].phase;
            const double c = std::cos(angle), sn = std::sin(angle);
            init += modes[q].amplitude * c;
            ref += modes[q].amplitude * (amp[q].re.hi * c - amp[q].im.hi * sn);
        }
        initial[cell] = init;
        reference[cell] = ref;
        for (int a = d - 1; a >= 0; --a) {  // next_index, row-major
            if (++idx[a] < s.dims[a]) break;
            idx[a] = 0;
        }
    }
}
}  // namespace modal
}  // namespace

extern "C" {

const char* orc_last_error(void) { return g_err.c_str(); }
void orc_set_threads(int n) { orc::g_thread_budget.store(n, std::memory_order_relaxed); }
int orc_thread_count(void) { return orc::threads_in_use(); }

// solve_periodic (fields == 1 or any m), solve_periodic_vector (m >= 2 check).
int orc_solve_periodic(int rank, const int64_t* dims, int fields, const double* a0,
                       int64_t ntaps, const int64_t* offsets, const double* blocks,
                       uint64_t T, double* out, double* timings) {
    return guard([&] {
        orc::Shape s(dims, rank, fields);
        orc::Kernel k = orc::kernel_from_arrays(rank, fields, ntaps, offsets, blocks);
        orc::Timings t;
        orc::solve_periodic<double>(a0, s, k, T, out, &t);
        put_timings(t, timings);
    });
}

int orc_solve_periodic_vector(int rank, const int64_t* dims, int fields, const double* a0,
                              int64_t ntaps, const int64_t* offsets, const double* blocks,
                              uint64_t T, double* out, double* timings) {
    return guard([&] {
        if (fields < 2) throw orc::SpecError("solve_periodic_vector: kernel must carry m > 1 blocks");
        orc::Shape s(dims, rank, fields);
        orc::Kernel k = orc::kernel_from_arrays(rank, fields, ntaps, offsets, blocks);
        orc::Timings t;
        orc::solve_periodic<double>(a0, s, k, T, out, &t);
        put_timings(t, timings);
    });
}

// Same algorithm in x87 long double: the "truth" of the config-5 protocol.
int orc_solve_periodic_ld(int rank, const int64_t* dims, int fields, const double* a0,
                          int64_t ntaps, const int64_t* offsets, const double* blocks,
                          uint64_t T, double* out) {
    return guard([&] {
        orc::Shape s(dims, rank, fields);
        orc::Kernel k = orc::kernel_from_arrays(rank, fields, ntaps, offsets, blocks);
        std::vector<long double> a(a0, a0 + s.values()), o(s.values());
        orc::solve_periodic<long double>(a.data(), s, k, T, o.data(), nullptr);
        for (int64_t i = 0; i < s.values(); ++i) out[i] = static_cast<double>(o[i]);
    });
}

int orc_solve_periodic_implicit(int rank, const int64_t* dims, const double* a0,
                                int64_t nq, const int64_t* qoff, const double* qval,
                                int64_t ns, const int64_t* soff, const double* sval,
                                uint64_t T, double* out, double* timings) {
    return guard([&] {
        orc::Shape s(dims, rank, 1);
        orc::Kernel q = orc::kernel_from_arrays(rank, 1, nq, qoff, qval);
        orc::Kernel sk = orc::kernel_from_arrays(rank, 1, ns, soff, sval);
        orc::Timings t;
        orc::solve_periodic_implicit<double>(q, sk, a0, s, T, out, &t);
        put_timings(t, timings);
    });
}

// multi_fft / multi_ifft on interleaved complex (re, im) doubles.
int orc_multi_fft(int rank, const int64_t* dims, int fields, const double* in, double* out,
                  int inverse) {
    return guard([&] {
        orc::Shape s(dims, rank, fields);
        std::vector<cd> g(reinterpret_cast<const cd*>(in), reinterpret_cast<const cd*>(in) + s.values());
        auto r = orc::multi_transform<double>(g, s, inverse != 0);
        std::memcpy(out, r.data(), r.size() * sizeof(cd));
    });
}

int orc_spectrum_from_kernel(int rank, const int64_t* dims, int fields, int64_t ntaps,
                             const int64_t* offsets, const double* blocks, double* out) {
    return guard([&] {
        orc::Shape s(dims, rank, fields);
        orc::Kernel k = orc::kernel_from_arrays(rank, fields, ntaps, offsets, blocks);
        auto lam = orc::spectrum_from_kernel<double>(k, s);
        std::memcpy(out, lam.blocks.data(), lam.blocks.size() * sizeof(cd));
    });
}

int orc_pow_spectrum(int rank, const int64_t* dims, int m, const double* in, uint64_t T,
                     double* out) {
    return guard([&] {
        orc::Shape s(dims, rank, m);
        orc::Spectrum<double> lam{s, {}};
        const size_t n = static_cast<size_t>(s.cells) * m * m;
        lam.blocks.assign(reinterpret_cast<const cd*>(in), reinterpret_cast<const cd*>(in) + n);
        auto r = orc::pow_spectrum<double>(lam, T);
        std::memcpy(out, r.blocks.data(), n * sizeof(cd));
    });
}

int orc_pseudo_inverse_spectrum(int rank, const int64_t* dims, int m, const double* in,
                                double* out) {
    return guard([&] {
        orc::Shape s(dims, rank, m);
        orc::Spectrum<double> lam{s, {}};
        const size_t n = static_cast<size_t>(s.cells) * m * m;
        lam.blocks.assign(reinterpret_cast<const cd*>(in), reinterpret_cast<const cd*>(in) + n);
        auto r = orc::pseudo_inverse_spectrum<double>(lam);
        std::memcpy(out, r.blocks.data(), n * sizeof(cd));
    });
}

int orc_multiply_spectra(int rank, const int64_t* dims, int m, const double* a, const double* b,
                         double* out) {
    return guard([&] {
        orc::Shape s(dims, rank, m);
        const size_t n = static_cast<size_t>(s.cells) * m * m;
        orc::Spectrum<double> A{s, {}}, B{s, {}};
        A.blocks.assign(reinterpret_cast<const cd*>(a), reinterpret_cast<const cd*>(a) + n);
        B.blocks.assign(reinterpret_cast<const cd*>(b), reinterpret_cast<const cd*>(b) + n);
        auto r = orc::multiply_spectra<double>(A, B);
        std::memcpy(out, r.blocks.data(), n * sizeof(cd));
    });
}

int orc_hadamard(int rank, const int64_t* dims, int m, const double* lam_blocks, const double* x,
                 double* out) {
    return guard([&] {
        orc::Shape s(dims, rank, m);
        const size_t nb = static_cast<size_t>(s.cells) * m * m;
        orc::Spectrum<double> L{s, {}};
        L.blocks.assign(reinterpret_cast<const cd*>(lam_blocks),
                        reinterpret_cast<const cd*>(lam_blocks) + nb);
        std::vector<cd> xv(reinterpret_cast<const cd*>(x), reinterpret_cast<const cd*>(x) + s.values());
        auto y = orc::hadamard<double>(L, xv, s);
        std::memcpy(out, y.data(), y.size() * sizeof(cd));
    });
}

int orc_step_periodic(int rank, const int64_t* dims, int fields, const double* a, int64_t ntaps,
                      const int64_t* offsets, const double* blocks, double* out) {
    return guard([&] {
        orc::Shape s(dims, rank, fields);
        orc::Kernel k = orc::kernel_from_arrays(rank, fields, ntaps, offsets, blocks);
        orc::step_periodic(a, s, k, out);
    });
}

int orc_evolve_periodic_naive(int rank, const int64_t* dims, int fields, const double* a0,
                              int64_t ntaps, const int64_t* offsets, const double* blocks,
                              uint64_t T, double* out) {
    return guard([&] {
        orc::Shape s(dims, rank, fields);
        orc::Kernel k = orc::kernel_from_arrays(rank, fields, ntaps, offsets, blocks);
        orc::evolve_naive(a0, s, k, T, out);
    });
}

int orc_dense_stencil_matrix(int rank, const int64_t* dims, int fields, int64_t ntaps,
                             const int64_t* offsets, const double* blocks, double* mat) {
    return guard([&] {
        orc::Shape s(dims, rank, fields);
        orc::Kernel k = orc::kernel_from_arrays(rank, fields, ntaps, offsets, blocks);
        orc::dense_matrix(s, k, mat);
    });
}

// modal_problem_periodic (proj/src/modal.cpp:99-145): initial grid and its
// double-double-amplified exact evolution after T steps (scalar fields).
int orc_modal_problem_periodic(int rank, const int64_t* dims, int64_t ntaps, const int64_t* offsets,
                               const double* blocks, uint64_t T, double* initial, double* reference) {
    return guard([&] {
        orc::Shape s(dims, rank, 1);
        orc::Kernel k = orc::kernel_from_arrays(rank, 1, ntaps, offsets, blocks);
        modal::problem_periodic(s, k, T, initial, reference);
    });
}

// SplitMix64 (proj/src/problem.cpp:222-228) and the U[-1,1) map
// (proj/src/problem.cpp:239-247); lo/hi select U[0,1) (0) or U[-1,1) (1).
void orc_splitmix_fill(uint64_t seed, int64_t n, int symmetric, double* out) {
    uint64_t st = seed;
    for (int64_t i = 0; i < n; ++i) {
        st += 0x9E3779B97F4A7C15ULL;
        uint64_t z = st;
        z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ULL;
        z = (z ^ (z >> 27)) * 0x94D049BB133111EBULL;
        z ^= z >> 31;
        const double u = static_cast<double>(z >> 11) * 0x1.0p-53;
        out[i] = symmetric ? 2.0 * u - 1.0 : u;
    }
}

}  // extern "C"
