// Host orchestration + C ABI of the B200 StencilFFT-P solver (include/fsx.h).
//
// Mirrors the reference periodic solver's contract (proj/src/periodic.cpp,
// proj/src/kernel.cpp:7-49): validation and error types, T == 0 short cut,
// stage timings accumulated with +=, NumericError on non-finite output (and
// on the imaginary residue where a complex pipeline exists).  The numerical
// work runs only on the GPU: there is no CPU fallback; a missing or failing
// device surfaces as FSX_ERR_CUDA.
//
// Three plan kinds:
//   1  fused R2C, rank 2/3, m = 1, pow2 dims: r2c rows -> strided passes ->
//      fused (axis-0 FFT, symbol^T, inverse FFT) -> strided passes -> c2r rows
//   2  1D, m in {1, 2}, pow2: four-step column pass -> fused row-pair pass
//      -> inverse column pass (real packing or two-for-one pairing)
//   3  general: complex promotion, per-axis passes (pow2 <= 8192 in one CTA,
//      pow2 up to 2^26 as a four-step split, other lengths by direct DFT),
//      m x m spectral kernel, inverse passes, real part + residue scan.
#include <array>
#include <chrono>
#include <cmath>
#include <cstdio>
#include <cstring>
#include <map>
#include <set>
#include <algorithm>
#include <memory>
#include <mutex>
#include <stdexcept>
#include <string>
#include <vector>

#include <cuda_runtime.h>
#include <dlfcn.h>
#include <nccl.h>
#include <type_traits>

#include "fsx.h"
#include "fsx_kernels.h"

namespace {

using fsx::i64;
using fsx::u64;

struct SpecErr : std::runtime_error {
    using std::runtime_error::runtime_error;
};
struct NumErr : std::runtime_error {
    using std::runtime_error::runtime_error;
};
struct CudaErr : std::runtime_error {
    cudaError_t code;
    CudaErr(cudaError_t c, const std::string& what)
        : std::runtime_error(what + ": " + cudaGetErrorString(c)), code(c) {}
};

thread_local std::string g_err;

#define FSX_CK(x)                                     \
    do {                                              \
        cudaError_t e_ = (x);                         \
        if (e_ != cudaSuccess) throw CudaErr(e_, #x); \
    } while (0)

bool is_pow2(i64 n) { return n > 0 && (n & (n - 1)) == 0; }
int ilog2(i64 n) {
    int r = 0;
    while ((i64(1) << r) < n) ++r;
    return r;
}

// ------------------------------------------------------------------ device buffers
struct DevBuf {
    void* p = nullptr;
    size_t bytes = 0;
    DevBuf() = default;
    DevBuf(const DevBuf&) = delete;
    DevBuf& operator=(const DevBuf&) = delete;
    ~DevBuf() { release(); }
    void release() {
        if (p) cudaFree(p);
        p = nullptr;
        bytes = 0;
    }
    void ensure(size_t b) {
        if (b == 0) b = 16;
        if (b <= bytes && p) return;
        release();
        cudaError_t e = cudaMalloc(&p, b);
        if (e != cudaSuccess) {
            cudaGetLastError();
            p = nullptr;
            throw CudaErr(e, "cudaMalloc(" + std::to_string(b) + " bytes)");
        }
        bytes = b;
    }
    template <class T>
    T* as() const { return reinterpret_cast<T*>(p); }
};

// ------------------------------------------------------------------ shapes and kernels
struct Shape {
    std::vector<i64> dims;
    int fields = 1;
    i64 cells = 1;
    int rank() const { return (int)dims.size(); }
    i64 values() const { return cells * fields; }
};

// GridShape invariants (proj/include/fftstencil/grid.hpp:21-45)
Shape parse_shape(const fsx_shape* s) {
    if (!s) throw SpecErr("GridShape: null shape");
    if (s->rank < 1 || s->rank > FSX_MAX_RANK) throw SpecErr("GridShape: need at least one dimension");
    if (s->fields < 1) throw SpecErr("GridShape: fields must be >= 1");
    Shape r;
    r.fields = s->fields;
    __int128 n = 1;
    for (int a = 0; a < s->rank; ++a) {
        if (s->dims[a] < 1) throw SpecErr("GridShape: every dimension must be >= 1");
        n *= s->dims[a];
        if (n * r.fields > (__int128)INT64_MAX) throw SpecErr("GridShape: total value count overflows");
        r.dims.push_back(s->dims[a]);
    }
    r.cells = (i64)n;
    return r;
}

struct Taps {
    int rank = 1, m = 1;
    std::map<std::vector<i64>, std::vector<double>> map;  // sorted offset -> m*m block
};

// StencilKernel + add_tap (proj/src/kernel.cpp:7-22): accumulate repeats,
// reject non-finite coefficients.
Taps parse_kernel(const fsx_kernel* k) {
    if (!k) throw SpecErr("StencilKernel: null kernel");
    if (k->rank < 1) throw SpecErr("StencilKernel: rank must be >= 1");
    if (k->fields < 1) throw SpecErr("StencilKernel: fields must be >= 1");
    if (k->ntaps < 0 || (k->ntaps > 0 && (!k->offsets || !k->blocks)))
        throw SpecErr("StencilKernel: bad tap arrays");
    Taps t;
    t.rank = k->rank;
    t.m = k->fields;
    const int mm = t.m * t.m;
    for (i64 j = 0; j < k->ntaps; ++j) {
        const double* b = k->blocks + j * mm;
        for (int i = 0; i < mm; ++i)
            if (!std::isfinite(b[i])) throw SpecErr("StencilKernel: non-finite coefficient");
        std::vector<i64> off(k->offsets + j * t.rank, k->offsets + (j + 1) * t.rank);
        auto it = t.map.find(off);
        if (it == t.map.end()) t.map.emplace(off, std::vector<double>(b, b + mm));
        else
            for (int i = 0; i < mm; ++i) it->second[i] += b[i];
    }
    return t;
}

// require_fits (proj/src/kernel.cpp:38-49)
void require_fits(const Taps& t, const Shape& s) {
    if (t.map.empty()) throw SpecErr("StencilKernel: at least one tap required");
    if (s.rank() != t.rank) throw SpecErr("StencilKernel: grid rank mismatch");
    if (s.fields != t.m) throw SpecErr("StencilKernel: grid field count mismatch");
    for (int a = 0; a < t.rank; ++a) {
        i64 reach = 0;
        for (const auto& kv : t.map) reach = std::max<i64>(reach, kv.first[a] < 0 ? -kv.first[a] : kv.first[a]);
        if (reach >= s.dims[a]) throw SpecErr("StencilKernel: tap offset exceeds dimension " + std::to_string(a));
    }
}

// ------------------------------------------------------------------ twiddle / phase tables
double2 expi_neg(i64 x, i64 n) {
    // exp(-2 pi i x / n) rounded from x87 long double
    const long double pi = 3.141592653589793238462643383279502884L;
    long double f = (long double)(x % n) / (long double)n;
    if (f > 0.5L) f -= 1.0L;
    const long double ang = -2.0L * pi * f;
    return make_double2((double)cosl(ang), (double)sinl(ang));
}

struct HostTable {
    std::vector<double2> lo, hi;
    int shift = 0;
    i64 mask = 0, n = 1;
};

HostTable make_phase(i64 n) {
    HostTable t;
    t.n = n;
    if (n <= 65536) {
        t.lo.resize(n);
        for (i64 x = 0; x < n; ++x) t.lo[x] = expi_neg(x, n);
        return t;
    }
    int bits = ilog2(n);
    int h = (bits + 1) / 2;
    const i64 lo_n = i64(1) << h;
    t.shift = h;
    t.mask = lo_n - 1;
    t.lo.resize(lo_n);
    for (i64 x = 0; x < lo_n; ++x) t.lo[x] = expi_neg(x, n);
    const i64 hi_n = (n + lo_n - 1) / lo_n;
    t.hi.resize(hi_n);
    for (i64 j = 0; j < hi_n; ++j) t.hi[j] = expi_neg(j * lo_n, n);
    return t;
}

// Packs several host tables into one device buffer; returns PhaseTables
// pointing into it.
// exp(-i pi x^2 / n) for x < n with x^2 reduced mod 2n exactly (proj/src/fft.cpp:20-25)
HostTable make_chirp(i64 n) {
    HostTable t;
    t.n = n;
    t.lo.resize(n);
    for (i64 x = 0; x < n; ++x) t.lo[x] = expi_neg((i64)(((__int128)x * x) % (2 * n)), 2 * n);
    return t;
}

struct TableSet {
    std::vector<double2> host;
    struct Ref {
        size_t lo, hi;
        int shift;
        i64 mask, n;
    };
    std::vector<Ref> refs;
    DevBuf dev;
    int add(const HostTable& t) {
        Ref r{host.size(), 0, t.shift, t.mask, t.n};
        host.insert(host.end(), t.lo.begin(), t.lo.end());
        r.hi = host.size();
        host.insert(host.end(), t.hi.begin(), t.hi.end());
        refs.push_back(r);
        return (int)refs.size() - 1;
    }
    void upload() {
        dev.ensure(host.size() * sizeof(double2));
        FSX_CK(cudaMemcpy(dev.p, host.data(), host.size() * sizeof(double2), cudaMemcpyHostToDevice));
    }
    fsx::PhaseTable get(int i) const {
        fsx::PhaseTable p;
        const Ref& r = refs[i];
        p.lo = dev.as<double2>() + r.lo;
        p.hi = dev.as<double2>() + r.hi;
        p.shift = r.shift;
        p.mask = r.mask;
        p.n = r.n;
        return p;
    }
};

// ------------------------------------------------------------------ plans
enum PlanKind { kFusedR2C = 1, kRowPair1D = 2, kGeneral = 3 };

struct AxisStep {
    int kind = 0;  // 0 pow2 pass, 1 direct DFT
    fsx::AxisGeom g;
    fsx::StepTwiddle tw;
    int table = -1;  // direct DFT phase table
};

struct GenAxis {
    i64 n = 1, n1 = 0, n2 = 0;  // split: n = n1 * n2 (n1 == 0: not split)
    int direct = 0;
    int table = -1;             // phase table for n
    // Bluestein (non-pow2 n > kBlueMin): convolution length P (pow2 >= 2n - 1)
    int blue = 0;
    i64 P = 0;
    int t_chirp = -1, t_P = -1;  // chirp e^(-i pi x^2 / n) (table lo = values), phase table of P
    i64 bhat_off = 0;            // filter spectrum offset in Plan::blue_bhat (complex elements)
};
constexpr i64 kBlueMin = 256;  // non-pow2 axes above this use Bluestein, below the direct DFT

struct Plan {
    int kind = 0;
    Shape full;                 // the caller's shape
    std::vector<i64> dims;      // squeezed dims (length-1 axes dropped)
    std::vector<int> axes;      // original axis index of each squeezed axis
    int m = 1;
    i64 cells = 1;
    TableSet tables;
    // kind 1
    i64 L = 0, M = 0, P = 0, rows = 0;
    // exact spectral cut / zero columns: column bounds per taps and the cut per T, cached (ColumnCut)
    std::shared_ptr<struct ColumnCut> cut;
    fsx::AxisGeom ax1, ax0;
    alignas(64) unsigned char map0[128], map1[128];  // CUtensorMaps for TMA column passes
    alignas(64) unsigned char map2[128];             // parity-split view (8192-point halves pass)
    bool tma0 = false, tma1 = false, halves = false;
    // kind 2
    i64 N1 = 1, N2 = 1, Mc = 0;
    i64 N1a = 0, N1b = 0;  // split column FFT (N1 > kMaxLine)
    int t_M = -1, t_wk = -1, t_N1 = -1;
    fsx::AxisGeom colg;
    // kind 3
    std::vector<GenAxis> gax;
    int gtab[fsx::kMaxRank];
    // workspaces
    DevBuf work;      // H (kind 1) / complex Z (kind 3)
    DevBuf d_in, d_out;
    DevBuf f_in, f_out;  // fp32 storage mode: host-API staging of float grids
    DevBuf taps_dev;  // general path tap arrays
    DevBuf blue_bhat, blue_buf;  // Bluestein filter spectra and [lines][P] workspace
    DevBuf qmax;      // implicit fused symbol: max |lamQ| (bits)
    std::vector<char> taps_host;
    int launches = 0;
    i64 alg_bytes = 0, fused_bytes = 0;
    const char* kernel = "";  // the dominant (fused) kernel of a solve, for measurement
    // batch > 1: that many grids of this shape stacked [batch][cells][m] and
    // solved together (fsx_solve_periodic_slabs): one launch per pass, the
    // batch as an outer dimension of every pass (plan 1 or plan 3)
    i64 batch = 1;
    int pins = 0;  // > 0: in use by a multi-plan call, exempt from cache eviction
    i64 sched_bytes = 0;  // bytes the launched pass schedule moves (0: = alg_bytes)
    // Cross-stream ordering of the plan's workspaces: `done` is recorded after
    // every enqueue on `last`; a solve on another stream first waits on it, so
    // two solves that share this plan's buffers never overlap on the GPU.
    cudaEvent_t done = nullptr;
    cudaStream_t last = nullptr;
    Plan() = default;
    Plan(const Plan&) = delete;
    Plan& operator=(const Plan&) = delete;
    ~Plan() {
        if (done) cudaEventDestroy(done);
    }
};

// Orders a solve on stream `st` after the plan's previous enqueue (on any stream).
void plan_enter(Plan& p, cudaStream_t st) {
    if (p.done && p.last != st) FSX_CK(cudaStreamWaitEvent(st, p.done, 0));
}
void plan_leave(Plan& p, cudaStream_t st) {
    if (!p.done) FSX_CK(cudaEventCreateWithFlags(&p.done, cudaEventDisableTiming));
    FSX_CK(cudaEventRecord(p.done, st));
    p.last = st;
}

// direct-stepping verifier buffers (per device)
struct NaiveBufs {
    DevBuf s0, s1, off, blk;
};

struct Device {
    // Serialises the host-side enqueueing of calls on THIS device; calls on
    // different devices run concurrently (the reference's solvers are safe to
    // call concurrently, proj/README.md:165-168).
    std::mutex mu;
    int ordinal = 0;
    cudaStream_t stream = nullptr;
    DevBuf tw_all;
    DevBuf tw_all_f;  // float2 copy (rounded once) for the fp32 mode's fused pass
    DevBuf flags;  // fsx::Flags of deferred device-mode / slab solves (read by fsx_device_check)
    DevBuf hflags; // fsx::Flags of synchronous host-pointer solves (checked and reset by each call)
    int dev_general = 0;  // a device-mode general-plan solve ran since the last fsx_device_check
    NaiveBufs naive;
    std::map<std::string, std::unique_ptr<Plan>> plans;
    cudaEvent_t ev[8];
    bool events = false;
    // pipelined batch solves: two lanes (stream + plan copy) keep one solve's
    // D2H, the next one's H2D and a third one's kernels in flight together
    cudaStream_t lanes[2] = {nullptr, nullptr};
    cudaEvent_t lane_ev[2];
    DevBuf bflags;  // per-solve Flags of a batch
};

std::mutex g_map_mu;  // guards g_devices (lookup and creation only)
std::map<int, std::unique_ptr<Device>> g_devices;

Device& device_create(int ordinal);

// The device object for an ordinal (created on first use), with that device
// selected on the calling thread.
Device& device_for(int ordinal) {
    Device* d = nullptr;
    {
        std::lock_guard<std::mutex> lk(g_map_mu);
        auto it = g_devices.find(ordinal);
        d = it != g_devices.end() ? it->second.get() : &device_create(ordinal);
    }
    FSX_CK(cudaSetDevice(ordinal));
    return *d;
}

// RAII: the device selected and its mutex held for one API call.
struct DevLock {
    Device& dev;
    std::unique_lock<std::mutex> lk;
    explicit DevLock(int ordinal) : dev(device_for(ordinal)), lk(dev.mu) {}
};

Device& device_create(int ordinal) {
    int count = 0;
    cudaError_t e = cudaGetDeviceCount(&count);
    if (e != cudaSuccess || count == 0) {
        cudaGetLastError();
        throw CudaErr(e == cudaSuccess ? cudaErrorNoDevice : e, "fsx: no CUDA device (the GPU path has no CPU fallback)");
    }
    if (ordinal < 0 || ordinal >= count) throw SpecErr("fsx: device ordinal out of range");
    FSX_CK(cudaSetDevice(ordinal));
    auto d = std::make_unique<Device>();
    d->ordinal = ordinal;
    FSX_CK(cudaStreamCreateWithFlags(&d->stream, cudaStreamNonBlocking));
    // pow2 line twiddles: tw_all[N + x] = exp(-2 pi i x / N)
    std::vector<double2> tw(fsx::kTwAllSize, make_double2(0, 0));
    for (i64 N = 1; N <= fsx::kMaxTwPow2; N <<= 1)
        for (i64 x = 0; x < N; ++x) tw[N + x] = expi_neg(x, N);
    // per-pass gathered copies for LineFFT<N> (fsx_kernels.h, kPassTabBase)
    for (i64 N = 16; N <= fsx::kMaxLine; N <<= 1) {
        const int logn = ilog2(N), p16 = logn / 4, rem = logn % 4, npass = p16 + (rem > 0 ? 1 : 0);
        i64 Ns = 1;
        for (int S = 0; S < npass; ++S) {
            const i64 r = S < p16 ? 16 : i64(1) << rem;
            if (S > 0)
                for (i64 u = 1; u < r; ++u)
                    for (i64 k = 0; k < Ns; ++k)
                        tw[fsx::kPassTabBase + 16 * N + 16 * Ns + (u - 1) * Ns + k] = tw[N + u * k * (N / (Ns * r))];
            Ns *= r;
        }
    }
    d->tw_all.ensure(tw.size() * sizeof(double2));
    FSX_CK(cudaMemcpy(d->tw_all.p, tw.data(), tw.size() * sizeof(double2), cudaMemcpyHostToDevice));
    {
        std::vector<float2> twf(tw.size());
        for (size_t i = 0; i < tw.size(); ++i) twf[i] = make_float2((float)tw[i].x, (float)tw[i].y);
        d->tw_all_f.ensure(twf.size() * sizeof(float2));
        FSX_CK(cudaMemcpy(d->tw_all_f.p, twf.data(), twf.size() * sizeof(float2), cudaMemcpyHostToDevice));
    }
    d->flags.ensure(sizeof(fsx::Flags));
    FSX_CK(cudaMemset(d->flags.p, 0, sizeof(fsx::Flags)));
    d->hflags.ensure(sizeof(fsx::Flags));
    FSX_CK(cudaMemset(d->hflags.p, 0, sizeof(fsx::Flags)));
    for (auto& e2 : d->ev) FSX_CK(cudaEventCreate(&e2));
    d->events = true;
    auto& ref = *d;
    g_devices.emplace(ordinal, std::move(d));
    return ref;
}

// FSX_TMA=0 keeps the strided passes on per-thread LDG/STG (A/B measurements).
bool tma_enabled() {
    const char* e = getenv("FSX_TMA");
    return !(e && e[0] == '0');
}

// Splits a pow2 length into n1 * n2 with both <= kMaxLine.
bool split_pow2(i64 n, i64& n1, i64& n2) {
    const int b = ilog2(n);
    if (b > 2 * ilog2(fsx::kMaxLine)) return false;
    const int b2 = std::min(ilog2(fsx::kMaxLine), (b + 1) / 2);
    n2 = i64(1) << b2;
    n1 = n / n2;
    return n1 <= fsx::kMaxLine;
}

int choose_kind(const Plan& p, const Taps& taps, int force_general) {
    if (force_general) return kGeneral;
    const int r = (int)p.dims.size();
    for (i64 d : p.dims)
        if (!is_pow2(d)) return kGeneral;
    if ((i64)taps.map.size() > fsx::kMaxFusedTaps) return kGeneral;
    if (p.m == 1 && (r == 2 || r == 3)) {
        const i64 L = p.dims[r - 1];
        if (L < 16 || L > 2 * fsx::kMaxLine) return kGeneral;
        // the fused axis-0 kernels are instantiated for 8 <= n0 <= 8192
        if (p.dims[0] < 8) return kGeneral;
        for (int a = 0; a + 1 < r; ++a)
            if (p.dims[a] < 2 || p.dims[a] > fsx::kMaxLine) return kGeneral;
        std::map<i64, int> groups;
        for (const auto& kv : taps.map) groups[kv.first[p.axes[0]]] = 1;
        if ((int)groups.size() > fsx::kMaxGroups) return kGeneral;
        return kFusedR2C;
    }
    if (r == 1 && (p.m == 1 || p.m == 2)) {
        const i64 n = p.dims[0];
        const i64 Mc = p.m == 1 ? n / 2 : n;
        if (Mc < 16) return kGeneral;
        if (Mc <= 256) return kRowPair1D;
        const int b = ilog2(Mc);
        const int b2 = std::min(12, (b + 1) / 2);
        // column FFT of N1 = 2^(b-b2): one CTA up to 8192, a 2-level split up to 8192^2
        if (b - b2 > 2 * ilog2(fsx::kMaxLine)) return kGeneral;
        return kRowPair1D;
    }
    return kGeneral;
}

std::string plan_key(const Shape& s, int kind_hint) {
    std::string k = std::to_string(s.fields) + "|" + std::to_string(kind_hint);
    for (i64 d : s.dims) k += ":" + std::to_string(d);
    return k;
}

// Batched pow2 FFT of `lines` contiguous lines of length P (P <= 2^26; above
// kMaxLine a four-step split whose frequency order is transposed -- the
// Bluestein filter spectrum is computed with the same split, so the pointwise
// product and the inverse split undo it).
void fft_lines(const Plan& p, const Device& dev, double2* buf, i64 lines, i64 P, int t_P, int sign, cudaStream_t st) {
    const double2* tw = dev.tw_all.as<double2>();
    fsx::StepTwiddle none;
    if (P <= fsx::kMaxLine) {
        const fsx::AxisGeom g{P, 1, lines, P, 1};
        FSX_CK(fsx::launch_axis_pow2(buf, buf, g, sign, none, tw, st));
        return;
    }
    i64 p1, p2;
    if (!split_pow2(P, p1, p2)) throw SpecErr("fsx: Bluestein length beyond 2^26");
    const fsx::AxisGeom g1{p1, p2, lines, P, p2};
    const fsx::AxisGeom g2{p2, 1, lines * p1, p2, 1};
    fsx::StepTwiddle t1;
    t1.col_div = 1;
    t1.tab = p.tables.get(t_P);
    if (sign < 0) {
        t1.mode = 1;
        FSX_CK(fsx::launch_axis_pow2(buf, buf, g1, sign, t1, tw, st));
        FSX_CK(fsx::launch_axis_pow2(buf, buf, g2, sign, none, tw, st));
    } else {
        t1.mode = 2;
        FSX_CK(fsx::launch_axis_pow2(buf, buf, g2, sign, none, tw, st));
        FSX_CK(fsx::launch_axis_pow2(buf, buf, g1, sign, t1, tw, st));
    }
}

// Filter spectra Bhat = FFT_P(b), b[x] = conj(chirp[x]) for |x| < n (wrapped),
// and the [lines][P] workspace of the general plan's Bluestein axes.
void setup_bluestein(Plan& p, Device& dev) {
    i64 total = 0, work = 0;
    for (auto& ga : p.gax)
        if (ga.blue) {
            ga.bhat_off = total;
            total += ga.P;
            work = std::max<i64>(work, p.cells * p.m * p.batch / ga.n * ga.P);
        }
    if (!total) return;
    p.blue_bhat.ensure((size_t)total * sizeof(double2));
    p.blue_buf.ensure((size_t)work * sizeof(double2));
    for (const auto& ga : p.gax) {
        if (!ga.blue) continue;
        std::vector<double2> b((size_t)ga.P, make_double2(0, 0));
        const HostTable ch = make_chirp(ga.n);
        for (i64 x = 0; x < ga.n; ++x) {
            const double2 c = make_double2(ch.lo[x].x, -ch.lo[x].y);
            b[x] = c;
            if (x) b[ga.P - x] = c;
        }
        double2* dst = p.blue_bhat.as<double2>() + ga.bhat_off;
        FSX_CK(cudaMemcpy(dst, b.data(), b.size() * sizeof(double2), cudaMemcpyHostToDevice));
        fft_lines(p, dev, dst, 1, ga.P, ga.t_P, -1, dev.stream);
    }
    FSX_CK(cudaStreamSynchronize(dev.stream));
}

// lane > 0: an independent copy of the plan (own workspaces and tensor maps)
// for the pipelined batch solve, which keeps two solves in flight.
Plan& get_plan(Device& dev, const Shape& s, const Taps& taps, int force_general, int lane = 0, i64 batch = 1) {
    // squeeze length-1 axes (their offsets are 0 by require_fits)
    Plan probe;
    probe.full = s;
    probe.m = s.fields;
    for (int a = 0; a < s.rank(); ++a)
        if (s.dims[a] > 1) {
            probe.dims.push_back(s.dims[a]);
            probe.axes.push_back(a);
        }
    if (probe.dims.empty()) {
        probe.dims.push_back(1);
        probe.axes.push_back(0);
    }
    int kind = choose_kind(probe, taps, force_general);
    if (batch > 1 && kind == kRowPair1D) kind = kGeneral;  // stacked 1D grids: the general passes
    const std::string base = plan_key(s, kind) + (batch > 1 ? "|b" + std::to_string(batch) : "");
    const std::string key = lane ? base + "|lane" + std::to_string(lane) : base;
    auto it = dev.plans.find(key);
    if (it != dev.plans.end()) return *it->second;
    if (dev.plans.size() >= 8) {  // bounded cache; keep this shape's other lanes (a batch holds them) and pinned plans
        for (auto e = dev.plans.begin(); e != dev.plans.end();)
            e = (e->first.rfind(base, 0) == 0 || e->second->pins > 0) ? std::next(e) : dev.plans.erase(e);
    }

    auto p = std::make_unique<Plan>();
    p->full = probe.full;
    p->dims = probe.dims;
    p->axes = probe.axes;
    p->m = probe.m;
    p->kind = kind;
    p->cells = s.cells;
    p->batch = batch;
    const int r = (int)p->dims.size();
    const i64 R = s.values() * 8 * batch;  // real bytes
    if (kind == kFusedR2C) {
        p->L = p->dims[r - 1];
        p->M = p->L / 2;
        p->P = p->M + 8;
        p->rows = s.cells / p->L * batch;
        p->work.ensure((size_t)p->rows * p->P * sizeof(double2));
        const i64 plane = (r == 3) ? p->dims[1] * p->P : p->P;
        if (r == 3) {
            p->ax1.n = p->dims[1];
            p->ax1.inner = p->P;
            p->ax1.outer = p->dims[0] * batch;
            p->ax1.block = p->dims[1] * p->P;
            p->ax1.ncols = p->M + 1;
        }
        p->ax0.n = p->dims[0];
        p->ax0.inner = plane;
        p->ax0.outer = batch;
        p->ax0.block = p->dims[0] * plane;
        p->ax0.ncols = (r == 3) ? plane : p->M + 1;
        if (tma_enabled()) {
            p->tma0 = fsx::tma_cols_ok(p->ax0.n) && fsx::make_cols_tensor_map(p->map0, p->work.p, p->ax0) == 0;
            p->tma1 = r == 3 && fsx::tma_cols_ok(p->ax1.n) && fsx::make_cols_tensor_map(p->map1, p->work.p, p->ax1) == 0;
            p->halves = fsx::halves_ok(p->ax0) && fsx::make_cols_tensor_map_par(p->map2, p->work.p, p->ax0) == 0;
        }
        const i64 H = p->rows * (p->M + 1) * 16;
        p->fused_bytes = 2 * H;
        p->alg_bytes = 2 * R + (r == 3 ? 8 : 4) * H;
        p->launches = (r == 3) ? 5 : 3;
    } else if (kind == kRowPair1D) {
        const i64 n = p->dims[0];
        p->Mc = p->m == 1 ? n / 2 : n;
        if (p->Mc <= 256) {
            p->N1 = 1;
            p->N2 = p->Mc;
        } else {
            const int b = ilog2(p->Mc);
            int b2 = std::min(12, (b + 1) / 2);
            // FSX_N2LOG: row length 2^b2 of the four-step split (A/B of the split of small grids)
            if (const char* e = getenv("FSX_N2LOG")) b2 = std::max(8, std::min(std::min(12, b - 1), atoi(e)));
            p->N2 = i64(1) << b2;
            p->N1 = p->Mc / p->N2;
        }
        p->t_M = p->tables.add(make_phase(p->Mc));
        p->t_wk = p->tables.add(make_phase(p->m == 1 ? n : p->Mc));
        p->colg.n = p->N1;
        p->colg.inner = p->N2;
        p->colg.outer = 1;
        p->colg.block = p->Mc;
        p->colg.ncols = p->N2;
        int col_passes = p->N1 > 1 ? 1 : 0;
        // FSX_COLSPLIT lowers the split threshold (tests exercise the 2^26 path small)
        const char* cs = getenv("FSX_COLSPLIT");
        const i64 max_col = cs ? std::max<i64>(4, atoll(cs)) : fsx::kMaxLine;
        if (p->N1 > max_col) {
            // the column FFT itself as a four-step split N1 = N1a x N1b
            const int b1 = ilog2(p->N1);
            p->N1b = i64(1) << ((b1 + 1) / 2);
            p->N1a = p->N1 / p->N1b;
            p->t_N1 = p->tables.add(make_phase(p->N1));
            col_passes = 2;
        }
        p->tables.upload();
        p->fused_bytes = 2 * R;
        // the minimal 1D four-step schedule is 3 passes (column,
        // row-pair, inverse column) = 6R; a split column FFT (N1 > 8192, e.g.
        // cfg5) launches 5 passes = 10R (sched_bytes)
        p->alg_bytes = 6 * R;
        p->sched_bytes = (i64)(2 + 4 * col_passes) * R;
        p->launches = 2 * col_passes + 1 + 1;
    } else {
        // general: complex Z of cells * m (block kernels instantiated for m <= 8)
        if (p->m > 8) throw SpecErr("fsx: more than 8 fields per cell is not supported on the GPU path");
        p->work.ensure((size_t)s.values() * batch * sizeof(double2));
        i64 nl = 0;
        for (int a = 0; a < r; ++a) {
            GenAxis ga;
            ga.n = p->dims[a];
            if (ga.n > 1) {
                if (is_pow2(ga.n) && ga.n <= fsx::kMaxLine) {
                    nl += 2;
                } else if (is_pow2(ga.n)) {
                    if (!split_pow2(ga.n, ga.n1, ga.n2))
                        throw SpecErr("fsx: axis length " + std::to_string(ga.n) + " exceeds the GPU path limit (2^26)");
                    nl += 4;
                } else if (ga.n <= kBlueMin) {
                    ga.direct = 1;
                    nl += 2;
                } else {
                    ga.blue = 1;
                    ga.P = 1;
                    while (ga.P < 2 * ga.n - 1) ga.P <<= 1;
                    i64 q1, q2;
                    if (ga.P > fsx::kMaxLine && !split_pow2(ga.P, q1, q2))
                        throw SpecErr("fsx: axis length " + std::to_string(ga.n) + " exceeds the GPU path limit (Bluestein 2^26)");
                    ga.t_chirp = p->tables.add(make_chirp(ga.n));
                    if (ga.P > fsx::kMaxLine) ga.t_P = p->tables.add(make_phase(ga.P));
                    nl += 8;
                }
            }
            ga.table = p->tables.add(make_phase(ga.n));
            p->gax.push_back(ga);
        }
        p->tables.upload();
        setup_bluestein(*p, dev);
        p->launches = (int)nl + 3;
        const i64 Z = s.values() * 16 * batch;
        p->fused_bytes = 2 * Z;
        p->alg_bytes = R + Z + (nl) * 2 * Z / 1 + 2 * Z + Z + R;
    }
    auto& ref = *p;
    dev.plans.emplace(key, std::move(p));
    return ref;
}

// ------------------------------------------------------------------ symbol setup
// Taps with c(o) == c(-o) for every offset give a real symbol
// sum_o c(o) cos(2 pi k.o / n) (blocks compared entry by entry, exactly).
bool symmetric_taps(const Taps& taps) {
    for (const auto& kv : taps.map) {
        std::vector<i64> neg(kv.first.size());
        for (size_t a = 0; a < neg.size(); ++a) neg[a] = -kv.first[a];
        auto it = taps.map.find(neg);
        if (it == taps.map.end() || it->second != kv.second) return false;
    }
    return true;
}

fsx::FusedSymbol fused_symbol(const Plan& p, const Taps& taps, u64 T, const Taps* q = nullptr,
                              const unsigned long long* qmax_bits = nullptr) {
    fsx::FusedSymbol s;
    const int r = (int)p.dims.size();
    s.rank = r;
    s.n0 = p.dims[0];
    s.n1 = r == 3 ? p.dims[1] : 1;
    s.L = p.L;
    s.P = p.P;
    s.M = p.M;
    s.T = T;
    // |lam|^2 < neg_mag2  <=>  |lam|^T < 2^-1100 (0 in fp64 for T = 1: never)
    s.neg_mag2 = std::exp2(-2200.0 / (double)T);
    s.scale = 1.0 / (double)p.cells;
    // groups keyed by (tap set, axis-0 offset): set 0 = S, set 1 = Q (implicit)
    std::map<std::pair<int, i64>, int> gid;
    int j = 0;
    auto add_set = [&](const Taps& t, int set) {
        for (const auto& kv : t.map) {
            const auto& off = kv.first;
            const std::pair<int, i64> key{set, off[p.axes[0]]};
            auto it = gid.find(key);
            int g;
            if (it == gid.end()) {
                g = (int)gid.size();
                gid.emplace(key, g);
                s.group_off[g] = (int)key.second;
                s.group_set[g] = set;
            } else {
                g = it->second;
            }
            s.tap_group[j] = g;
            s.tap_o1[j] = r == 3 ? (int)off[p.axes[1]] : 0;
            s.tap_olast[j] = (int)off[p.axes[r - 1]];
            s.tap_c[j] = kv.second[0];
            ++j;
        }
    };
    add_set(taps, 0);
    if (q) {
        add_set(*q, 1);
        s.implicit = 1;
        s.qmax_bits = qmax_bits;
    }
    s.ntaps = j;
    s.ngroups = (int)gid.size();
    s.real = symmetric_taps(taps) && (!q || symmetric_taps(*q)) ? 1 : 0;
    // +-og partner groups of one tap set (complex symbols share their phase reads)
    for (int g = 0; g < s.ngroups; ++g) {
        if (s.group_off[g] <= 0) continue;
        for (int h = 0; h < s.ngroups; ++h)
            if (s.group_off[h] == -s.group_off[g] && s.group_set[h] == s.group_set[g]) {
                s.group_partner[g] = 1 + h;
                s.group_partner[h] = -1;
            }
    }
    return s;
}

// Exact spectral cut (2D fused plan, explicit scalar solve).  The fused pass
// sets an element's multiplier to exactly 0 when |lam|^2 < neg_mag2 =
// 2^(-2200/T) (|lam|^T < 2^-1100: below every representable contribution,
// where the reference's own repeated squaring underflows).  With taps grouped
// by their axis-0 offset O_g, lam(k0, kx) = sum_g A_g(kx) e^{2 pi i k0 O_g / n0},
// so |lam(k0, kx)| <= B(kx) = sum_g |A_g(kx)| for every k0: a column with
// B(kx)^2 below neg_mag2 (with a 1e-9 relative margin for the device's
// rounding of lam) is exactly 0 after the fused pass in the full solve.
// Returns the largest column that is not provably 0 (>= 0, so column 0 -- and
// with it a non-finite input -- always goes through), or -1 when the cut does
// not apply.  Columns above it are neither stored by the forward rows, nor
// transformed, nor read by the inverse rows (which take them as 0).
// The bounds B(kx)^2 do not depend on T, so they are computed once per (plan, taps) --
// exact integer phase reduction, one cos/sin pair per distinct last-axis offset and column --
// and a new T costs only the threshold scan (a caller stepping T pays microseconds, not the
// ~M trigonometric evaluations, on every solve).
bool column_cut_applies(const Plan& p) {
    return p.kind == kFusedR2C && p.dims.size() == 2 && p.m == 1 && fsx::rows_f32_ok(p.L);
}

std::vector<double> column_bounds_sq(const Plan& p, const Taps& taps) {
    std::map<i64, std::vector<std::pair<i64, double>>> groups;  // O_g -> (o_last, c)
    std::vector<i64> offs;                                      // distinct o_last
    for (const auto& kv : taps.map) {
        const i64 ol = kv.first[p.axes[1]];
        groups[kv.first[p.axes[0]]].push_back({ol, kv.second[0]});
        if (std::find(offs.begin(), offs.end(), ol) == offs.end()) offs.push_back(ol);
    }
    // each group's taps as (index into offs, c)
    std::vector<std::vector<std::pair<size_t, double>>> gs;
    for (const auto& g : groups) {
        gs.emplace_back();
        for (const auto& oc : g.second)
            gs.back().push_back({(size_t)(std::find(offs.begin(), offs.end(), oc.first) - offs.begin()), oc.second});
    }
    const double w = 2.0 * 3.14159265358979323846 / (double)p.L;
    std::vector<double> bsq((size_t)p.M + 1, 0.0), cs(offs.size()), sn(offs.size());
    for (i64 kx = 0; kx <= p.M; ++kx) {
        for (size_t a = 0; a < offs.size(); ++a) {
            const i64 ph = ((kx * offs[a]) % p.L + p.L) % p.L;  // exact integer phase
            cs[a] = std::cos(w * (double)ph);
            sn[a] = std::sin(w * (double)ph);
        }
        double B = 0.0;
        for (const auto& g : gs) {
            double re = 0.0, im = 0.0;
            for (const auto& oc : g) {
                re += oc.second * cs[oc.first];
                im += oc.second * sn[oc.first];
            }
            B += std::sqrt(re * re + im * im);
        }
        bsq[(size_t)kx] = B * B;
    }
    return bsq;
}

i64 cut_from_bounds(const std::vector<double>& bsq, u64 T) {
    const double neg = std::exp2(-2200.0 / (double)T);
    if (!(neg > 0.0)) return -1;
    const double thr = neg * (1.0 - 1e-9);
    for (i64 kx = (i64)bsq.size() - 1; kx > 0; --kx)
        if (bsq[(size_t)kx] >= thr) return kx;
    return 0;
}

// cache of the above: bounds per taps, cut per T
struct ColumnCut {
    bool taps_valid = false, t_valid = false;
    Taps taps;
    std::vector<double> bsq;
    u64 T = 0;
    i64 kcut = -1;
    i64 get(const Plan& p, const Taps& tp, u64 t) {
        if (!column_cut_applies(p)) return -1;
        if (!(taps_valid && taps.map == tp.map)) {
            bsq = column_bounds_sq(p, tp);
            taps = tp;
            taps_valid = true;
            t_valid = false;
        }
        if (!(t_valid && T == t)) {
            kcut = cut_from_bounds(bsq, t);
            T = t;
            t_valid = true;
        }
        return kcut;
    }
};

// FSX_ZEROCOL=0: the fused pass evaluates the symbol of every column (A/B and the bitwise
// test; read per solve so a test can flip it in-process)
static bool zero_columns_enabled() {
    const char* e = getenv("FSX_ZEROCOL");
    return !e || atoi(e) != 0;
}

i64 plan_kcut(Plan& p, const Taps& taps, u64 T) {
    if (!p.cut) p.cut = std::make_shared<ColumnCut>();
    return p.cut->get(p, taps, T);
}

// The implicit solve fuses into plan 1 when the symbol is real and the fused
// pass is the TMA column kernel that precomputes its multipliers (N <= 4096).
bool implicit_fusable(const Plan& p, const Taps& s, const Taps& q) {
    if (p.kind != kFusedR2C || !p.tma0 || p.halves || p.ax0.n > 4096) return false;
    if (!symmetric_taps(s) || !symmetric_taps(q)) return false;
    if ((i64)(s.map.size() + q.map.size()) > fsx::kMaxFusedTaps) return false;
    std::set<std::pair<int, i64>> g;
    for (const auto& kv : s.map) g.insert({0, kv.first[p.axes[0]]});
    for (const auto& kv : q.map) g.insert({1, kv.first[p.axes[0]]});
    return (int)g.size() <= fsx::kMaxGroups;
}

fsx::RowPairArgs rowpair_args(const Plan& p, const Taps& taps, u64 T, double2* z, const Device& dev) {
    fsx::RowPairArgs a;
    a.z = z;
    a.N1 = p.N1;
    a.N2 = p.N2;
    a.mode = p.m == 1 ? 0 : 1;
    a.tw_all = dev.tw_all.as<double2>();
    a.wk = p.tables.get(p.t_wk);
    a.T = T;
    a.neg_mag2 = std::exp2(-2200.0 / (double)T);
    a.scale = 1.0 / (double)(p.m == 1 ? p.dims[0] : p.Mc);
    int j = 0;
    for (const auto& kv : taps.map) {
        a.tap_off[j] = (int)kv.first[p.axes[0]];
        for (int i = 0; i < p.m * p.m; ++i) a.tap_b[j][i] = kv.second[i];
        ++j;
    }
    a.ntaps = j;
    a.real = symmetric_taps(taps) ? 1 : 0;
    if (a.real && a.mode == 1) {
        // real block symbol B(0) + sum_{o>0} (B(o) + B(-o)) cos(2 pi k o / N): the
        // +-o taps folded into one cosine term each (one phase read and one
        // fma per entry per |o|; cfg5's three taps become two)
        std::map<int, std::array<double, 4>> fold;
        for (int t = 0; t < a.ntaps; ++t) {
            auto& b = fold[a.tap_off[t] < 0 ? -a.tap_off[t] : a.tap_off[t]];
            for (int i = 0; i < 4; ++i) b[i] += a.tap_b[t][i];
        }
        j = 0;
        for (const auto& kv : fold) {
            a.tap_off[j] = kv.first;
            for (int i = 0; i < 4; ++i) a.tap_b[j][i] = kv.second[i];
            ++j;
        }
        a.ntaps = j;
    }
    a.row_split = p.N1b;
    return a;
}

// General symbol: uploads the (squeezed) tap arrays into the plan.
fsx::GeneralSymbol general_symbol(Plan& p, const Taps& taps, const Taps* q, u64 T, cudaStream_t st) {
    fsx::GeneralSymbol s;
    const int r = (int)p.dims.size();
    s.rank = r;
    s.m = p.m;
    s.cells = p.cells;
    for (int a = 0; a < r; ++a) {
        s.dims[a] = p.dims[a];
        s.split[a] = p.gax[a].n1;
        s.tab[a] = p.tables.get(p.gax[a].table);
    }
    s.T = T;
    s.scale = 1.0 / (double)p.cells;
    s.batch = p.batch;
    const int mm = p.m * p.m;
    auto pack = [&](const Taps& t, std::vector<long long>& off, std::vector<double>& blk) {
        for (const auto& kv : t.map) {
            for (int a = 0; a < r; ++a) off.push_back(kv.first[p.axes[a]]);
            blk.insert(blk.end(), kv.second.begin(), kv.second.end());
        }
    };
    std::vector<long long> off, offq;
    std::vector<double> blk, blkq;
    pack(taps, off, blk);
    if (q) pack(*q, offq, blkq);
    const size_t b_off = off.size() * 8, b_blk = blk.size() * 8, b_offq = offq.size() * 8, b_blkq = blkq.size() * 8;
    const size_t total = b_off + b_blk + b_offq + b_blkq + 64;
    p.taps_host.assign(total, 0);
    std::memcpy(p.taps_host.data(), off.data(), b_off);
    std::memcpy(p.taps_host.data() + b_off, blk.data(), b_blk);
    std::memcpy(p.taps_host.data() + b_off + b_blk, offq.data(), b_offq);
    std::memcpy(p.taps_host.data() + b_off + b_blk + b_offq, blkq.data(), b_blkq);
    p.taps_dev.ensure(total);
    FSX_CK(cudaMemcpyAsync(p.taps_dev.p, p.taps_host.data(), total, cudaMemcpyHostToDevice, st));
    char* base = p.taps_dev.as<char>();
    s.ntaps = (int)taps.map.size();
    s.offsets = reinterpret_cast<const long long*>(base);
    s.blocks = reinterpret_cast<const double*>(base + b_off);
    if (q) {
        s.implicit = 1;
        s.ntaps_q = (int)q->map.size();
        s.offsets_q = reinterpret_cast<const long long*>(base + b_off + b_blk);
        s.blocks_q = reinterpret_cast<const double*>(base + b_off + b_blk + b_offq);
        s.qmax = reinterpret_cast<const double*>(base + total - 8);
    }
    (void)mm;
    return s;
}

// ------------------------------------------------------------------ general axis passes
void general_axes(Plan& p, const Device& dev, double2* Z, bool inverse, cudaStream_t st) {
    const int r = (int)p.dims.size();
    const int sign = inverse ? +1 : -1;
    auto run_axis = [&](int a) {
        const GenAxis& ga = p.gax[a];
        if (ga.n <= 1) return;
        i64 inner = p.m, outer = p.batch;  // stacked grids are outer blocks of every axis
        for (int b = a + 1; b < r; ++b) inner *= p.dims[b];
        for (int b = 0; b < a; ++b) outer *= p.dims[b];
        fsx::StepTwiddle none;
        if (ga.blue) {
            // proj/src/fft.cpp:103-139; inverse as conj(forward(conj x)) (fft.cpp:151-154)
            const fsx::AxisGeom g{ga.n, inner, outer, ga.n * inner, inner};
            const i64 lines = outer * inner;
            double2* buf = p.blue_buf.as<double2>();
            const double2* chirp = p.tables.get(ga.t_chirp).lo;
            const int cj = inverse ? 1 : 0;
            FSX_CK(fsx::launch_blue_pre(Z, buf, g, ga.P, chirp, cj, st));
            fft_lines(p, dev, buf, lines, ga.P, ga.t_P, -1, st);
            FSX_CK(fsx::launch_blue_mul(buf, lines, ga.P, p.blue_bhat.as<double2>() + ga.bhat_off, st));
            fft_lines(p, dev, buf, lines, ga.P, ga.t_P, +1, st);
            FSX_CK(fsx::launch_blue_post(buf, Z, g, ga.P, chirp, 1.0 / (double)ga.P, cj, st));
        } else if (ga.direct) {
            fsx::AxisGeom g{ga.n, inner, outer, ga.n * inner, inner};
            FSX_CK(fsx::launch_axis_direct(Z, Z, g, sign, p.tables.get(ga.table), st));
        } else if (!ga.n1) {
            fsx::AxisGeom g{ga.n, inner, outer, ga.n * inner, inner};
            FSX_CK(fsx::launch_axis_pow2(Z, Z, g, sign, none, dev.tw_all.as<double2>(), st));
        } else {
            // four-step split: [outer][n1][n2][inner]
            fsx::AxisGeom g1{ga.n1, ga.n2 * inner, outer, ga.n * inner, ga.n2 * inner};
            fsx::AxisGeom g2{ga.n2, inner, outer * ga.n1, ga.n2 * inner, inner};
            fsx::StepTwiddle tw;
            tw.col_div = inner;
            tw.tab = p.tables.get(ga.table);
            if (!inverse) {
                tw.mode = 1;
                FSX_CK(fsx::launch_axis_pow2(Z, Z, g1, sign, tw, dev.tw_all.as<double2>(), st));
                FSX_CK(fsx::launch_axis_pow2(Z, Z, g2, sign, none, dev.tw_all.as<double2>(), st));
            } else {
                tw.mode = 2;
                FSX_CK(fsx::launch_axis_pow2(Z, Z, g2, sign, none, dev.tw_all.as<double2>(), st));
                FSX_CK(fsx::launch_axis_pow2(Z, Z, g1, sign, tw, dev.tw_all.as<double2>(), st));
            }
        }
    };
    if (!inverse)
        for (int a = 0; a < r; ++a) run_axis(a);
    else
        for (int a = r - 1; a >= 0; --a) run_axis(a);
}

// ------------------------------------------------------------------ solve
struct Stamps {
    Device* dev;
    bool on;
    cudaStream_t st;
    int n = 0;
    void mark() {
        if (on) FSX_CK(cudaEventRecord(dev->ev[n++], st));
    }
};

// Runs one solve on device pointers; stage boundaries are stamped into
// ev[0..3] when timings are requested.
// fin / fout (fp32 storage mode, plan 1 only): the row passes read and write
// floats directly instead of d_a0 / d_out.
void run_plan(Plan& p, Device& dev, const Taps& taps, const Taps* q, u64 T, const double* d_a0, double* d_out,
              cudaStream_t st, Stamps& sp, fsx::Flags* flags_at = nullptr, const float* fin = nullptr,
              float* fout = nullptr, bool cut = false) {
    fsx::Flags* flags = flags_at ? flags_at : dev.flags.as<fsx::Flags>();
    const double2* tw = dev.tw_all.as<double2>();
    const int r = (int)p.dims.size();
    sp.mark();
    if (p.kind == kFusedR2C) {
        double2* H = p.work.as<double2>();
        fsx::RowLayout lay{p.P, 0, p.rows};
        const i64 kcut = (cut && !q) ? plan_kcut(p, taps, T) : -1;
        lay.kcut = kcut;
        fsx::AxisGeom ax0 = p.ax0;  // the fused pass covers columns 0..kcut only
        if (kcut >= 0) ax0.ncols = kcut + 1;
        // fp32 mode: fp32 arithmetic in the row FFTs too (FSX_F32_COMPUTE, real symbols as the fused pass)
        const bool f32rows = (fin || fout) && !q && symmetric_taps(taps) && fsx::f32_compute_enabled();
        const float2* twf = f32rows ? dev.tw_all_f.as<float2>() : nullptr;
        if (fin) FSX_CK(fsx::launch_r2c_rows_f32(fin, H, p.rows, p.L, lay, tw, twf, st));
        else FSX_CK(fsx::launch_r2c_rows(d_a0, H, p.rows, p.L, lay, tw, st));
        fsx::StepTwiddle none;
        fsx::FusedSymbol sym = fused_symbol(p, taps, T, q, q ? p.qmax.as<unsigned long long>() : nullptr);
        if (!q && zero_columns_enabled()) {
            // columns whose multipliers all underflow to exactly 0: known from the host-side column
            // bound (cached per taps and T), so the fused pass need not evaluate the symbol there
            const i64 kz = plan_kcut(p, taps, T);
            if (kz >= 0) sym.kzero = kz;
        }
        fsx::FusedSymbol nosym;
        if (r == 3) {
            if (p.tma1 && twf && p.ax1.n <= 4096) FSX_CK(fsx::launch_cols_tma_f32(p.map1, p.ax1, 0, nosym, tw, twf, st));
            else if (p.tma1) FSX_CK(fsx::launch_cols_tma(p.map1, p.ax1, 0, nosym, tw, st));
            else FSX_CK(fsx::launch_axis_pow2(H, H, p.ax1, -1, none, tw, st));
        }
        sp.mark();
        if (q) {  // implicit: max |lamQ| for the pinv threshold first
            FSX_CK(cudaMemsetAsync(p.qmax.p, 0, 8, st));
            FSX_CK(fsx::launch_fused_qmax(sym, p.ax0.ncols, p.qmax.as<unsigned long long>(), tw, st));
        }
        // fp32 mode (float grids in / out): the fused pass in fp32 arithmetic where it exists
        const bool f32c = (fin || fout) && !q && sym.real && p.tma0 && !p.halves && p.ax0.n <= 4096 &&
                          fsx::f32_compute_enabled();
        if (f32c) FSX_CK(fsx::launch_cols_tma_f32(p.map0, ax0, 2, sym, tw, dev.tw_all_f.as<float2>(), st));
        else if (p.halves) FSX_CK(fsx::launch_fused_halves(p.map2, ax0, sym, tw, st, H));
        else if (p.tma0) FSX_CK(fsx::launch_cols_tma(p.map0, ax0, 2, sym, tw, st));
        else FSX_CK(fsx::launch_fused_r2c(H, ax0, sym, tw, st));
        sp.mark();
        if (r == 3) {
            if (p.tma1 && twf && p.ax1.n <= 4096) FSX_CK(fsx::launch_cols_tma_f32(p.map1, p.ax1, 1, nosym, tw, twf, st));
            else if (p.tma1) FSX_CK(fsx::launch_cols_tma(p.map1, p.ax1, 1, nosym, tw, st));
            else FSX_CK(fsx::launch_axis_pow2(H, H, p.ax1, +1, none, tw, st));
        }
        if (fout) FSX_CK(fsx::launch_c2r_rows_f32(H, fout, p.rows, p.L, lay, tw, twf, flags, st));
        else FSX_CK(fsx::launch_c2r_rows(H, d_out, p.rows, p.L, lay, tw, flags, st));
        sp.mark();
    } else if (p.kind == kRowPair1D) {
        // the first column pass reads a0 and writes the output buffer (out of
        // place); only without a column pass is a0 copied in first
        if (d_out != d_a0 && p.N1 <= 1)
            FSX_CK(cudaMemcpyAsync(d_out, d_a0, (size_t)p.cells * p.m * 8, cudaMemcpyDeviceToDevice, st));
        double2* z = reinterpret_cast<double2*>(d_out);
        const double2* z0 = reinterpret_cast<const double2*>(d_a0);
        fsx::StepTwiddle tf;
        tf.mode = 1;
        tf.col_div = 1;
        tf.tab = p.tables.get(p.t_M);
        // split column FFT: A over a (stride N1b N2) x W_N1^(b ka), then B over b
        // (stride N2) x W_M^(n2 (ka + N1a kb)); rows end digit-reversed
        const fsx::AxisGeom gA{p.N1a, p.N1b * p.N2, 1, p.Mc, p.N1b * p.N2};
        const fsx::AxisGeom gB{p.N1b, p.N2, p.N1a, p.N1b * p.N2, p.N2};
        fsx::StepTwiddle tA, tB;
        if (p.N1a) {
            tA.mode = 1;
            tA.col_div = p.N2;
            tA.tab = p.tables.get(p.t_N1);
            tB.mode = 1;
            tB.kmul = p.N1a;
            tB.omul = 1;
            tB.tab = p.tables.get(p.t_M);
            if (fin) FSX_CK(fsx::launch_axis_f32(fin, z, gA, -1, tA, tw, st, nullptr));
            else FSX_CK(fsx::launch_axis_pow2(z0, z, gA, -1, tA, tw, st));
            FSX_CK(fsx::launch_axis_pow2(z, z, gB, -1, tB, tw, st));
        } else if (p.N1 > 1) {
            if (fin) FSX_CK(fsx::launch_axis_f32(fin, z, p.colg, -1, tf, tw, st, nullptr));
            else FSX_CK(fsx::launch_axis_pow2(z0, z, p.colg, -1, tf, tw, st));
        }
        sp.mark();
        const fsx::RowPairArgs a = rowpair_args(p, taps, T, z, dev);
        FSX_CK(fsx::launch_rowpair(a, st));
        sp.mark();
        fsx::StepTwiddle ti = tf;
        ti.mode = 2;
        // the last inverse column pass also does the non-finite scan
        if (p.N1a) {
            tA.mode = 2;
            tB.mode = 2;
            FSX_CK(fsx::launch_axis_pow2(z, z, gB, +1, tB, tw, st));
            if (fout) FSX_CK(fsx::launch_axis_f32(z, fout, gA, +1, tA, tw, st, flags));
            else FSX_CK(fsx::launch_axis_pow2(z, z, gA, +1, tA, tw, st, flags));
        } else if (p.N1 > 1) {
            if (fout) FSX_CK(fsx::launch_axis_f32(z, fout, p.colg, +1, ti, tw, st, flags));
            else FSX_CK(fsx::launch_axis_pow2(z, z, p.colg, +1, ti, tw, st, flags));
        } else {
            FSX_CK(fsx::launch_finite_check(d_out, p.cells * p.m, flags, st));
        }
        sp.mark();
    } else {
        double2* Z = p.work.as<double2>();
        FSX_CK(fsx::launch_promote(d_a0, Z, p.cells * p.m * p.batch, st));
        general_axes(p, dev, Z, false, st);
        sp.mark();
        fsx::GeneralSymbol sym = general_symbol(p, taps, q, T, st);
        if (q) {
            FSX_CK(cudaMemsetAsync(const_cast<double*>(sym.qmax), 0, 8, st));
            FSX_CK(fsx::launch_symbol_absmax(sym, const_cast<double*>(sym.qmax), st));
        }
        FSX_CK(fsx::launch_spectral_general(Z, sym, st));
        sp.mark();
        general_axes(p, dev, Z, true, st);
        // realize_checked per stacked grid: flags[b] (the residue test is per solve)
        const i64 nv = p.cells * p.m;
        for (i64 b = 0; b < p.batch; ++b) FSX_CK(fsx::launch_extract(Z + b * nv, d_out + b * nv, nv, flags + b, st));
        sp.mark();
    }
}

// ------------------------------------------------------------------ slab decomposition
struct SlabPlan {
    std::vector<i64> dims;
    int P = 1, r = 0;
    i64 n0l = 0, L = 0, M = 0, Pp = 0, n1 = 1, n1b = 0, CB = 0;
    i64 xcount = 0;  // complex elements per exchange buffer
    DevBuf H;        // 3D: local half spectrum [n0l][n1][Pp]
    alignas(64) unsigned char mapH[128];
    bool tmaH = false;
    fsx::AxisGeom axy;  // 3D local y pass
    // 2D: the largest global column not provably zero (FusedSymbol::kzero), cached (ColumnCut)
    std::shared_ptr<struct ColumnCut> cut;
};

std::mutex g_slab_mu;  // guards the g_slabs map (entries are per device, used under that device's lock)
std::map<std::string, std::unique_ptr<SlabPlan>> g_slabs;

// Geometry only (no device work): validates and fills the sizes.
void slab_geom(const fsx_shape* global, int P, int r, SlabPlan& sp) {
    const Shape s = parse_shape(global);
    const int rk = s.rank();
    if (rk != 2 && rk != 3) throw SpecErr("slab: rank-2 or rank-3 grids only");
    if (s.fields != 1) throw SpecErr("slab: scalar fields only");
    if (P < 1 || r < 0 || r >= P) throw SpecErr("slab: bad rank / world size");
    for (i64 d : s.dims)
        if (!is_pow2(d)) throw SpecErr("slab: power-of-two dims only");
    const i64 L = s.dims[rk - 1];
    if (L < 16 || L > 2 * fsx::kMaxLine || s.dims[0] > fsx::kMaxLine || s.dims[0] % P)
        throw SpecErr("slab: axis 0 must divide by the world size; line lengths as plan 1");
    if (rk == 3 && (s.dims[1] % P || s.dims[1] > fsx::kMaxLine))
        throw SpecErr("slab: axis 1 must divide by the world size");
    sp.dims = s.dims;
    sp.P = P;
    sp.r = r;
    sp.n0l = s.dims[0] / P;
    sp.L = L;
    sp.M = L / 2;
    sp.Pp = sp.M + 8;
    if (rk == 2) {
        sp.CB = ((sp.M + 1 + P - 1) / P + 7) / 8 * 8;
        sp.xcount = s.dims[0] * sp.CB;
    } else {
        sp.n1 = s.dims[1];
        sp.n1b = sp.n1 / P;
        sp.CB = sp.n1b;
        sp.xcount = s.dims[0] * sp.n1b * sp.Pp;
        sp.axy = fsx::AxisGeom{sp.n1, sp.Pp, sp.n0l, sp.n1 * sp.Pp, sp.M + 1};
    }
}

// A slab plan with its device buffers on the current device.
std::unique_ptr<SlabPlan> make_slab_plan(const fsx_shape* global, int P, int r) {
    auto sp = std::make_unique<SlabPlan>();
    slab_geom(global, P, r, *sp);
    if (sp->dims.size() == 3) {
        sp->H.ensure((size_t)sp->n0l * sp->n1 * sp->Pp * 16);
        sp->tmaH = tma_enabled() && fsx::tma_cols_ok(sp->n1) &&
                   fsx::make_cols_tensor_map(sp->mapH, sp->H.p, sp->axy) == 0;
    }
    return sp;
}

// Device plan (call with the device's lock held and the device selected).
SlabPlan& slab_plan(const fsx_shape* global, int P, int r) {
    const Shape s = parse_shape(global);
    int dev = 0;
    cudaGetDevice(&dev);  // the caller selected the device (device_for): plans hold its buffers
    const std::string prefix = std::to_string(dev) + "#";
    std::string key = prefix + std::to_string(P) + "/" + std::to_string(r);
    for (i64 d : s.dims) key += ":" + std::to_string(d);
    std::lock_guard<std::mutex> lk(g_slab_mu);
    auto it = g_slabs.find(key);
    if (it != g_slabs.end()) return *it->second;
    // bounded: drop this device's other slab plans (never another device's, which may be in use)
    int mine = 0;
    for (const auto& e : g_slabs) mine += e.first.rfind(prefix, 0) == 0;
    if (mine >= 16)
        for (auto e = g_slabs.begin(); e != g_slabs.end();) e = e->first.rfind(prefix, 0) == 0 ? g_slabs.erase(e) : std::next(e);
    auto sp = make_slab_plan(global, P, r);
    auto& ref = *sp;
    g_slabs.emplace(key, std::move(sp));
    return ref;
}

void slab_forward(SlabPlan& sp, Device& dev, const double* in, double2* send, cudaStream_t st) {
    const double2* tw = dev.tw_all.as<double2>();
    if (sp.dims.size() == 2) {
        const fsx::RowLayout lay{0, sp.CB, sp.n0l};
        FSX_CK(fsx::launch_r2c_rows(in, send, sp.n0l, sp.L, lay, tw, st));
        return;
    }
    double2* H = sp.H.as<double2>();
    const fsx::RowLayout lay{sp.Pp, 0, sp.n0l * sp.n1};
    FSX_CK(fsx::launch_r2c_rows(in, H, sp.n0l * sp.n1, sp.L, lay, tw, st));
    fsx::FusedSymbol none;
    fsx::StepTwiddle nt;
    if (sp.tmaH) FSX_CK(fsx::launch_cols_tma(sp.mapH, sp.axy, 0, none, tw, st));
    else FSX_CK(fsx::launch_axis_pow2(H, H, sp.axy, -1, nt, tw, st));
    const size_t w = (size_t)sp.n1b * sp.Pp * 16;
    for (int d = 0; d < sp.P; ++d)
        FSX_CK(cudaMemcpy2DAsync(send + (i64)d * sp.n0l * sp.n1b * sp.Pp, w, H + (i64)d * sp.n1b * sp.Pp,
                                 (size_t)sp.n1 * sp.Pp * 16, w, (size_t)sp.n0l, cudaMemcpyDeviceToDevice, st));
}

void slab_inverse(SlabPlan& sp, Device& dev, const double2* send, double* out, cudaStream_t st,
                  fsx::Flags* flags_at = nullptr) {
    const double2* tw = dev.tw_all.as<double2>();
    fsx::Flags* flags = flags_at ? flags_at : dev.flags.as<fsx::Flags>();
    if (sp.dims.size() == 2) {
        const fsx::RowLayout lay{0, sp.CB, sp.n0l};
        FSX_CK(fsx::launch_c2r_rows(send, out, sp.n0l, sp.L, lay, tw, flags, st));
        return;
    }
    double2* H = sp.H.as<double2>();
    const size_t w = (size_t)sp.n1b * sp.Pp * 16;
    for (int d = 0; d < sp.P; ++d)
        FSX_CK(cudaMemcpy2DAsync(H + (i64)d * sp.n1b * sp.Pp, (size_t)sp.n1 * sp.Pp * 16,
                                 send + (i64)d * sp.n0l * sp.n1b * sp.Pp, w, w, (size_t)sp.n0l,
                                 cudaMemcpyDeviceToDevice, st));
    fsx::FusedSymbol none;
    fsx::StepTwiddle nt;
    if (sp.tmaH) FSX_CK(fsx::launch_cols_tma(sp.mapH, sp.axy, 1, none, tw, st));
    else FSX_CK(fsx::launch_axis_pow2(H, H, sp.axy, +1, nt, tw, st));
    const fsx::RowLayout lay{sp.Pp, 0, sp.n0l * sp.n1};
    FSX_CK(fsx::launch_c2r_rows(H, out, sp.n0l * sp.n1, sp.L, lay, tw, flags, st));
}

void slab_spectral(SlabPlan& sp, Device& dev, const Taps& taps, u64 T, double2* recv, cudaStream_t st) {
    const double2* tw = dev.tw_all.as<double2>();
    const int rk = (int)sp.dims.size();
    // a plan-1 view of the global grid for the symbol fields
    Plan view;
    view.dims = sp.dims;
    for (int a = 0; a < rk; ++a) view.axes.push_back(a);
    view.L = sp.L;
    view.M = sp.M;
    view.P = rk == 3 ? sp.Pp : sp.CB;
    view.cells = 1;
    for (i64 d : sp.dims) view.cells *= d;
    fsx::FusedSymbol sym = fused_symbol(view, taps, T);
    sym.c_off = (i64)sp.r * sp.CB;
    if (rk == 2 && zero_columns_enabled()) {
        // host-proved zero columns (global kx, as fused_col_freqs gives it with c_off): same shortcut
        // and same bits as the single-GPU fused pass
        view.kind = kFusedR2C;
        view.m = 1;
        if (!sp.cut) sp.cut = std::make_shared<ColumnCut>();
        const i64 kz = sp.cut->get(view, taps, T);
        if (kz >= 0) sym.kzero = kz;
    }
    const i64 inner = rk == 3 ? sp.n1b * sp.Pp : sp.CB;
    const fsx::AxisGeom g{sp.dims[0], inner, 1, sp.dims[0] * inner, inner};
    alignas(64) unsigned char map[128];
    if (tma_enabled() && fsx::halves_ok(g) && fsx::make_cols_tensor_map_par(map, recv, g) == 0)
        FSX_CK(fsx::launch_fused_halves(map, g, sym, tw, st));
    else if (tma_enabled() && fsx::tma_cols_ok(g.n) && fsx::make_cols_tensor_map(map, recv, g) == 0)
        FSX_CK(fsx::launch_cols_tma(map, g, 2, sym, tw, st));
    else
        FSX_CK(fsx::launch_fused_r2c(recv, g, sym, tw, st));
}

double bits_to_double(unsigned long long b) {
    double d;
    std::memcpy(&d, &b, 8);
    return d;
}

// Decide NumericError from the device flags (realize_checked,
// proj/src/periodic.cpp:53-63) and reset them.
void judge_flags(const fsx::Flags& h, int kind, const std::string& where = "") {
    if (h.nonfinite) throw NumErr("solve_periodic: non-finite value after inverse FFT" + where);
    if (kind == kGeneral) {
        const double mre = bits_to_double(h.max_re_bits), mim = bits_to_double(h.max_im_bits);
        if (mim > 1e-6 * mre) {
            char buf[256];
            std::snprintf(buf, sizeof buf,
                          "solve_periodic: imaginary residue %f exceeds 1e-6 * max |real| (%f); spectrum likely blew up",
                          mim, mre);
            throw NumErr(buf + where);
        }
    }
}

void check_flags(const DevBuf& fl, int kind, cudaStream_t st) {
    fsx::Flags h;
    FSX_CK(cudaMemcpyAsync(&h, fl.p, sizeof(h), cudaMemcpyDeviceToHost, st));
    FSX_CK(cudaStreamSynchronize(st));
    FSX_CK(cudaMemsetAsync(fl.p, 0, sizeof(fsx::Flags), st));
    judge_flags(h, kind);
}

cudaStream_t stream_of(Device& dev, const fsx_options* opt) {
    return (opt && opt->stream) ? reinterpret_cast<cudaStream_t>(opt->stream) : dev.stream;
}

// ------------------------------------------------------------------ naive stepping verifier
// evolve_periodic_naive / step_periodic (proj/src/oracle.cpp:90-115) on the
// GPU: T direct stencil steps, bitwise equal to the reference loop.  Not on
// the solve path; a full-size independent check of the FFT solver.

void evolve_naive(const fsx_shape* shape, const double* a0, const fsx_kernel* k, u64 T, double* out,
                  const fsx_options* opt, bool device_ptrs) {
    const Shape s = parse_shape(shape);
    const Taps taps = parse_kernel(k);
    require_fits(taps, s);
    if (!a0 || !out) throw SpecErr("fsx: null grid pointer");
    const size_t bytes = (size_t)s.values() * 8;
    if (T == 0 && !device_ptrs) {  // proj/src/oracle.cpp:103
        if (out != a0) std::memmove(out, a0, bytes);
        return;
    }
    if (s.fields > fsx::kMaxNaiveFields) throw SpecErr("evolve_periodic_naive: at most 8 fields on the GPU verifier");
    const int rk = s.rank();
    if (rk <= 3 && ((rk == 3 && s.dims[0] > 65535) || (rk >= 2 && s.dims[rk - 2] > 65535)))
        throw SpecErr("evolve_periodic_naive: leading axes must be <= 65535");
    DevLock dlk(opt ? opt->device : 0);
    Device& dev = dlk.dev;
    cudaStream_t st = stream_of(dev, opt);
    if (T == 0) {
        if (out != a0) FSX_CK(cudaMemcpyAsync(out, a0, bytes, cudaMemcpyDeviceToDevice, st));
        return;
    }
    NaiveBufs& nb = dev.naive;
    fsx::NaiveGeom g;
    g.rank = rk;
    g.m = s.fields;
    g.ntaps = (int)taps.map.size();
    g.cells = s.cells;
    const int ra = rk <= 3 ? 3 : rk;
    for (int a = 0; a < ra; ++a) g.n[a] = 1;
    for (int a = 0; a < rk; ++a) g.n[ra - rk + a] = s.dims[a];
    std::vector<long long> off;
    std::vector<double> blk;
    for (const auto& kv : taps.map) {  // sorted offset order, as the reference's map
        for (int a = 0; a < ra - rk; ++a) off.push_back(0);
        for (int a = 0; a < rk; ++a) off.push_back(kv.first[a]);
        blk.insert(blk.end(), kv.second.begin(), kv.second.end());
    }
    nb.off.ensure(off.size() * sizeof(long long));
    nb.blk.ensure(blk.size() * sizeof(double));
    nb.s0.ensure(bytes);
    nb.s1.ensure(bytes);
    // pageable sources: these copies complete before the call returns
    FSX_CK(cudaMemcpyAsync(nb.off.p, off.data(), off.size() * sizeof(long long), cudaMemcpyHostToDevice, st));
    FSX_CK(cudaMemcpyAsync(nb.blk.p, blk.data(), blk.size() * sizeof(double), cudaMemcpyHostToDevice, st));
    FSX_CK(cudaMemcpyAsync(nb.s0.p, a0, bytes, device_ptrs ? cudaMemcpyDeviceToDevice : cudaMemcpyHostToDevice, st));
    double* cur = nb.s0.as<double>();
    double* nxt = nb.s1.as<double>();
    for (u64 t = 0; t < T; ++t) {
        FSX_CK(fsx::launch_step_naive(cur, nxt, g, nb.off.as<long long>(), nb.blk.as<double>(), st));
        std::swap(cur, nxt);
    }
    FSX_CK(cudaMemcpyAsync(out, cur, bytes, device_ptrs ? cudaMemcpyDeviceToDevice : cudaMemcpyDeviceToHost, st));
    if (!device_ptrs) FSX_CK(cudaStreamSynchronize(st));
}

// fp32 storage mode (float grids in and out, fp64 arithmetic): plan 1 reads and
// writes the floats in its row passes; the other plans widen into / narrow out
// of their fp64 buffers (the narrowing flags values outside the float range).
void run_plan_f32(Plan& p, Device& dev, const Taps& taps, u64 T, const float* fin, float* fout, cudaStream_t st,
                  Stamps& sp, fsx::Flags* flags_at = nullptr, bool cut = false) {
    const auto a16 = [](const void* x) { return (reinterpret_cast<uintptr_t>(x) & 15) == 0; };
    if (p.kind == kFusedR2C && fsx::rows_f32_ok(p.L) && a16(fin) && a16(fout)) {
        run_plan(p, dev, taps, nullptr, T, nullptr, nullptr, st, sp, flags_at, fin, fout, cut);
        return;
    }
    const i64 n = p.cells * p.m;
    // 1D plan: the first / last column pass reads / writes the floats (strided
    // route, column length <= 256: the split passes of the large 1D grids);
    // the plan's complex work buffer is d_out
    if (p.kind == kRowPair1D && (reinterpret_cast<uintptr_t>(fin) & 7) == 0 &&
        (reinterpret_cast<uintptr_t>(fout) & 7) == 0 &&
        (p.N1a ? fsx::axis_f32_ok(fsx::AxisGeom{p.N1a, p.N1b * p.N2, 1, p.Mc, p.N1b * p.N2})
               : (p.N1 > 1 && fsx::axis_f32_ok(p.colg)))) {
        p.d_out.ensure((size_t)n * 8);
        run_plan(p, dev, taps, nullptr, T, nullptr, p.d_out.as<double>(), st, sp, flags_at, fin, fout, cut);
        return;
    }
    p.d_in.ensure((size_t)n * 8);
    p.d_out.ensure((size_t)n * 8);
    FSX_CK(fsx::launch_widen(fin, p.d_in.as<double>(), n, st));
    run_plan(p, dev, taps, nullptr, T, p.d_in.as<double>(), p.d_out.as<double>(), st, sp, flags_at, nullptr, nullptr,
             cut);
    FSX_CK(fsx::launch_narrow(p.d_out.as<double>(), fout, n, flags_at ? flags_at : dev.flags.as<fsx::Flags>(), st));
}

// ------------------------------------------------------------------ single-process multi-GPU
// fsx_options.num_gpus / .devices (or the process default of fsx_set_devices):
// one host call slab-decomposes a rank-2/3 grid over P devices of this
// process, like the reference's process-wide thread budget spreads its line
// FFTs over threads (proj/src/parallel.cpp:11-21).  The exchange is either
//   p2p   the NVLink peer-memory transpose: 2D -- the R2C row kernel stores
//         column block d straight into rank d's exchange buffer and the C2R
//         row kernel loads its blocks from every rank's buffer (the
//         all-to-all fused into the row passes); 3D -- the R2C rows and the
//         y pass run in plane chunks and each finished chunk is put into the
//         owners' buffers by the copy engines while the next chunk computes
//         (the inverse pulls chunk by chunk ahead of the y pass and C2R rows);
//   nccl  fsx_slab_forward -> grouped ncclSend/ncclRecv -> fused pass ->
//         grouped ncclSend/ncclRecv -> fsx_slab_inverse (NCCL loaded with
//         dlopen on first use).
// Cross-device ordering is by CUDA events (no device-side spinning): every
// stream waits on all ranks' "exchange written" events before the fused pass
// and on all "fused pass done" events before the inverse reads.  Repeated
// device ordinals run several ranks on one device (the p2p exchange then
// moves within that device's memory): one-GPU emulation for tests.
struct NcclErr : std::runtime_error {
    using std::runtime_error::runtime_error;
};

struct NcclApi {
    bool tried = false, ok = false;
    std::string why;
    decltype(&ncclCommInitAll) CommInitAll = nullptr;
    decltype(&ncclCommDestroy) CommDestroy = nullptr;
    decltype(&ncclGroupStart) GroupStart = nullptr;
    decltype(&ncclGroupEnd) GroupEnd = nullptr;
    decltype(&ncclSend) Send = nullptr;
    decltype(&ncclRecv) Recv = nullptr;
    decltype(&ncclGetErrorString) ErrStr = nullptr;
};
std::mutex g_nccl_mu;
NcclApi g_nccl;

const NcclApi& nccl_api() {
    std::lock_guard<std::mutex> lk(g_nccl_mu);
    if (g_nccl.tried) return g_nccl;
    g_nccl.tried = true;
    void* h = dlopen("libnccl.so.2", RTLD_NOW | RTLD_GLOBAL);
    if (!h) {
        g_nccl.why = std::string("dlopen(libnccl.so.2): ") + dlerror();
        return g_nccl;
    }
    auto sym = [&](auto& fn, const char* name) {
        fn = reinterpret_cast<std::remove_reference_t<decltype(fn)>>(dlsym(h, name));
        return fn != nullptr;
    };
    g_nccl.ok = sym(g_nccl.CommInitAll, "ncclCommInitAll") && sym(g_nccl.CommDestroy, "ncclCommDestroy") &&
                sym(g_nccl.GroupStart, "ncclGroupStart") && sym(g_nccl.GroupEnd, "ncclGroupEnd") &&
                sym(g_nccl.Send, "ncclSend") && sym(g_nccl.Recv, "ncclRecv") &&
                sym(g_nccl.ErrStr, "ncclGetErrorString");
    if (!g_nccl.ok) g_nccl.why = "libnccl.so.2 lacks the point-to-point API";
    return g_nccl;
}

#define FSX_NCCL(api, x)                                                                         \
    do {                                                                                         \
        ncclResult_t r_ = (x);                                                                   \
        if (r_ != ncclSuccess) throw NcclErr(std::string(#x) + ": " + (api).ErrStr(r_));         \
    } while (0)

enum { kExAuto = 0, kExP2P = 1, kExNccl = 2 };

// process default of fsx_set_devices (empty: single GPU)
std::mutex g_multi_default_mu;
std::vector<int> g_multi_default;

struct alignas(64) TmaMap {
    unsigned char b[128];
};

struct MultiRank {
    Device* dev = nullptr;
    int ordinal = 0;
    cudaStream_t st = nullptr;   // kernels
    cudaStream_t cst = nullptr;  // 3D p2p: chunk puts / pulls (copy engines)
    std::unique_ptr<SlabPlan> sp;
    DevBuf in, out, send, recv, peers, flags;
    DevBuf H1, H2, H3;                  // pencils: x-, y- and z-pencil half spectra
    TmaMap map_y, map_z, map_z2;        // pencils: y pass over H2, fused pass over H3 (map_z2: parity view)
    bool tma_y = false, tma_z = false, halves_z = false;
    cudaEvent_t ev_fwd = nullptr, ev_spec = nullptr, ev_done = nullptr;
    cudaEvent_t ev_a = nullptr, ev_b = nullptr;  // pencils: transposes A and B (reverse) written
    std::vector<cudaEvent_t> ev_chunk;  // 3D p2p: per plane chunk
    std::vector<TmaMap> ymaps;          // 3D: y-pass tensor map per plane chunk
    std::vector<bool> ytma;
    ncclComm_t comm = nullptr;
    ~MultiRank() {
        cudaSetDevice(ordinal);
        for (cudaEvent_t e : {ev_fwd, ev_spec, ev_done, ev_a, ev_b})
            if (e) cudaEventDestroy(e);
        for (cudaEvent_t e : ev_chunk) cudaEventDestroy(e);
        if (st) cudaStreamDestroy(st);
        if (cst) cudaStreamDestroy(cst);
        if (comm && g_nccl.ok) g_nccl.CommDestroy(comm);
    }
};

struct MultiCtx {
    std::vector<int> devs;
    std::vector<i64> dims;
    int exchange = kExP2P;
    int P = 1, chunks = 1;
    int decomp = 1;        // 1 slabs, 2 pencils
    // pencils: grid Pr x Pc; local sizes n0r = n0/Pr planes, n1c = n1/Pc rows (x pencils),
    // n1r = n1/Pr (z pencils); kx blocks of CBx columns; H1 row pitch Pp1
    int Pr = 1, Pc = 1;
    i64 n0r = 0, n1c = 0, n1r = 0, CBx = 0, Pp1 = 0, L = 0, M = 0;
    i64 local_values = 0;  // real values per rank's slab / pencil
    std::vector<std::unique_ptr<MultiRank>> ranks;
    bool fresh = true;         // no solve enqueued yet (no ev_done to wait on)
    cudaEvent_t tev[4] = {};   // stage stamps on rank 0's stream
    std::mutex mu;             // one solve per context at a time
    ~MultiCtx() {
        if (!ranks.empty()) cudaSetDevice(ranks[0]->ordinal);
        for (cudaEvent_t e : tev)
            if (e) cudaEventDestroy(e);
        ranks.clear();
    }
};

std::mutex g_multi_mu;
std::map<std::string, std::unique_ptr<MultiCtx>> g_multi;

// The device list a host solve runs on: opt->devices[0..num_gpus) or
// 0..num_gpus-1 when opt->num_gpus > 1 (or devices are given); else the
// process default (fsx_set_devices); empty = single GPU.
std::vector<int> multi_devices(const fsx_options* opt) {
    std::vector<int> devs;
    if (opt && (opt->num_gpus > 1 || (opt->devices && opt->num_gpus >= 1))) {
        for (int r = 0; r < opt->num_gpus; ++r) devs.push_back(opt->devices ? opt->devices[r] : r);
        return devs;
    }
    if (opt && opt->num_gpus == 1) return devs;  // explicitly one GPU
    std::lock_guard<std::mutex> lk(g_multi_default_mu);
    return g_multi_default;
}

// How a problem decomposes over P ranks: 0 = it does not (it runs on one GPU:
// same result contract, the decomposition is a performance choice), 1 = slabs
// along axis 0, 2 = a Pr x Pc pencil grid (3D; Pr returned).  Slabs whenever
// they apply (two transposes against a pencil grid's four), unless pencils
// are asked for.
int multi_decomp(const Shape& s, const Taps& taps, int P, const fsx_options* opt, int exchange, int& Pr) {
    Pr = 1;
    const int rk = s.rank();
    if ((rk != 2 && rk != 3) || s.fields != 1 || P < 1) return 0;
    for (i64 d : s.dims)
        if (!is_pow2(d)) return 0;
    const i64 L = s.dims[rk - 1];
    if (L < 16 || L > 2 * fsx::kMaxLine || s.dims[0] < 8 || s.dims[0] > fsx::kMaxLine) return 0;
    if (rk == 3 && (s.dims[1] < 2 || s.dims[1] > fsx::kMaxLine)) return 0;
    if ((i64)taps.map.size() > fsx::kMaxFusedTaps) return 0;
    std::set<i64> groups;
    for (const auto& kv : taps.map) groups.insert(kv.first[0]);
    if ((int)groups.size() > fsx::kMaxGroups) return 0;
    const int want = opt ? opt->decomp : 0;
    if (want < 0 || want > 2) throw SpecErr("fsx_options.decomp: 0 auto, 1 slab, 2 pencil");
    const bool slab_ok = s.dims[0] % P == 0 && (rk == 2 || s.dims[1] % P == 0);
    if (want != 2 && slab_ok) return 1;
    if (want == 1 || rk != 3 || exchange == kExNccl) return 0;
    // pencils: Pr from the options, else the most square factorization (Pr <= Pc)
    int pr = opt ? opt->pencil_rows : 0;
    if (pr <= 0)
        for (int d = 1; d * d <= P; ++d)
            if (P % d == 0) pr = d;
    if (pr < 1 || P % pr) return 0;
    const int pc = P / pr;
    const i64 n0 = s.dims[0], n1 = s.dims[1];
    if (n0 % pr || n1 % pc || n1 % pr || (L / 2 + 1) < pc) return 0;
    Pr = pr;
    return 2;
}


// The context for (device list, dims, exchange), created on first use; returned
// with its mutex held (taken under g_multi_mu, so the bounded cache cannot
// evict a context between its lookup and its use).
// p2p when every pair of the devices has peer access, else NCCL
int resolve_exchange(const std::vector<int>& devs, int exchange) {
    if (exchange != kExAuto) return exchange;
    std::set<int> distinct(devs.begin(), devs.end());
    for (int a : distinct)
        for (int b : distinct) {
            int can = 1;
            if (a != b) FSX_CK(cudaDeviceCanAccessPeer(&can, a, b));
            if (!can) return kExNccl;
        }
    return kExP2P;
}

MultiCtx& multi_ctx(const fsx_shape* global, const Shape& s, const std::vector<int>& devs, int exchange, int decomp,
                    int Pr, std::unique_lock<std::mutex>& held) {
    const int P = (int)devs.size();
    std::set<int> distinct(devs.begin(), devs.end());
    std::string key = std::to_string(exchange) + "|" + std::to_string(decomp) + "x" + std::to_string(Pr) + "|";
    for (int d : devs) key += std::to_string(d) + ",";
    for (i64 d : s.dims) key += ":" + std::to_string(d);
    std::lock_guard<std::mutex> lk(g_multi_mu);
    auto it = g_multi.find(key);
    if (it != g_multi.end()) {
        held = std::unique_lock<std::mutex>(it->second->mu);
        return *it->second;
    }
    if (g_multi.size() >= 4) {  // bounded: drop idle contexts
        for (auto e = g_multi.begin(); e != g_multi.end();) {
            std::unique_lock<std::mutex> busy(e->second->mu, std::try_to_lock);
            if (busy.owns_lock()) {
                busy.unlock();
                e = g_multi.erase(e);
            } else {
                ++e;
            }
        }
    }
    auto c = std::make_unique<MultiCtx>();
    c->devs = devs;
    c->dims = s.dims;
    c->exchange = exchange;
    c->P = P;
    c->local_values = s.cells / P;
    c->decomp = decomp;
    const bool three = s.rank() == 3;
    if (decomp == 2) {
        c->Pr = Pr;
        c->Pc = P / Pr;
        c->L = s.dims[2];
        c->M = c->L / 2;
        c->n0r = s.dims[0] / c->Pr;
        c->n1c = s.dims[1] / c->Pc;
        c->n1r = s.dims[1] / c->Pr;
        c->CBx = (c->M + 1 + c->Pc - 1) / c->Pc;
        c->Pp1 = (std::max<i64>(c->M + 8, c->Pc * c->CBx) + 7) / 8 * 8;
    }
    // peer access between every pair of distinct devices (NVLink / NVSwitch)
    if (exchange == kExP2P)
        for (int a : distinct)
            for (int b : distinct) {
                if (a == b) continue;
                int can = 0;
                FSX_CK(cudaDeviceCanAccessPeer(&can, a, b));
                if (!can) throw SpecErr("multi-GPU p2p exchange: device " + std::to_string(a) + " cannot access device " +
                                        std::to_string(b) + " (use the nccl exchange)");
                FSX_CK(cudaSetDevice(a));
                const cudaError_t e = cudaDeviceEnablePeerAccess(b, 0);
                if (e == cudaErrorPeerAccessAlreadyEnabled) cudaGetLastError();
                else FSX_CK(e);
            }
    for (int r = 0; r < P; ++r) {
        auto mr = std::make_unique<MultiRank>();
        mr->ordinal = devs[r];
        mr->dev = &device_for(devs[r]);  // selects the device
        FSX_CK(cudaStreamCreateWithFlags(&mr->st, cudaStreamNonBlocking));
        FSX_CK(cudaStreamCreateWithFlags(&mr->cst, cudaStreamNonBlocking));
        for (cudaEvent_t* e : {&mr->ev_fwd, &mr->ev_spec, &mr->ev_done, &mr->ev_a, &mr->ev_b})
            FSX_CK(cudaEventCreateWithFlags(e, cudaEventDisableTiming));
        if (decomp == 2) {
            // pencils: x (H1 [n0r][n1c][Pp1]), y (H2 [n0r][n1][CBx]), z (H3 [n0][n1r][CBx])
            mr->in.ensure((size_t)c->local_values * 8);
            mr->out.ensure((size_t)c->local_values * 8);
            mr->H1.ensure((size_t)c->n0r * c->n1c * c->Pp1 * 16);
            mr->H2.ensure((size_t)c->n0r * s.dims[1] * c->CBx * 16);
            mr->H3.ensure((size_t)s.dims[0] * c->n1r * c->CBx * 16);
            FSX_CK(cudaMemset(mr->H1.p, 0, mr->H1.bytes));  // the kx padding of the last block stays finite
            mr->flags.ensure(sizeof(fsx::Flags));
            FSX_CK(cudaMemset(mr->flags.p, 0, sizeof(fsx::Flags)));
            const fsx::AxisGeom gy{s.dims[1], c->CBx, c->n0r, s.dims[1] * c->CBx, c->CBx};
            mr->tma_y = tma_enabled() && fsx::tma_cols_ok(s.dims[1]) && c->CBx % fsx::tma_cols_width(s.dims[1]) == 0 &&
                        fsx::make_cols_tensor_map(mr->map_y.b, mr->H2.p, gy) == 0;
            const i64 inz = c->n1r * c->CBx;
            const fsx::AxisGeom gz{s.dims[0], inz, 1, s.dims[0] * inz, inz};
            mr->halves_z = tma_enabled() && fsx::halves_ok(gz) && fsx::make_cols_tensor_map_par(mr->map_z2.b, mr->H3.p, gz) == 0;
            mr->tma_z = tma_enabled() && fsx::tma_cols_ok(s.dims[0]) && inz % fsx::tma_cols_width(s.dims[0]) == 0 &&
                        fsx::make_cols_tensor_map(mr->map_z.b, mr->H3.p, gz) == 0;
            c->ranks.push_back(std::move(mr));
            continue;
        }
        mr->sp = make_slab_plan(global, P, r);
        const SlabPlan& sp = *mr->sp;
        mr->in.ensure((size_t)c->local_values * 8);
        mr->out.ensure((size_t)c->local_values * 8);
        mr->recv.ensure((size_t)sp.xcount * 16);
        if (exchange == kExNccl) mr->send.ensure((size_t)sp.xcount * 16);
        mr->flags.ensure(sizeof(fsx::Flags));
        FSX_CK(cudaMemset(mr->flags.p, 0, sizeof(fsx::Flags)));
        if (three) {
            // plane chunks of the 3D exchange: up to 4, each >= 1 plane
            c->chunks = (int)std::min<i64>(4, sp.n0l);
            const i64 pc = sp.n0l / c->chunks;
            mr->ymaps.resize(c->chunks);
            mr->ytma.assign(c->chunks, false);
            mr->ev_chunk.resize(c->chunks);
            for (int q = 0; q < c->chunks; ++q) {
                FSX_CK(cudaEventCreateWithFlags(&mr->ev_chunk[q], cudaEventDisableTiming));
                fsx::AxisGeom g = sp.axy;
                g.outer = pc;
                mr->ytma[q] = tma_enabled() && fsx::tma_cols_ok(sp.n1) &&
                              fsx::make_cols_tensor_map(mr->ymaps[q].b, sp.H.as<double2>() + q * pc * sp.n1 * sp.Pp,
                                                        g) == 0;
            }
        }
        c->ranks.push_back(std::move(mr));
    }
    if (exchange == kExP2P && !three && decomp == 1) {
        // 2D: each rank's device array of every rank's exchange buffer
        std::vector<void*> ptrs(P);
        for (int d = 0; d < P; ++d) ptrs[d] = c->ranks[d]->recv.p;
        for (auto& mr : c->ranks) {
            FSX_CK(cudaSetDevice(mr->ordinal));
            mr->peers.ensure(P * sizeof(void*));
            FSX_CK(cudaMemcpy(mr->peers.p, ptrs.data(), P * sizeof(void*), cudaMemcpyHostToDevice));
        }
    }
    if (exchange == kExNccl) {
        const NcclApi& api = nccl_api();
        if (!api.ok) throw NcclErr("multi-GPU nccl exchange: " + api.why);
        if ((int)distinct.size() != P)
            throw SpecErr("multi-GPU nccl exchange: one rank per device (repeated ordinals need the p2p exchange)");
        std::vector<ncclComm_t> comms(P);
        FSX_NCCL(api, api.CommInitAll(comms.data(), P, devs.data()));
        for (int r = 0; r < P; ++r) c->ranks[r]->comm = comms[r];
    }
    FSX_CK(cudaSetDevice(devs[0]));
    for (cudaEvent_t& e : c->tev) FSX_CK(cudaEventCreate(&e));
    auto& ref = *c;
    g_multi.emplace(key, std::move(c));
    held = std::unique_lock<std::mutex>(ref.mu);
    return ref;
}

// One grouped all-to-all of equal blocks: rank r sends src_r block d to rank
// d, which receives it as dst_d block r (NCCL point-to-point, one group).
void nccl_all_to_all(MultiCtx& c, bool back) {
    const NcclApi& api = nccl_api();
    const size_t blk = (size_t)c.ranks[0]->sp->xcount / c.P * 2;  // doubles per block
    FSX_NCCL(api, api.GroupStart());
    for (int r = 0; r < c.P; ++r) {
        MultiRank& mr = *c.ranks[r];
        const double* src = (back ? mr.recv : mr.send).as<double>();
        double* dst = (back ? mr.send : mr.recv).as<double>();
        for (int d = 0; d < c.P; ++d) {
            FSX_NCCL(api, api.Send(src + d * blk, blk, ncclDouble, d, mr.comm, mr.st));
            FSX_NCCL(api, api.Recv(dst + d * blk, blk, ncclDouble, d, mr.comm, mr.st));
        }
    }
    FSX_NCCL(api, api.GroupEnd());
}

// Every rank's stream st (or cst) waits on event ev of every rank.
void multi_barrier(MultiCtx& c, cudaEvent_t MultiRank::*ev, bool copy_stream = false) {
    for (auto& mr : c.ranks) {
        FSX_CK(cudaSetDevice(mr->ordinal));
        for (auto& other : c.ranks) FSX_CK(cudaStreamWaitEvent(copy_stream ? mr->cst : mr->st, (*other).*ev, 0));
    }
}

// One host-pointer solve over the context's ranks (the caller holds every
// involved device's lock and the context's).
void multi_solve(MultiCtx& c, const Taps& taps, u64 T, const double* a0, double* out, fsx_stage_timings* stt,
                 std::chrono::steady_clock::time_point t_entry) {
    using clk = std::chrono::steady_clock;
    const int P = c.P;
    const bool three = c.dims.size() == 3;
    const size_t lbytes = (size_t)c.local_values * 8;
    const auto t_enq = clk::now();
    // the previous solve's inverse reads every exchange buffer: all of it
    // must have finished before this solve writes into them
    if (!c.fresh) multi_barrier(c, &MultiRank::ev_done);
    FSX_CK(cudaSetDevice(c.ranks[0]->ordinal));
    if (stt) FSX_CK(cudaEventRecord(c.tev[0], c.ranks[0]->st));
    for (int r = 0; r < P; ++r) {
        MultiRank& mr = *c.ranks[r];
        SlabPlan& sp = *mr.sp;
        const double2* tw = mr.dev->tw_all.as<double2>();
        FSX_CK(cudaSetDevice(mr.ordinal));
        FSX_CK(cudaMemcpyAsync(mr.in.p, a0 + (size_t)r * c.local_values, lbytes, cudaMemcpyHostToDevice, mr.st));
        if (c.exchange == kExNccl) {
            slab_forward(sp, *mr.dev, mr.in.as<double>(), mr.send.as<double2>(), mr.st);
        } else if (!three) {
            const fsx::RowLayout lay{0, sp.CB, sp.n0l, mr.peers.as<double2* const>(), (i64)r * sp.n0l};
            FSX_CK(fsx::launch_r2c_rows(mr.in.as<double>(), nullptr, sp.n0l, sp.L, lay, tw, mr.st));
            FSX_CK(cudaEventRecord(mr.ev_fwd, mr.st));
        } else {
            // chunked: R2C rows + y pass of a plane chunk, then its puts on the copy stream
            const i64 pc = sp.n0l / c.chunks, crow = pc * sp.n1;
            double2* H = sp.H.as<double2>();
            const size_t w = (size_t)sp.n1b * sp.Pp * 16;
            for (int q = 0; q < c.chunks; ++q) {
                const fsx::RowLayout lay{sp.Pp, 0, crow};
                double2* Hq = H + q * crow * sp.Pp;
                FSX_CK(fsx::launch_r2c_rows(mr.in.as<double>() + q * crow * sp.L, Hq, crow, sp.L, lay, tw, mr.st));
                fsx::AxisGeom g = sp.axy;
                g.outer = pc;
                fsx::FusedSymbol none;
                fsx::StepTwiddle nt;
                if (mr.ytma[q]) FSX_CK(fsx::launch_cols_tma(mr.ymaps[q].b, g, 0, none, tw, mr.st));
                else FSX_CK(fsx::launch_axis_pow2(Hq, Hq, g, -1, nt, tw, mr.st));
                FSX_CK(cudaEventRecord(mr.ev_chunk[q], mr.st));
                FSX_CK(cudaStreamWaitEvent(mr.cst, mr.ev_chunk[q], 0));
                for (int d = 0; d < P; ++d) {
                    double2* dst = c.ranks[d]->recv.as<double2>() + ((i64)r * sp.n0l + q * pc) * sp.n1b * sp.Pp;
                    FSX_CK(cudaMemcpy2DAsync(dst, w, Hq + d * sp.n1b * sp.Pp, (size_t)sp.n1 * sp.Pp * 16, w,
                                             (size_t)pc, cudaMemcpyDefault, mr.cst));
                }
            }
            FSX_CK(cudaEventRecord(mr.ev_fwd, mr.cst));
        }
    }
    if (c.exchange == kExNccl) nccl_all_to_all(c, false);
    else multi_barrier(c, &MultiRank::ev_fwd);
    FSX_CK(cudaSetDevice(c.ranks[0]->ordinal));
    if (stt) FSX_CK(cudaEventRecord(c.tev[1], c.ranks[0]->st));
    for (auto& mr : c.ranks) {
        FSX_CK(cudaSetDevice(mr->ordinal));
        slab_spectral(*mr->sp, *mr->dev, taps, T, mr->recv.as<double2>(), mr->st);
        FSX_CK(cudaEventRecord(mr->ev_spec, mr->st));
    }
    FSX_CK(cudaSetDevice(c.ranks[0]->ordinal));
    if (stt) FSX_CK(cudaEventRecord(c.tev[2], c.ranks[0]->st));
    if (c.exchange == kExNccl) nccl_all_to_all(c, true);
    else multi_barrier(c, &MultiRank::ev_spec, three);
    for (int r = 0; r < P; ++r) {
        MultiRank& mr = *c.ranks[r];
        SlabPlan& sp = *mr.sp;
        const double2* tw = mr.dev->tw_all.as<double2>();
        fsx::Flags* fl = mr.flags.as<fsx::Flags>();
        FSX_CK(cudaSetDevice(mr.ordinal));
        if (c.exchange == kExNccl) {
            slab_inverse(sp, *mr.dev, mr.send.as<double2>(), mr.out.as<double>(), mr.st, fl);
        } else if (!three) {
            const fsx::RowLayout lay{0, sp.CB, sp.n0l, mr.peers.as<double2* const>(), (i64)r * sp.n0l};
            FSX_CK(fsx::launch_c2r_rows(nullptr, mr.out.as<double>(), sp.n0l, sp.L, lay, tw, fl, mr.st));
        } else {
            // chunked pulls of this rank's blocks ahead of the inverse y pass and C2R rows
            const i64 pc = sp.n0l / c.chunks, crow = pc * sp.n1;
            double2* H = sp.H.as<double2>();
            const size_t w = (size_t)sp.n1b * sp.Pp * 16;
            for (int q = 0; q < c.chunks; ++q) {
                double2* Hq = H + q * crow * sp.Pp;
                for (int d = 0; d < P; ++d) {
                    const double2* src = c.ranks[d]->recv.as<double2>() + ((i64)r * sp.n0l + q * pc) * sp.n1b * sp.Pp;
                    FSX_CK(cudaMemcpy2DAsync(Hq + d * sp.n1b * sp.Pp, (size_t)sp.n1 * sp.Pp * 16, src, w, w, (size_t)pc,
                                             cudaMemcpyDefault, mr.cst));
                }
                FSX_CK(cudaEventRecord(mr.ev_chunk[q], mr.cst));
                FSX_CK(cudaStreamWaitEvent(mr.st, mr.ev_chunk[q], 0));
                fsx::AxisGeom g = sp.axy;
                g.outer = pc;
                fsx::FusedSymbol none;
                fsx::StepTwiddle nt;
                if (mr.ytma[q]) FSX_CK(fsx::launch_cols_tma(mr.ymaps[q].b, g, 1, none, tw, mr.st));
                else FSX_CK(fsx::launch_axis_pow2(Hq, Hq, g, +1, nt, tw, mr.st));
                const fsx::RowLayout lay{sp.Pp, 0, crow};
                FSX_CK(fsx::launch_c2r_rows(Hq, mr.out.as<double>() + q * crow * sp.L, crow, sp.L, lay, tw, fl, mr.st));
            }
        }
        FSX_CK(cudaMemcpyAsync(out + (size_t)r * c.local_values, mr.out.p, lbytes, cudaMemcpyDeviceToHost, mr.st));
        FSX_CK(cudaEventRecord(mr.ev_done, mr.st));
    }
    FSX_CK(cudaSetDevice(c.ranks[0]->ordinal));
    if (stt) FSX_CK(cudaEventRecord(c.tev[3], c.ranks[0]->st));
    c.fresh = false;
    // synchronize, then the reference's realize check on every slab
    std::string err;
    for (int r = 0; r < P; ++r) {
        MultiRank& mr = *c.ranks[r];
        FSX_CK(cudaSetDevice(mr.ordinal));
        FSX_CK(cudaStreamSynchronize(mr.st));
        fsx::Flags h;
        FSX_CK(cudaMemcpy(&h, mr.flags.p, sizeof(h), cudaMemcpyDeviceToHost));
        FSX_CK(cudaMemset(mr.flags.p, 0, sizeof(h)));
        if (h.nonfinite && err.empty()) err = " (slab " + std::to_string(r) + " of " + std::to_string(P) + ")";
    }
    if (!err.empty()) throw NumErr("solve_periodic: non-finite value after inverse FFT" + err);
    if (stt) {
        // wait for rank 0's last stamp: every rank's stream joined it through the barriers
        FSX_CK(cudaSetDevice(c.ranks[0]->ordinal));
        FSX_CK(cudaEventSynchronize(c.tev[3]));
        float t01 = 0, t12 = 0, t23 = 0;
        FSX_CK(cudaEventElapsedTime(&t01, c.tev[0], c.tev[1]));
        FSX_CK(cudaEventElapsedTime(&t12, c.tev[1], c.tev[2]));
        FSX_CK(cudaEventElapsedTime(&t23, c.tev[2], c.tev[3]));
        const double setup = std::chrono::duration<double>(t_enq - t_entry).count();
        const double total = std::chrono::duration<double>(clk::now() - t_entry).count();
        const double gpu = (t01 + t12 + t23) * 1e-3;
        stt->forward_fft += setup + t01 * 1e-3;
        stt->squaring += t12 * 1e-3;
        stt->inverse_fft += t23 * 1e-3 + std::max(0.0, total - setup - gpu);
    }
}

// 3D grid on a Pr x Pc pencil grid (rank r = pr Pc + pc): x pencils (planes
// [pr n0r, ...), rows [pc n1c, ...), full L) -> R2C rows -> transpose A within
// the row group (kx blocks of CBx columns; full y lines) -> y pass ->
// transpose B within the column group (y blocks of n1r rows; full z lines) ->
// fused axis-0 pass with the tile's (ky, kx) offsets -> the reverse.  Every
// transpose is one pitched copy per peer by the copy engines straight into
// the peer's buffer (no pack buffers); each is closed by an event barrier
// before its data is read.  Same kernels per line as the single-GPU solve.
void multi_solve_pencil(MultiCtx& c, const Taps& taps, u64 T, const double* a0, double* out, fsx_stage_timings* stt,
                        std::chrono::steady_clock::time_point t_entry) {
    using clk = std::chrono::steady_clock;
    const int P = c.P, Pc = c.Pc;
    const i64 n0 = c.dims[0], n1 = c.dims[1], L = c.L;
    const auto t_enq = clk::now();
    auto copy3d = [](void* dst, size_t dpitch, size_t dysize, const void* src, size_t spitch, size_t sysize, size_t w,
                     size_t h, size_t d, cudaStream_t st) {
        cudaMemcpy3DParms p = {};
        p.srcPtr = make_cudaPitchedPtr(const_cast<void*>(src), spitch, w, sysize);
        p.dstPtr = make_cudaPitchedPtr(dst, dpitch, w, dysize);
        p.extent = make_cudaExtent(w, h, d);
        p.kind = cudaMemcpyDefault;
        FSX_CK(cudaMemcpy3DAsync(&p, st));
    };
    if (!c.fresh) multi_barrier(c, &MultiRank::ev_done);
    FSX_CK(cudaSetDevice(c.ranks[0]->ordinal));
    if (stt) FSX_CK(cudaEventRecord(c.tev[0], c.ranks[0]->st));
    // x pencils: H2D, R2C rows, transpose A (kx block pc' to rank (pr, pc'), at its y offset pc n1c)
    for (int r = 0; r < P; ++r) {
        MultiRank& mr = *c.ranks[r];
        const int pr = r / Pc, pc = r % Pc;
        const double2* tw = mr.dev->tw_all.as<double2>();
        FSX_CK(cudaSetDevice(mr.ordinal));
        const double* src = a0 + ((size_t)pr * c.n0r * n1 + (size_t)pc * c.n1c) * L;
        FSX_CK(cudaMemcpy2DAsync(mr.in.p, (size_t)c.n1c * L * 8, src, (size_t)n1 * L * 8, (size_t)c.n1c * L * 8,
                                 (size_t)c.n0r, cudaMemcpyHostToDevice, mr.st));
        const fsx::RowLayout lay{c.Pp1, 0, c.n0r * c.n1c};
        FSX_CK(fsx::launch_r2c_rows(mr.in.as<double>(), mr.H1.as<double2>(), c.n0r * c.n1c, L, lay, tw, mr.st));
        for (int q = 0; q < Pc; ++q) {
            MultiRank& dst = *c.ranks[pr * Pc + q];
            copy3d(dst.H2.as<double2>() + (size_t)pc * c.n1c * c.CBx, (size_t)c.CBx * 16, (size_t)n1,
                   mr.H1.as<double2>() + (size_t)q * c.CBx, (size_t)c.Pp1 * 16, (size_t)c.n1c, (size_t)c.CBx * 16,
                   (size_t)c.n1c, (size_t)c.n0r, mr.st);
        }
        FSX_CK(cudaEventRecord(mr.ev_a, mr.st));
    }
    multi_barrier(c, &MultiRank::ev_a);
    // y pass, transpose B (y block pr' to rank (pr', pc), at its plane offset pr n0r)
    fsx::StepTwiddle nt;
    fsx::FusedSymbol none;
    for (int r = 0; r < P; ++r) {
        MultiRank& mr = *c.ranks[r];
        const int pr = r / Pc, pc = r % Pc;
        const double2* tw = mr.dev->tw_all.as<double2>();
        FSX_CK(cudaSetDevice(mr.ordinal));
        const fsx::AxisGeom gy{n1, c.CBx, c.n0r, n1 * c.CBx, c.CBx};
        if (mr.tma_y) FSX_CK(fsx::launch_cols_tma(mr.map_y.b, gy, 0, none, tw, mr.st));
        else FSX_CK(fsx::launch_axis_pow2(mr.H2.as<double2>(), mr.H2.as<double2>(), gy, -1, nt, tw, mr.st));
        const size_t w = (size_t)c.n1r * c.CBx * 16;
        for (int q = 0; q < c.Pr; ++q) {
            MultiRank& dst = *c.ranks[q * Pc + pc];
            FSX_CK(cudaMemcpy2DAsync(dst.H3.as<double2>() + (size_t)pr * c.n0r * c.n1r * c.CBx, w,
                                     mr.H2.as<double2>() + (size_t)q * c.n1r * c.CBx, (size_t)n1 * c.CBx * 16, w,
                                     (size_t)c.n0r, cudaMemcpyDefault, mr.st));
        }
        FSX_CK(cudaEventRecord(mr.ev_fwd, mr.st));
    }
    multi_barrier(c, &MultiRank::ev_fwd);
    FSX_CK(cudaSetDevice(c.ranks[0]->ordinal));
    if (stt) FSX_CK(cudaEventRecord(c.tev[1], c.ranks[0]->st));
    // fused axis-0 pass on the z pencils: local tile [ky][kx] of pitch CBx at (pr n1r, pc CBx)
    Plan view;
    view.dims = c.dims;
    view.axes = {0, 1, 2};
    view.L = L;
    view.M = c.M;
    view.P = c.CBx;
    view.cells = n0 * n1 * L;
    for (int r = 0; r < P; ++r) {
        MultiRank& mr = *c.ranks[r];
        const int pr = r / Pc, pc = r % Pc;
        const double2* tw = mr.dev->tw_all.as<double2>();
        FSX_CK(cudaSetDevice(mr.ordinal));
        fsx::FusedSymbol sym = fused_symbol(view, taps, T);
        sym.c_off = (i64)pr * c.n1r;
        sym.c_off_x = (i64)pc * c.CBx;
        const i64 inz = c.n1r * c.CBx;
        const fsx::AxisGeom gz{n0, inz, 1, n0 * inz, inz};
        if (mr.halves_z) FSX_CK(fsx::launch_fused_halves(mr.map_z2.b, gz, sym, tw, mr.st));
        else if (mr.tma_z) FSX_CK(fsx::launch_cols_tma(mr.map_z.b, gz, 2, sym, tw, mr.st));
        else FSX_CK(fsx::launch_fused_r2c(mr.H3.as<double2>(), gz, sym, tw, mr.st));
        FSX_CK(cudaEventRecord(mr.ev_spec, mr.st));
    }
    multi_barrier(c, &MultiRank::ev_spec);
    FSX_CK(cudaSetDevice(c.ranks[0]->ordinal));
    if (stt) FSX_CK(cudaEventRecord(c.tev[2], c.ranks[0]->st));
    // reverse transpose B: my planes block pr' back to rank (pr', pc)'s y block pr
    for (int r = 0; r < P; ++r) {
        MultiRank& mr = *c.ranks[r];
        const int pr = r / Pc, pc = r % Pc;
        FSX_CK(cudaSetDevice(mr.ordinal));
        const size_t w = (size_t)c.n1r * c.CBx * 16;
        for (int q = 0; q < c.Pr; ++q) {
            MultiRank& dst = *c.ranks[q * Pc + pc];
            FSX_CK(cudaMemcpy2DAsync(dst.H2.as<double2>() + (size_t)pr * c.n1r * c.CBx, (size_t)n1 * c.CBx * 16,
                                     mr.H3.as<double2>() + (size_t)q * c.n0r * c.n1r * c.CBx, w, w, (size_t)c.n0r,
                                     cudaMemcpyDefault, mr.st));
        }
        FSX_CK(cudaEventRecord(mr.ev_b, mr.st));
    }
    multi_barrier(c, &MultiRank::ev_b);
    // inverse y pass, reverse transpose A: my y block pc' back to rank (pr, pc')'s kx block pc
    for (int r = 0; r < P; ++r) {
        MultiRank& mr = *c.ranks[r];
        const int pr = r / Pc, pc = r % Pc;
        const double2* tw = mr.dev->tw_all.as<double2>();
        FSX_CK(cudaSetDevice(mr.ordinal));
        const fsx::AxisGeom gy{n1, c.CBx, c.n0r, n1 * c.CBx, c.CBx};
        if (mr.tma_y) FSX_CK(fsx::launch_cols_tma(mr.map_y.b, gy, 1, none, tw, mr.st));
        else FSX_CK(fsx::launch_axis_pow2(mr.H2.as<double2>(), mr.H2.as<double2>(), gy, +1, nt, tw, mr.st));
        for (int q = 0; q < Pc; ++q) {
            MultiRank& dst = *c.ranks[pr * Pc + q];
            copy3d(dst.H1.as<double2>() + (size_t)pc * c.CBx, (size_t)c.Pp1 * 16, (size_t)c.n1c,
                   mr.H2.as<double2>() + (size_t)q * c.n1c * c.CBx, (size_t)c.CBx * 16, (size_t)n1, (size_t)c.CBx * 16,
                   (size_t)c.n1c, (size_t)c.n0r, mr.st);
        }
        FSX_CK(cudaEventRecord(mr.ev_a, mr.st));
    }
    multi_barrier(c, &MultiRank::ev_a);
    // C2R rows, D2H of the x pencil
    for (int r = 0; r < P; ++r) {
        MultiRank& mr = *c.ranks[r];
        const int pr = r / Pc, pc = r % Pc;
        const double2* tw = mr.dev->tw_all.as<double2>();
        FSX_CK(cudaSetDevice(mr.ordinal));
        const fsx::RowLayout lay{c.Pp1, 0, c.n0r * c.n1c};
        FSX_CK(fsx::launch_c2r_rows(mr.H1.as<double2>(), mr.out.as<double>(), c.n0r * c.n1c, L, lay, tw,
                                    mr.flags.as<fsx::Flags>(), mr.st));
        double* dsth = out + ((size_t)pr * c.n0r * n1 + (size_t)pc * c.n1c) * L;
        FSX_CK(cudaMemcpy2DAsync(dsth, (size_t)n1 * L * 8, mr.out.p, (size_t)c.n1c * L * 8, (size_t)c.n1c * L * 8,
                                 (size_t)c.n0r, cudaMemcpyDeviceToHost, mr.st));
        FSX_CK(cudaEventRecord(mr.ev_done, mr.st));
    }
    FSX_CK(cudaSetDevice(c.ranks[0]->ordinal));
    if (stt) FSX_CK(cudaEventRecord(c.tev[3], c.ranks[0]->st));
    c.fresh = false;
    std::string err;
    for (int r = 0; r < P; ++r) {
        MultiRank& mr = *c.ranks[r];
        FSX_CK(cudaSetDevice(mr.ordinal));
        FSX_CK(cudaStreamSynchronize(mr.st));
        fsx::Flags h;
        FSX_CK(cudaMemcpy(&h, mr.flags.p, sizeof(h), cudaMemcpyDeviceToHost));
        FSX_CK(cudaMemset(mr.flags.p, 0, sizeof(h)));
        if (h.nonfinite && err.empty())
            err = " (pencil " + std::to_string(r / Pc) + "," + std::to_string(r % Pc) + " of " + std::to_string(c.Pr) +
                  "x" + std::to_string(Pc) + ")";
    }
    if (!err.empty()) throw NumErr("solve_periodic: non-finite value after inverse FFT" + err);
    if (stt) {
        FSX_CK(cudaSetDevice(c.ranks[0]->ordinal));
        FSX_CK(cudaEventSynchronize(c.tev[3]));
        float t01 = 0, t12 = 0, t23 = 0;
        FSX_CK(cudaEventElapsedTime(&t01, c.tev[0], c.tev[1]));
        FSX_CK(cudaEventElapsedTime(&t12, c.tev[1], c.tev[2]));
        FSX_CK(cudaEventElapsedTime(&t23, c.tev[2], c.tev[3]));
        const double setup = std::chrono::duration<double>(t_enq - t_entry).count();
        const double total = std::chrono::duration<double>(clk::now() - t_entry).count();
        const double gpu = (t01 + t12 + t23) * 1e-3;
        stt->forward_fft += setup + t01 * 1e-3;
        stt->squaring += t12 * 1e-3;
        stt->inverse_fft += t23 * 1e-3 + std::max(0.0, total - setup - gpu);
    }
}

// Routes a host solve to the multi-GPU path; false when it runs on one GPU.
bool try_multi(const fsx_shape* shape, const Shape& s, const Taps& taps, u64 T, const double* a0, double* out,
               const fsx_options* opt, fsx_stage_timings* stt, std::chrono::steady_clock::time_point t_entry) {
    const std::vector<int> devs = multi_devices(opt);
    if (devs.empty()) return false;
    const int ex_opt = opt ? opt->exchange : kExAuto;
    if (ex_opt < kExAuto || ex_opt > kExNccl) throw SpecErr("fsx_options.exchange: 0 auto, 1 p2p, 2 nccl");
    // validate the ordinals (DevLock below) before any peer query
    std::set<int> distinct(devs.begin(), devs.end());
    for (int d : distinct) device_for(d);
    const int exchange = resolve_exchange(devs, ex_opt);
    int Pr = 1;
    const int decomp = multi_decomp(s, taps, (int)devs.size(), opt, exchange, Pr);
    if (!decomp) return false;
    // every involved device's lock, in ordinal order (no lock-order inversion)
    std::vector<std::unique_ptr<DevLock>> locks;
    for (int d : distinct) locks.push_back(std::make_unique<DevLock>(d));
    std::unique_lock<std::mutex> held;
    MultiCtx& c = multi_ctx(shape, s, devs, exchange, decomp, Pr, held);
    if (decomp == 2) multi_solve_pencil(c, taps, T, a0, out, stt, t_entry);
    else multi_solve(c, taps, T, a0, out, stt, t_entry);
    return true;
}

struct SolveReq {
    const fsx_shape* shape;
    const double* a0;
    const fsx_kernel* k;
    const fsx_kernel* q;  // implicit: q (mass), k = s
    u64 T;
    double* out;
    const fsx_options* opt;
    fsx_stage_timings* st;
    bool vector = false;
    bool device_ptrs = false;
    const Taps* cached = nullptr;  // solve_periodic_cached: the spectrum's kernel from the cache
    const float* a0f = nullptr;    // fp32 storage mode (a0 / out unused)
    float* outf = nullptr;
};

void solve(const SolveReq& rq) {
    using clk = std::chrono::steady_clock;
    const auto t_entry = clk::now();  // StageTimings cover the whole call (below)
    const Shape s = parse_shape(rq.shape);
    Taps taps, qtaps;
    if (rq.vector) {
        // proj/src/periodic.cpp:103-104 checks the kernel's fields first
        if (!rq.k || rq.k->fields < 2) throw SpecErr("solve_periodic_vector: kernel must carry m > 1 blocks");
    }
    if (rq.q) {
        if (!rq.q || !rq.k || rq.q->fields != 1 || rq.k->fields != 1)
            throw SpecErr("solve_periodic_implicit: scalar kernels only");
        qtaps = parse_kernel(rq.q);
        taps = parse_kernel(rq.k);
        require_fits(qtaps, s);
        require_fits(taps, s);
    } else {
        taps = parse_kernel(rq.k);
        require_fits(taps, s);
        if (rq.cached) taps = *rq.cached;
    }
    const bool f32 = rq.a0f || rq.outf;
    const void* in = f32 ? (const void*)rq.a0f : (const void*)rq.a0;
    void* out = f32 ? (void*)rq.outf : (void*)rq.out;
    if (!in || !out) throw SpecErr("fsx: null grid pointer");
    if (f32 && rq.q) throw SpecErr("fsx: fp32 storage mode covers solve_periodic only");
    const size_t bytes = (size_t)s.values() * (f32 ? 4 : 8);
    const int ordinal = rq.opt ? rq.opt->device : 0;
    if (rq.T == 0 && !rq.device_ptrs) {
        // proj/src/periodic.cpp:79: the input, bit for bit (a copy, no arithmetic)
        if (out != in) std::memmove(out, in, bytes);
        return;
    }
    // host-pointer explicit scalar solves of slab-decomposable grids go to the
    // multi-GPU path when more than one device is asked for
    if (!rq.device_ptrs && !f32 && !rq.q && try_multi(rq.shape, s, taps, rq.T, rq.a0, rq.out, rq.opt, rq.st, t_entry))
        return;
    DevLock dlk(ordinal);
    Device& dev = dlk.dev;
    cudaStream_t st = stream_of(dev, rq.opt);
    if (rq.T == 0) {
        if (out != in) FSX_CK(cudaMemcpyAsync(out, in, bytes, cudaMemcpyDeviceToDevice, st));
        return;
    }
    const int force_general = rq.opt && rq.opt->path == 1;
    const bool cut = rq.opt && rq.opt->spectral_cut;
    Plan* pp = &get_plan(dev, s, taps, force_general);
    if (rq.q && !implicit_fusable(*pp, taps, qtaps)) pp = &get_plan(dev, s, taps, 1);
    Plan& p = *pp;
    if (rq.q && p.kind == kFusedR2C) p.qmax.ensure(8);
    Stamps sp{&dev, rq.st != nullptr || (rq.device_ptrs && rq.opt && rq.opt->stage_events), st};
    plan_enter(p, st);
    if (rq.device_ptrs) {
        if (f32) run_plan_f32(p, dev, taps, rq.T, rq.a0f, rq.outf, st, sp, nullptr, cut);
        else run_plan(p, dev, taps, rq.q ? &qtaps : nullptr, rq.T, rq.a0, rq.out, st, sp, nullptr, nullptr, nullptr, cut);
        plan_leave(p, st);
        if (p.kind == kGeneral) dev.dev_general = 1;  // fsx_device_check applies the residue test
        return;
    }
    // host solves: their own flags slot (a deferred device-mode solve's flags
    // must neither fail nor mask this call's check)
    fsx::Flags* hfl = dev.hflags.as<fsx::Flags>();
    DevBuf& bin = f32 ? p.f_in : p.d_in;
    DevBuf& bout = f32 ? p.f_out : p.d_out;
    bin.ensure(bytes);
    bout.ensure(bytes);
    cudaEvent_t h0 = dev.ev[6], h1 = dev.ev[7];
    const auto t_enq = clk::now();
    if (sp.on) FSX_CK(cudaEventRecord(h0, st));
    FSX_CK(cudaMemcpyAsync(bin.p, in, bytes, cudaMemcpyHostToDevice, st));
    if (f32) run_plan_f32(p, dev, taps, rq.T, p.f_in.as<float>(), p.f_out.as<float>(), st, sp, hfl, cut);
    else run_plan(p, dev, taps, rq.q ? &qtaps : nullptr, rq.T, p.d_in.as<double>(), p.d_out.as<double>(), st, sp,
                  hfl, nullptr, nullptr, cut);
    FSX_CK(cudaMemcpyAsync(out, bout.p, bytes, cudaMemcpyDeviceToHost, st));
    if (sp.on) FSX_CK(cudaEventRecord(h1, st));
    plan_leave(p, st);
    check_flags(dev.hflags, p.kind, st);
    if (sp.on) {
        float t[4] = {0, 0, 0, 0}, pre = 0, post = 0;
        for (int i = 0; i < 3; ++i) FSX_CK(cudaEventElapsedTime(&t[i], dev.ev[i], dev.ev[i + 1]));
        FSX_CK(cudaEventElapsedTime(&pre, h0, dev.ev[0]));
        FSX_CK(cudaEventElapsedTime(&post, dev.ev[3], h1));
        // The reference's stopwatches cover the whole call (spectrum build in
        // forward_fft, the residue scan and real part in inverse_fft,
        // proj/src/periodic.cpp:27-86).  Here: GPU stage intervals from the
        // events, the H2D with forward_fft and the D2H with inverse_fft; the
        // host set-up before the first enqueue (validation, plan, symbol) is
        // added to forward_fft and the host tail (wait, flag check) to
        // inverse_fft, so the stages sum to the call's steady-clock time.
        const double setup = std::chrono::duration<double>(t_enq - t_entry).count();
        const double host_total = std::chrono::duration<double>(clk::now() - t_entry).count();
        const double gpu = (pre + t[0] + t[1] + t[2] + post) * 1e-3;
        const double tail = std::max(0.0, host_total - setup - gpu);
        rq.st->forward_fft += setup + (pre + t[0]) * 1e-3;
        rq.st->squaring += t[1] * 1e-3;
        rq.st->hadamard += 0.0;
        rq.st->inverse_fft += (t[2] + post) * 1e-3 + tail;
    }
}

// Pipelined batch of independent solves of one shape / kernel / T (host
// pointers).  Solve i runs on lane i % 2 (own stream and plan copy): its H2D,
// kernels and D2H are stream-ordered, and the two lanes overlap one solve's
// D2H with the next one's H2D (PCIe is full duplex) and with kernels.  With
// pinned host buffers the batch runs at ~max(H2D, D2H, kernels) per solve
// instead of their sum.  Non-finite / residue checks per solve, reported for
// the first failing index after the batch completes (outputs of the others
// are valid).  SURVEY.md §8(f) item 1 (batched slab solves).
template <class TE>
void solve_batch(const fsx_shape* shape, i64 nb, const TE* const* a0s, const fsx_kernel* k, u64 T,
                 TE* const* outs, const fsx_options* opt) {
    constexpr bool f32 = sizeof(TE) == 4;
    const Shape s = parse_shape(shape);
    const Taps taps = parse_kernel(k);
    require_fits(taps, s);
    if (nb < 0) throw SpecErr("fsx_solve_periodic_batch: negative batch size");
    if (nb > 0 && (!a0s || !outs)) throw SpecErr("fsx: null grid pointer");
    for (i64 i = 0; i < nb; ++i)
        if (!a0s[i] || !outs[i]) throw SpecErr("fsx: null grid pointer");
    const size_t bytes = (size_t)s.values() * sizeof(TE);
    if (T == 0) {
        for (i64 i = 0; i < nb; ++i)
            if (outs[i] != a0s[i]) std::memmove(outs[i], a0s[i], bytes);
        return;
    }
    if (nb == 0) return;
    DevLock dlk(opt ? opt->device : 0);
    Device& dev = dlk.dev;
    const int force_general = opt && opt->path == 1;
    const bool cut = opt && opt->spectral_cut;
    Plan* pl[2];
    for (int l = 0; l < 2; ++l) {
        if (!dev.lanes[l]) {
            FSX_CK(cudaStreamCreateWithFlags(&dev.lanes[l], cudaStreamNonBlocking));
            FSX_CK(cudaEventCreateWithFlags(&dev.lane_ev[l], cudaEventDisableTiming));
        }
        pl[l] = &get_plan(dev, s, taps, force_general, l);
        (f32 ? pl[l]->f_in : pl[l]->d_in).ensure(bytes);
        (f32 ? pl[l]->f_out : pl[l]->d_out).ensure(bytes);
    }
    dev.bflags.ensure((size_t)nb * sizeof(fsx::Flags));
    fsx::Flags* fl = dev.bflags.as<fsx::Flags>();
    FSX_CK(cudaMemsetAsync(fl, 0, (size_t)nb * sizeof(fsx::Flags), dev.lanes[0]));
    // order after the caller's stream (if any) and the flag reset
    if (opt && opt->stream) {
        FSX_CK(cudaEventRecord(dev.lane_ev[1], reinterpret_cast<cudaStream_t>(opt->stream)));
        FSX_CK(cudaStreamWaitEvent(dev.lanes[0], dev.lane_ev[1], 0));
    }
    plan_enter(*pl[0], dev.lanes[0]);
    plan_enter(*pl[1], dev.lanes[0]);
    FSX_CK(cudaEventRecord(dev.lane_ev[0], dev.lanes[0]));
    FSX_CK(cudaStreamWaitEvent(dev.lanes[1], dev.lane_ev[0], 0));
    for (i64 i = 0; i < nb; ++i) {
        const int l = (int)(i & 1);
        Plan& p = *pl[l];
        cudaStream_t st = dev.lanes[l];
        Stamps sp{&dev, false, st};
        DevBuf& bin = f32 ? p.f_in : p.d_in;
        DevBuf& bout = f32 ? p.f_out : p.d_out;
        FSX_CK(cudaMemcpyAsync(bin.p, a0s[i], bytes, cudaMemcpyHostToDevice, st));
        if constexpr (f32) run_plan_f32(p, dev, taps, T, p.f_in.as<float>(), p.f_out.as<float>(), st, sp, fl + i, cut);
        else run_plan(p, dev, taps, nullptr, T, p.d_in.as<double>(), p.d_out.as<double>(), st, sp, fl + i, nullptr,
                      nullptr, cut);
        FSX_CK(cudaMemcpyAsync(outs[i], bout.p, bytes, cudaMemcpyDeviceToHost, st));
    }
    plan_leave(*pl[1], dev.lanes[1]);
    plan_leave(*pl[0], dev.lanes[0]);
    std::vector<fsx::Flags> h((size_t)nb);
    FSX_CK(cudaStreamSynchronize(dev.lanes[1]));
    FSX_CK(cudaMemcpyAsync(h.data(), fl, (size_t)nb * sizeof(fsx::Flags), cudaMemcpyDeviceToHost, dev.lanes[0]));
    FSX_CK(cudaStreamSynchronize(dev.lanes[0]));
    for (i64 i = 0; i < nb; ++i) judge_flags(h[(size_t)i], pl[0]->kind, " (batch item " + std::to_string(i) + ")");
}

// One recursion level's slab solves (the aperiodic recursion's rb_run issues
// the 2d face-slab solve_periodic_cached calls of a level one after another,
// proj/src/aperiodic.cpp:224-228,240-244): slabs of equal shape are stacked
// and solved as one batched plan -- one launch per pass for all of them, the
// stack an outer dimension of every pass -- and the shape groups run on the
// device's two lanes (H2D, kernels and D2H of different groups overlap).
// The spectrum follows SpectrumCache semantics when a cache is given: the
// first kernel seen for a dims vector is the one used for every later slab of
// those dims (proj/src/periodic.cpp:67-74, 88-99).  Plans stay resident in
// the device's plan cache (keyed by shape and stack size) across levels.
// NumericError names the first failing slab in argument order.
void solve_slabs(i64 n, const fsx_shape* shapes, const double* const* a0s, const fsx_kernel* k, u64 T,
                 fsx_spectrum_cache* cache, double* const* outs, const fsx_options* opt, fsx_stage_timings* stt);

template <class F>
fsx_status guarded(F&& f) {
    try {
        f();
        g_err.clear();
        return FSX_OK;
    } catch (const SpecErr& e) {
        g_err = e.what();
        return FSX_ERR_SPEC;
    } catch (const NumErr& e) {
        g_err = e.what();
        return FSX_ERR_NUMERIC;
    } catch (const CudaErr& e) {
        g_err = e.what();
        return e.code == cudaErrorMemoryAllocation ? FSX_ERR_OOM : FSX_ERR_CUDA;
    } catch (const NcclErr& e) {
        g_err = e.what();
        return FSX_ERR_NCCL;
    } catch (const std::bad_alloc&) {
        g_err = "fsx: host allocation failed";
        return FSX_ERR_OOM;
    } catch (const std::exception& e) {
        g_err = e.what();
        return FSX_ERR_CUDA;
    }
}

}  // namespace

// SpectrumCache (proj/include/fftstencil/periodic.hpp:28-35, periodic.cpp:67-74):
// memoised by dims only -- the first kernel seen for a dims vector defines
// the spectrum every later call with those dims uses, as in the reference.
// The spectrum itself is analytic on the GPU, so the cache keeps the kernel.
struct fsx_spectrum_cache {
    std::mutex mu;
    std::map<std::vector<i64>, Taps> by_dims;  // the first kernel seen for a dims vector (Taps::m = its fields)
};

namespace {

// The kernel a dims vector uses under SpectrumCache semantics (the first one
// seen); without a cache, the passed kernel.
Taps cached_taps(fsx_spectrum_cache* cache, const Shape& sh, const Taps& taps) {
    if (!cache) return taps;
    Taps cached;
    {
        std::lock_guard<std::mutex> lk(cache->mu);
        auto it = cache->by_dims.find(sh.dims);
        if (it == cache->by_dims.end()) it = cache->by_dims.emplace(sh.dims, taps).first;
        cached = it->second;
    }
    // the cached spectrum keeps its own block size: a grid with another
    // field count fails in hadamard, as in the reference (spectrum.cpp:111-116)
    if (cached.m != sh.fields) throw SpecErr("hadamard: shape mismatch");
    return cached;
}

struct PlanPin {
    Plan* p;
    explicit PlanPin(Plan* q) : p(q) { ++p->pins; }
    ~PlanPin() { --p->pins; }
    PlanPin(const PlanPin&) = delete;
    PlanPin& operator=(const PlanPin&) = delete;
};

void solve_slabs(i64 n, const fsx_shape* shapes, const double* const* a0s, const fsx_kernel* k, u64 T,
                 fsx_spectrum_cache* cache, double* const* outs, const fsx_options* opt, fsx_stage_timings* stt) {
    using clk = std::chrono::steady_clock;
    const auto t_entry = clk::now();
    if (n < 0) throw SpecErr("fsx_solve_periodic_slabs: negative slab count");
    if (n > 0 && (!shapes || !a0s || !outs)) throw SpecErr("fsx: null grid pointer");
    const Taps taps = parse_kernel(k);
    std::vector<Shape> sh((size_t)n);
    for (i64 i = 0; i < n; ++i) {
        sh[i] = parse_shape(&shapes[i]);
        require_fits(taps, sh[i]);  // the passed kernel is checked (periodic.cpp:91)
        if (!a0s[i] || !outs[i]) throw SpecErr("fsx: null grid pointer");
    }
    // shape groups in first-seen order, each with its (cached) kernel
    std::vector<std::string> order;
    std::map<std::string, std::vector<i64>> groups;
    std::map<std::string, Taps> gtaps;
    for (i64 i = 0; i < n; ++i) {
        const std::string key = plan_key(sh[i], 0);
        if (!groups.count(key)) {
            order.push_back(key);
            gtaps.emplace(key, cached_taps(cache, sh[i], taps));
        }
        groups[key].push_back(i);
    }
    if (T == 0) {  // proj/src/periodic.cpp:79 per slab
        for (i64 i = 0; i < n; ++i)
            if (outs[i] != a0s[i]) std::memmove(outs[i], a0s[i], (size_t)sh[i].values() * 8);
        return;
    }
    if (n == 0) return;
    DevLock dlk(opt ? opt->device : 0);
    Device& dev = dlk.dev;
    for (int l = 0; l < 2; ++l)
        if (!dev.lanes[l]) {
            FSX_CK(cudaStreamCreateWithFlags(&dev.lanes[l], cudaStreamNonBlocking));
            FSX_CK(cudaEventCreateWithFlags(&dev.lane_ev[l], cudaEventDisableTiming));
        }
    dev.bflags.ensure((size_t)n * sizeof(fsx::Flags));
    fsx::Flags* fl = dev.bflags.as<fsx::Flags>();
    FSX_CK(cudaMemsetAsync(fl, 0, (size_t)n * sizeof(fsx::Flags), dev.lanes[0]));
    if (opt && opt->stream) {
        FSX_CK(cudaEventRecord(dev.lane_ev[1], reinterpret_cast<cudaStream_t>(opt->stream)));
        FSX_CK(cudaStreamWaitEvent(dev.lanes[0], dev.lane_ev[1], 0));
    }
    FSX_CK(cudaEventRecord(dev.lane_ev[0], dev.lanes[0]));
    FSX_CK(cudaStreamWaitEvent(dev.lanes[1], dev.lane_ev[0], 0));
    // every group's plan first (pinned: a later group's plan must not evict an earlier one)
    std::vector<Plan*> plans;
    std::vector<std::unique_ptr<PlanPin>> pins;
    for (const std::string& key : order) {
        const std::vector<i64>& idx = groups[key];
        Plan* p = &get_plan(dev, sh[idx[0]], gtaps[key], 0, 0, (i64)idx.size());
        pins.push_back(std::make_unique<PlanPin>(p));
        plans.push_back(p);
    }
    // flag slots: group gi owns the contiguous range [gofs, gofs + B) -- one per
    // stacked grid on the general plan (the residue test is per solve), the
    // first one for a stacked plan-1 group (its C2R pass sets one flag)
    std::vector<i64> flag_of((size_t)n);
    i64 gofs = 0;
    for (size_t gi = 0; gi < order.size(); ++gi) {
        const std::vector<i64>& idx = groups[order[gi]];
        Plan& p = *plans[gi];
        cudaStream_t st = dev.lanes[gi & 1];
        const i64 B = (i64)idx.size();
        const size_t bytes = (size_t)sh[idx[0]].values() * 8;
        p.d_in.ensure(bytes * B);
        p.d_out.ensure(bytes * B);
        plan_enter(p, st);
        for (i64 b = 0; b < B; ++b)
            FSX_CK(cudaMemcpyAsync(p.d_in.as<char>() + b * bytes, a0s[idx[b]], bytes, cudaMemcpyHostToDevice, st));
        Stamps sp{&dev, false, st};
        run_plan(p, dev, gtaps[order[gi]], nullptr, T, p.d_in.as<double>(), p.d_out.as<double>(), st, sp, fl + gofs);
        for (i64 b = 0; b < B; ++b) {
            FSX_CK(cudaMemcpyAsync(outs[idx[b]], p.d_out.as<char>() + b * bytes, bytes, cudaMemcpyDeviceToHost, st));
            flag_of[idx[b]] = gofs + (p.kind == kGeneral ? b : 0);
        }
        plan_leave(p, st);
        gofs += B;
    }
    std::vector<fsx::Flags> h((size_t)n);
    FSX_CK(cudaStreamSynchronize(dev.lanes[1]));
    FSX_CK(cudaMemcpyAsync(h.data(), fl, (size_t)n * sizeof(fsx::Flags), cudaMemcpyDeviceToHost, dev.lanes[0]));
    FSX_CK(cudaStreamSynchronize(dev.lanes[0]));
    for (i64 i = 0; i < n; ++i) {
        const fsx::Flags& f = h[(size_t)flag_of[i]];
        int kind = kGeneral;
        for (size_t gi = 0; gi < order.size(); ++gi)
            if (plan_key(sh[i], 0) == order[gi]) kind = plans[gi]->kind;
        if (kind != kGeneral && f.nonfinite) {
            // one flag for a stacked plan-1 group: name the slab whose output is non-finite
            const double* o = outs[i];
            bool bad = false;
            for (i64 j = 0; j < sh[i].values() && !bad; ++j) bad = !std::isfinite(o[j]);
            if (!bad) continue;
        }
        judge_flags(f, kind, " (slab " + std::to_string(i) + ")");
    }
    if (stt) stt->boundary_recursion += std::chrono::duration<double>(clk::now() - t_entry).count();
}

}  // namespace

extern "C" {

// the I/O module's errors (fsx_io.cpp) land in the same thread-local message
__attribute__((visibility("hidden"))) void fsx_internal_set_error(const char* msg) { g_err = msg ? msg : ""; }

const char* fsx_last_error(void) { return g_err.c_str(); }
int32_t fsx_version(void) { return FSX_ABI_VERSION; }

fsx_status fsx_set_devices(const int32_t* devices, int32_t n) {
    return guarded([&] {
        if (n < 0 || n > 1024) throw SpecErr("fsx_set_devices: bad device count");
        std::vector<int> devs;
        if (n > 1 || (n == 1 && devices)) {
            int count = 0;
            if (cudaGetDeviceCount(&count) != cudaSuccess) {
                cudaGetLastError();
                count = 0;
            }
            for (int r = 0; r < n; ++r) {
                const int d = devices ? devices[r] : r;
                if (d < 0 || d >= count) throw SpecErr("fsx_set_devices: device ordinal out of range");
                devs.push_back(d);
            }
        }
        std::lock_guard<std::mutex> lk(g_multi_default_mu);
        g_multi_default = devs;
    });
}

int32_t fsx_get_devices(int32_t* devices, int32_t cap) {
    std::lock_guard<std::mutex> lk(g_multi_default_mu);
    for (int32_t r = 0; devices && r < cap && r < (int32_t)g_multi_default.size(); ++r) devices[r] = g_multi_default[r];
    return (int32_t)g_multi_default.size();
}

int32_t fsx_device_count(void) {
    int n = 0;
    if (cudaGetDeviceCount(&n) != cudaSuccess) {
        cudaGetLastError();
        return 0;
    }
    return n;
}

fsx_status fsx_solve_periodic(const fsx_shape* shape, const double* a0, const fsx_kernel* k, uint64_t T,
                              double* out, const fsx_options* opt, fsx_stage_timings* st) {
    return guarded([&] { solve({shape, a0, k, nullptr, T, out, opt, st}); });
}

fsx_status fsx_solve_periodic_vector(const fsx_shape* shape, const double* a0, const fsx_kernel* k, uint64_t T,
                                     double* out, const fsx_options* opt, fsx_stage_timings* st) {
    return guarded([&] {
        SolveReq rq{shape, a0, k, nullptr, T, out, opt, st};
        rq.vector = true;
        solve(rq);
    });
}

fsx_spectrum_cache* fsx_spectrum_cache_create(void) { return new (std::nothrow) fsx_spectrum_cache(); }
void fsx_spectrum_cache_destroy(fsx_spectrum_cache* c) { delete c; }

fsx_status fsx_solve_periodic_cached(const fsx_shape* shape, const double* a0, const fsx_kernel* k, uint64_t T,
                                     fsx_spectrum_cache* cache, double* out, const fsx_options* opt,
                                     fsx_stage_timings* st) {
    return guarded([&] {
        if (!cache) throw SpecErr("solve_periodic_cached: null cache");
        const Shape sh = parse_shape(shape);
        const Taps taps = parse_kernel(k);
        require_fits(taps, sh);  // the passed kernel is checked (periodic.cpp:91)
        const Taps cached = cached_taps(cache, sh, taps);
        SolveReq rq{shape, a0, k, nullptr, T, out, opt, st};
        rq.cached = &cached;
        solve(rq);
    });
}

fsx_status fsx_solve_periodic_implicit(const fsx_shape* shape, const double* a0, const fsx_kernel* q,
                                       const fsx_kernel* s, uint64_t T, double* out, const fsx_options* opt,
                                       fsx_stage_timings* st) {
    return guarded([&] {
        if (!q || !s) throw SpecErr("solve_periodic_implicit: null kernel");
        SolveReq rq{shape, a0, s, q, T, out, opt, st};
        solve(rq);
    });
}

fsx_status fsx_solve_periodic_device(const fsx_shape* shape, const double* d_a0, const fsx_kernel* k, uint64_t T,
                                     double* d_out, const fsx_options* opt) {
    return guarded([&] {
        SolveReq rq{shape, d_a0, k, nullptr, T, d_out, opt, nullptr};
        rq.device_ptrs = true;
        solve(rq);
    });
}

fsx_status fsx_step_periodic(const fsx_shape* shape, const double* a, const fsx_kernel* k, double* out,
                             const fsx_options* opt) {
    return guarded([&] { evolve_naive(shape, a, k, 1, out, opt, false); });
}

fsx_status fsx_evolve_periodic_naive(const fsx_shape* shape, const double* a0, const fsx_kernel* k, uint64_t T,
                                     double* out, const fsx_options* opt) {
    return guarded([&] { evolve_naive(shape, a0, k, T, out, opt, false); });
}

fsx_status fsx_evolve_periodic_naive_device(const fsx_shape* shape, const double* d_a0, const fsx_kernel* k,
                                            uint64_t T, double* d_out, const fsx_options* opt) {
    return guarded([&] { evolve_naive(shape, d_a0, k, T, d_out, opt, true); });
}

fsx_status fsx_solve_periodic_batch(const fsx_shape* shape, int64_t nbatch, const double* const* a0s,
                                    const fsx_kernel* k, uint64_t T, double* const* outs, const fsx_options* opt) {
    return guarded([&] { solve_batch<double>(shape, nbatch, a0s, k, T, outs, opt); });
}

fsx_status fsx_solve_periodic_f32(const fsx_shape* shape, const float* a0, const fsx_kernel* k, uint64_t T, float* out,
                                  const fsx_options* opt, fsx_stage_timings* st) {
    return guarded([&] {
        SolveReq rq{shape, nullptr, k, nullptr, T, nullptr, opt, st};
        rq.a0f = a0;
        rq.outf = out;
        solve(rq);
    });
}

fsx_status fsx_solve_periodic_device_f32(const fsx_shape* shape, const float* d_a0, const fsx_kernel* k, uint64_t T,
                                         float* d_out, const fsx_options* opt) {
    return guarded([&] {
        SolveReq rq{shape, nullptr, k, nullptr, T, nullptr, opt, nullptr};
        rq.a0f = d_a0;
        rq.outf = d_out;
        rq.device_ptrs = true;
        solve(rq);
    });
}

fsx_status fsx_solve_periodic_slabs(int64_t nslabs, const fsx_shape* shapes, const double* const* a0s,
                                    const fsx_kernel* k, uint64_t T, fsx_spectrum_cache* cache, double* const* outs,
                                    const fsx_options* opt, fsx_stage_timings* st) {
    return guarded([&] { solve_slabs(nslabs, shapes, a0s, k, T, cache, outs, opt, st); });
}

fsx_status fsx_solve_periodic_batch_f32(const fsx_shape* shape, int64_t nbatch, const float* const* a0s,
                                        const fsx_kernel* k, uint64_t T, float* const* outs, const fsx_options* opt) {
    return guarded([&] { solve_batch<float>(shape, nbatch, a0s, k, T, outs, opt); });
}

fsx_status fsx_device_check(const fsx_options* opt) {
    return guarded([&] {
        DevLock dlk(opt ? opt->device : 0);
        Device& dev = dlk.dev;
        // the reference's imaginary-residue test applies when a complex
        // (general-plan) solve was enqueued since the last check
        const int kind = dev.dev_general ? kGeneral : kFusedR2C;
        dev.dev_general = 0;
        check_flags(dev.flags, kind, stream_of(dev, opt));
    });
}

fsx_status fsx_last_stage_ms(const fsx_options* opt, double* ms) {
    return guarded([&] {
        if (!ms) throw SpecErr("fsx_last_stage_ms: null output");
        DevLock dlk(opt ? opt->device : 0);
        Device& dev = dlk.dev;
        FSX_CK(cudaEventSynchronize(dev.ev[3]));
        for (int i = 0; i < 3; ++i) {
            float t = 0;
            FSX_CK(cudaEventElapsedTime(&t, dev.ev[i], dev.ev[i + 1]));
            ms[i] = t;
        }
    });
}

fsx_status fsx_slab_describe(const fsx_shape* global, int32_t nranks, int32_t rank, fsx_slab_info* info) {
    return guarded([&] {
        if (!info) throw SpecErr("fsx_slab_describe: null info");
        SlabPlan sp;
        slab_geom(global, nranks, rank, sp);
        std::memset(info, 0, sizeof(*info));
        info->nranks = nranks;
        info->rank = rank;
        for (size_t a = 0; a < sp.dims.size(); ++a) info->local_dims[a] = sp.dims[a];
        info->local_dims[0] = sp.n0l;
        info->plane_offset = (int64_t)rank * sp.n0l;
        info->col_block = sp.CB;
        info->xbuf_bytes = sp.xcount * 16;
    });
}

fsx_status fsx_slab_forward(const fsx_shape* global, int32_t nranks, int32_t rank, const double* d_local_in,
                            double* d_send, const fsx_options* opt) {
    return guarded([&] {
        if (!d_local_in || !d_send) throw SpecErr("fsx_slab_forward: null pointer");
        DevLock dlk(opt ? opt->device : 0);
        Device& dev = dlk.dev;
        SlabPlan& sp = slab_plan(global, nranks, rank);
        slab_forward(sp, dev, d_local_in, reinterpret_cast<double2*>(d_send), stream_of(dev, opt));
    });
}

fsx_status fsx_slab_spectral(const fsx_shape* global, const fsx_kernel* k, uint64_t T, int32_t nranks, int32_t rank,
                             double* d_recv, const fsx_options* opt) {
    return guarded([&] {
        if (!d_recv) throw SpecErr("fsx_slab_spectral: null pointer");
        const Shape s = parse_shape(global);
        const Taps taps = parse_kernel(k);
        require_fits(taps, s);
        if ((i64)taps.map.size() > fsx::kMaxFusedTaps) throw SpecErr("slab: at most 64 taps");
        DevLock dlk(opt ? opt->device : 0);
        Device& dev = dlk.dev;
        SlabPlan& sp = slab_plan(global, nranks, rank);
        slab_spectral(sp, dev, taps, T, reinterpret_cast<double2*>(d_recv), stream_of(dev, opt));
    });
}

fsx_status fsx_slab_inverse(const fsx_shape* global, int32_t nranks, int32_t rank, const double* d_send,
                            double* d_local_out, const fsx_options* opt) {
    return guarded([&] {
        if (!d_send || !d_local_out) throw SpecErr("fsx_slab_inverse: null pointer");
        DevLock dlk(opt ? opt->device : 0);
        Device& dev = dlk.dev;
        SlabPlan& sp = slab_plan(global, nranks, rank);
        slab_inverse(sp, dev, reinterpret_cast<const double2*>(d_send), d_local_out, stream_of(dev, opt));
    });
}

// Fused row pass + exchange over NVLink peer memory (2D): the R2C rows store
// column block d straight into rank d's exchange buffer (recv_peers[d]); the
// inverse C2R rows load their blocks from every rank's buffer.  The caller
// separates the stages with a cross-rank barrier (symmetric-memory signal
// pads), which replaces the two NCCL all-to-alls.
SlabPlan& slab_p2p_plan(const fsx_shape* global, int32_t nranks, int32_t rank, void* const* peers) {
    if (!peers) throw SpecErr("slab p2p: null peer pointer array");
    SlabPlan& sp = slab_plan(global, nranks, rank);
    if (sp.dims.size() != 2) throw SpecErr("slab p2p: rank-2 grids only (3D exchanges through NCCL)");
    return sp;
}

fsx_status fsx_slab_forward_p2p(const fsx_shape* global, int32_t nranks, int32_t rank, const double* d_local_in,
                                void* const* d_recv_peers, const fsx_options* opt) {
    return guarded([&] {
        if (!d_local_in) throw SpecErr("fsx_slab_forward_p2p: null pointer");
        DevLock dlk(opt ? opt->device : 0);
        Device& dev = dlk.dev;
        SlabPlan& sp = slab_p2p_plan(global, nranks, rank, d_recv_peers);
        fsx::RowLayout lay{0, sp.CB, sp.n0l, reinterpret_cast<double2* const*>(d_recv_peers), (i64)rank * sp.n0l};
        FSX_CK(fsx::launch_r2c_rows(d_local_in, nullptr, sp.n0l, sp.L, lay, dev.tw_all.as<double2>(), stream_of(dev, opt)));
    });
}

fsx_status fsx_slab_inverse_p2p(const fsx_shape* global, int32_t nranks, int32_t rank, void* const* d_recv_peers,
                                double* d_local_out, const fsx_options* opt) {
    return guarded([&] {
        if (!d_local_out) throw SpecErr("fsx_slab_inverse_p2p: null pointer");
        DevLock dlk(opt ? opt->device : 0);
        Device& dev = dlk.dev;
        SlabPlan& sp = slab_p2p_plan(global, nranks, rank, d_recv_peers);
        fsx::RowLayout lay{0, sp.CB, sp.n0l, reinterpret_cast<double2* const*>(d_recv_peers), (i64)rank * sp.n0l};
        FSX_CK(fsx::launch_c2r_rows(nullptr, d_local_out, sp.n0l, sp.L, lay, dev.tw_all.as<double2>(),
                                    dev.flags.as<fsx::Flags>(), stream_of(dev, opt)));
    });
}

fsx_status fsx_spectral_cut_columns(const fsx_shape* shape, const fsx_kernel* k, uint64_t T, int64_t* kept,
                                    int64_t* total) {
    return guarded([&] {
        const Shape s = parse_shape(shape);
        const Taps taps = parse_kernel(k);
        require_fits(taps, s);
        DevLock dlk(0);
        Device& dev = dlk.dev;
        Plan& p = get_plan(dev, s, taps, 0);
        const i64 all = p.kind == kFusedR2C ? p.M + 1 : 0;
        const i64 kc = T == 0 ? -1 : plan_kcut(p, taps, T);
        if (kept) *kept = kc >= 0 ? kc + 1 : all;
        if (total) *total = all;
    });
}

fsx_status fsx_plan_describe(const fsx_shape* shape, const fsx_kernel* k, const fsx_options* opt,
                             fsx_plan_info* info) {
    return guarded([&] {
        if (!info) throw SpecErr("fsx_plan_describe: null info");
        const Shape s = parse_shape(shape);
        const Taps taps = parse_kernel(k);
        require_fits(taps, s);
        DevLock dlk(opt ? opt->device : 0);
        Device& dev = dlk.dev;
        Plan& p = get_plan(dev, s, taps, opt && opt->path == 1);
        info->path = p.kind;
        info->launches = p.launches;
        info->alg_bytes = p.alg_bytes;
        info->fused_bytes = p.fused_bytes;
        info->work_bytes = (int64_t)p.work.bytes;
        info->sched_bytes = p.sched_bytes ? p.sched_bytes : p.alg_bytes;
        info->ranks = 1;
        info->exchange = 0;
        const std::vector<int> devs = multi_devices(opt);
        info->decomp = 0;
        info->pencil_rows = 0;
        if (!devs.empty()) {
            std::set<int> distinct(devs.begin(), devs.end());
            for (int d : distinct) device_for(d);
            const int ex = resolve_exchange(devs, opt ? opt->exchange : kExAuto);
            int Pr = 1;
            const int dc = multi_decomp(s, taps, (int)devs.size(), opt, ex, Pr);
            if (dc) {
                info->ranks = (int32_t)devs.size();
                info->exchange = ex;
                info->decomp = dc;
                info->pencil_rows = dc == 2 ? Pr : 0;
            }
        }
    });
}

// ---------------------------------------------------------------- building blocks
fsx_status fsx_multi_fft(const fsx_shape* shape, const double* in, double* out, int32_t inverse) {
    return guarded([&] {
        const Shape s = parse_shape(shape);
        if (!in || !out) throw SpecErr("multi_fft: null pointer");
        DevLock dlk(0);
        Device& dev = dlk.dev;
        cudaStream_t st = dev.stream;
        Taps dummy;
        dummy.rank = s.rank();
        dummy.m = s.fields;
        dummy.map.emplace(std::vector<i64>(s.rank(), 0), std::vector<double>(s.fields * s.fields, 0.0));
        Plan& p = get_plan(dev, s, dummy, 1);
        const size_t bytes = (size_t)s.values() * 16;
        double2* Z = p.work.as<double2>();
        p.d_in.ensure(bytes);
        FSX_CK(cudaMemcpyAsync(Z, in, bytes, cudaMemcpyHostToDevice, st));
        const int r = (int)p.dims.size();
        // split axes are stored [k1][k2] between the passes; present natural order
        auto permute = [&](int to_natural) {
            for (int a = 0; a < r; ++a) {
                const GenAxis& ga = p.gax[a];
                if (!ga.n1) continue;
                i64 inner = p.m, outer = 1;
                for (int b = a + 1; b < r; ++b) inner *= p.dims[b];
                for (int b = 0; b < a; ++b) outer *= p.dims[b];
                FSX_CK(fsx::launch_transpose_split(Z, p.d_in.as<double2>(), outer, ga.n1, ga.n2, inner, to_natural, st));
                FSX_CK(cudaMemcpyAsync(Z, p.d_in.p, bytes, cudaMemcpyDeviceToDevice, st));
            }
        };
        if (inverse) permute(0);
        general_axes(p, dev, Z, inverse != 0, st);
        if (!inverse) permute(1);
        // inverse: 1/n per axis (proj/src/fft.cpp:151-154)
        if (inverse) FSX_CK(fsx::launch_scale(Z, s.values(), 1.0 / (double)s.cells, st));
        FSX_CK(cudaMemcpyAsync(out, Z, bytes, cudaMemcpyDeviceToHost, st));
        FSX_CK(cudaStreamSynchronize(st));
    });
}

fsx_status fsx_spectrum_from_kernel(const fsx_shape* shape, const fsx_kernel* k, double* out) {
    return guarded([&] {
        const Shape s = parse_shape(shape);
        const Taps taps = parse_kernel(k);
        require_fits(taps, s);
        if (!out) throw SpecErr("spectrum_from_kernel: null output");
        if (s.fields > 8) throw SpecErr("spectrum_from_kernel: fields > 8 not supported on the GPU path");
        DevLock dlk(0);
        Device& dev = dlk.dev;
        cudaStream_t st = dev.stream;
        Plan& p = get_plan(dev, s, taps, 1);
        fsx::GeneralSymbol sym = general_symbol(p, taps, nullptr, 1, st);
        for (int a = 0; a < sym.rank; ++a) sym.split[a] = 0;
        const size_t bytes = (size_t)s.cells * s.fields * s.fields * 16;
        DevBuf o;
        o.ensure(bytes);
        FSX_CK(fsx::launch_symbol_blocks(o.as<double2>(), sym, 0, st));
        FSX_CK(cudaMemcpyAsync(out, o.p, bytes, cudaMemcpyDeviceToHost, st));
        FSX_CK(cudaStreamSynchronize(st));
    });
}

static void spectral_io(const fsx_shape* shape, Shape& s, size_t& bytes) {
    s = parse_shape(shape);
    if (s.fields > 8) throw SpecErr("spectrum: fields > 8 not supported on the GPU path");
    bytes = (size_t)s.cells * s.fields * s.fields * 16;
}

fsx_status fsx_pow_spectrum(const fsx_shape* shape, const double* blocks, uint64_t T, double* out) {
    return guarded([&] {
        Shape s;
        size_t bytes;
        spectral_io(shape, s, bytes);
        DevLock dlk(0);
        Device& dev = dlk.dev;
        cudaStream_t st = dev.stream;
        DevBuf a, b;
        a.ensure(bytes);
        b.ensure(bytes);
        FSX_CK(cudaMemcpyAsync(a.p, blocks, bytes, cudaMemcpyHostToDevice, st));
        FSX_CK(fsx::launch_pow_blocks(a.as<double2>(), b.as<double2>(), s.cells, s.fields, T, st));
        FSX_CK(cudaMemcpyAsync(out, b.p, bytes, cudaMemcpyDeviceToHost, st));
        FSX_CK(cudaStreamSynchronize(st));
    });
}

fsx_status fsx_pseudo_inverse_spectrum(const fsx_shape* shape, const double* blocks, double* out) {
    return guarded([&] {
        Shape s;
        size_t bytes;
        spectral_io(shape, s, bytes);
        if (s.fields != 1) throw SpecErr("pseudo_inverse_spectrum: scalar spectra only");
        DevLock dlk(0);
        Device& dev = dlk.dev;
        cudaStream_t st = dev.stream;
        DevBuf a, b, mx;
        a.ensure(bytes);
        b.ensure(bytes);
        mx.ensure(8);
        FSX_CK(cudaMemcpyAsync(a.p, blocks, bytes, cudaMemcpyHostToDevice, st));
        FSX_CK(cudaMemsetAsync(mx.p, 0, 8, st));
        FSX_CK(fsx::launch_absmax(a.as<double2>(), s.cells, mx.as<double>(), st));
        FSX_CK(fsx::launch_pinv(a.as<double2>(), b.as<double2>(), s.cells, mx.as<double>(), st));
        FSX_CK(cudaMemcpyAsync(out, b.p, bytes, cudaMemcpyDeviceToHost, st));
        FSX_CK(cudaStreamSynchronize(st));
    });
}

fsx_status fsx_multiply_spectra(const fsx_shape* shape, const double* a, const double* b, double* out) {
    return guarded([&] {
        Shape s;
        size_t bytes;
        spectral_io(shape, s, bytes);
        DevLock dlk(0);
        Device& dev = dlk.dev;
        cudaStream_t st = dev.stream;
        DevBuf da, db, dc;
        da.ensure(bytes);
        db.ensure(bytes);
        dc.ensure(bytes);
        FSX_CK(cudaMemcpyAsync(da.p, a, bytes, cudaMemcpyHostToDevice, st));
        FSX_CK(cudaMemcpyAsync(db.p, b, bytes, cudaMemcpyHostToDevice, st));
        FSX_CK(fsx::launch_block_mul(da.as<double2>(), db.as<double2>(), dc.as<double2>(), s.cells, s.fields, st));
        FSX_CK(cudaMemcpyAsync(out, dc.p, bytes, cudaMemcpyDeviceToHost, st));
        FSX_CK(cudaStreamSynchronize(st));
    });
}

fsx_status fsx_hadamard(const fsx_shape* shape, const double* lam, const double* x, double* y) {
    return guarded([&] {
        Shape s;
        size_t bytes;
        spectral_io(shape, s, bytes);
        const size_t xb = (size_t)s.values() * 16;
        DevLock dlk(0);
        Device& dev = dlk.dev;
        cudaStream_t st = dev.stream;
        DevBuf dl, dx, dy;
        dl.ensure(bytes);
        dx.ensure(xb);
        dy.ensure(xb);
        FSX_CK(cudaMemcpyAsync(dl.p, lam, bytes, cudaMemcpyHostToDevice, st));
        FSX_CK(cudaMemcpyAsync(dx.p, x, xb, cudaMemcpyHostToDevice, st));
        FSX_CK(fsx::launch_block_matvec(dl.as<double2>(), dx.as<double2>(), dy.as<double2>(), s.cells, s.fields, st));
        FSX_CK(cudaMemcpyAsync(y, dy.p, xb, cudaMemcpyDeviceToHost, st));
        FSX_CK(cudaStreamSynchronize(st));
    });
}

}  // extern "C"
