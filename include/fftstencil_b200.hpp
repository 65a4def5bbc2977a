// fftstencil_b200.hpp — header-only, Eigen-free C++ drop-in over the C ABI
// (fsx.h / libfsx.so) for the reference fftstencil periodic API
// (proj/include/fftstencil/{errors,grid,kernel,periodic}.hpp).
//
// Same names, argument meaning and error types:
//   FieldGrid solve_periodic(const FieldGrid& a0, const StencilKernel& k,
//                            std::uint64_t T, StageTimings* st = nullptr);
// (+ solve_periodic_vector / solve_periodic_cached / solve_periodic_implicit)
// SpecError / NumericError are thrown from the C status codes; CUDA failures
// throw fftstencil_b200::Error.  Link with -lfsx (paper_2105_06676_b200/libfsx.so).
#pragma once

#include <cstdint>
#include <map>
#include <stdexcept>
#include <string>
#include <utility>
#include <vector>

#include "fsx.h"

namespace fftstencil_b200 {

using Index = std::int64_t;

class Error : public std::runtime_error {
public:
    using std::runtime_error::runtime_error;
};
class SpecError : public Error {
public:
    using Error::Error;
};
class NumericError : public Error {
public:
    using Error::Error;
};

inline void check(fsx_status s) {
    if (s == FSX_OK) return;
    const std::string msg = fsx_last_error();
    if (s == FSX_ERR_SPEC) throw SpecError(msg);
    if (s == FSX_ERR_NUMERIC) throw NumericError(msg);
    throw Error("[fsx " + std::to_string((int)s) + "] " + msg);
}

class GridShape {
public:
    GridShape() = default;
    GridShape(std::vector<Index> dims, int fields = 1) : dims_(std::move(dims)), fields_(fields) {
        if (dims_.empty()) throw SpecError("GridShape: need at least one dimension");
        if (dims_.size() > FSX_MAX_RANK) throw SpecError("GridShape: rank too large");
        if (fields_ < 1) throw SpecError("GridShape: fields must be >= 1");
        cells_ = 1;
        for (Index d : dims_) {
            if (d < 1) throw SpecError("GridShape: every dimension must be >= 1");
            cells_ *= d;
        }
    }
    int rank() const { return (int)dims_.size(); }
    const std::vector<Index>& dims() const { return dims_; }
    Index dim(int a) const { return dims_[a]; }
    int fields() const { return fields_; }
    Index cells() const { return cells_; }
    Index values() const { return cells_ * fields_; }
    bool operator==(const GridShape& o) const { return dims_ == o.dims_ && fields_ == o.fields_; }
    fsx_shape c() const {
        fsx_shape s{};
        s.rank = rank();
        s.fields = fields_;
        for (int a = 0; a < rank(); ++a) s.dims[a] = dims_[a];
        return s;
    }

private:
    std::vector<Index> dims_;
    int fields_ = 1;
    Index cells_ = 0;
};

struct FieldGrid {
    GridShape shape;
    std::vector<double> data;  // row-major cells, field innermost
    FieldGrid() = default;
    explicit FieldGrid(GridShape s) : shape(std::move(s)), data(shape.values(), 0.0) {}
    double& at(Index cell, int field = 0) { return data[cell * shape.fields() + field]; }
    double at(Index cell, int field = 0) const { return data[cell * shape.fields() + field]; }
};

class StencilKernel {
public:
    using Offset = std::vector<Index>;
    StencilKernel(int rank, int fields = 1) : rank_(rank), fields_(fields) {
        if (rank < 1) throw SpecError("StencilKernel: rank must be >= 1");
        if (fields < 1) throw SpecError("StencilKernel: fields must be >= 1");
    }
    // m x m row-major block; accumulates (proj/src/kernel.cpp:7-22)
    void add_tap(Offset off, const std::vector<double>& block) {
        if ((int)off.size() != rank_) throw SpecError("StencilKernel: offset rank mismatch");
        if ((int)block.size() != fields_ * fields_) throw SpecError("StencilKernel: block must be fields x fields");
        for (double v : block)
            if (!(v - v == 0.0)) throw SpecError("StencilKernel: non-finite coefficient");
        auto it = taps_.find(off);
        if (it == taps_.end()) taps_.emplace(std::move(off), block);
        else
            for (size_t i = 0; i < block.size(); ++i) it->second[i] += block[i];
    }
    void add_tap(Offset off, double coeff) {
        if (fields_ != 1) throw SpecError("StencilKernel: scalar tap on a multi-field kernel");
        add_tap(std::move(off), std::vector<double>{coeff});
    }
    const std::map<Offset, std::vector<double>>& taps() const { return taps_; }
    int rank() const { return rank_; }
    int fields() const { return fields_; }
    bool empty() const { return taps_.empty(); }

    // flattened arrays kept alive with the returned fsx_kernel
    struct CView {
        std::vector<int64_t> off;
        std::vector<double> blk;
        fsx_kernel k{};
    };
    CView c() const {
        CView v;
        for (const auto& kv : taps_) {
            v.off.insert(v.off.end(), kv.first.begin(), kv.first.end());
            v.blk.insert(v.blk.end(), kv.second.begin(), kv.second.end());
        }
        v.k.rank = rank_;
        v.k.fields = fields_;
        v.k.ntaps = (int64_t)taps_.size();
        v.k.offsets = v.off.data();
        v.k.blocks = v.blk.data();
        return v;
    }

private:
    int rank_, fields_;
    std::map<Offset, std::vector<double>> taps_;
};

struct StageTimings {
    double forward_fft = 0, squaring = 0, hadamard = 0, inverse_fft = 0, boundary_recursion = 0;
    double sum() const { return forward_fft + squaring + hadamard + inverse_fft + boundary_recursion; }
};

class SpectrumCache {
public:
    SpectrumCache() : h_(fsx_spectrum_cache_create()) {}
    ~SpectrumCache() { fsx_spectrum_cache_destroy(h_); }
    SpectrumCache(const SpectrumCache&) = delete;
    SpectrumCache& operator=(const SpectrumCache&) = delete;
    fsx_spectrum_cache* handle() { return h_; }

private:
    fsx_spectrum_cache* h_;
};

// Multi-GPU for every later solve_periodic / solve_periodic_cached of an
// eligible 2D/3D grid in this process (fsx_set_devices): the GPU counterpart
// of the reference's process-wide set_num_threads (proj/src/parallel.cpp:11-21).
// An empty list (or one device) returns to a single GPU.
inline void set_devices(const std::vector<int>& devices) {
    std::vector<std::int32_t> d(devices.begin(), devices.end());
    check(fsx_set_devices(d.empty() ? nullptr : d.data(), (std::int32_t)d.size()));
}
inline void set_num_gpus(int n) { check(fsx_set_devices(nullptr, n)); }

namespace detail {
inline fsx_stage_timings to_c(const StageTimings* st) {
    fsx_stage_timings t{};
    if (st) t = {st->forward_fft, st->squaring, st->hadamard, st->inverse_fft, st->boundary_recursion};
    return t;
}
inline void from_c(const fsx_stage_timings& t, StageTimings* st) {
    if (st) *st = {t.forward_fft, t.squaring, t.hadamard, t.inverse_fft, t.boundary_recursion};
}
}  // namespace detail

inline FieldGrid solve_periodic(const FieldGrid& a0, const StencilKernel& k, std::uint64_t T,
                                StageTimings* st = nullptr) {
    FieldGrid out(a0.shape);
    const fsx_shape s = a0.shape.c();
    auto kv = k.c();
    fsx_stage_timings t = detail::to_c(st);
    check(fsx_solve_periodic(&s, a0.data.data(), &kv.k, T, out.data.data(), nullptr, st ? &t : nullptr));
    detail::from_c(t, st);
    return out;
}

inline FieldGrid solve_periodic_vector(const FieldGrid& a0, const StencilKernel& k, std::uint64_t T,
                                       StageTimings* st = nullptr) {
    FieldGrid out(a0.shape);
    const fsx_shape s = a0.shape.c();
    auto kv = k.c();
    fsx_stage_timings t = detail::to_c(st);
    check(fsx_solve_periodic_vector(&s, a0.data.data(), &kv.k, T, out.data.data(), nullptr, st ? &t : nullptr));
    detail::from_c(t, st);
    return out;
}

inline FieldGrid solve_periodic_cached(const FieldGrid& a0, const StencilKernel& k, std::uint64_t T,
                                       SpectrumCache& cache, StageTimings* st = nullptr) {
    FieldGrid out(a0.shape);
    const fsx_shape s = a0.shape.c();
    auto kv = k.c();
    fsx_stage_timings t = detail::to_c(st);
    check(fsx_solve_periodic_cached(&s, a0.data.data(), &kv.k, T, cache.handle(), out.data.data(), nullptr,
                                    st ? &t : nullptr));
    detail::from_c(t, st);
    return out;
}

inline FieldGrid solve_periodic_implicit(const StencilKernel& q, const StencilKernel& s, const FieldGrid& a0,
                                         std::uint64_t T, StageTimings* st = nullptr) {
    FieldGrid out(a0.shape);
    const fsx_shape sh = a0.shape.c();
    auto qv = q.c();
    auto sv = s.c();
    fsx_stage_timings t = detail::to_c(st);
    check(fsx_solve_periodic_implicit(&sh, a0.data.data(), &qv.k, &sv.k, T, out.data.data(), nullptr,
                                      st ? &t : nullptr));
    detail::from_c(t, st);
    return out;
}

// One recursion level's slab solves in one call (fsx_solve_periodic_slabs):
// the 2d face slabs rb_run hands to solve_periodic_cached one after another
// (proj/src/aperiodic.cpp:224-228,240-244); shapes may differ, equal shapes
// are stacked into one batched plan.  Same results as the sequential calls.
inline std::vector<FieldGrid> solve_periodic_slabs(const std::vector<FieldGrid>& slabs, const StencilKernel& k,
                                                   std::uint64_t T, SpectrumCache* cache = nullptr,
                                                   StageTimings* st = nullptr) {
    std::vector<FieldGrid> out;
    out.reserve(slabs.size());
    std::vector<fsx_shape> shapes;
    std::vector<const double*> ins;
    std::vector<double*> outs;
    for (const FieldGrid& g : slabs) {
        out.emplace_back(g.shape);
        shapes.push_back(g.shape.c());
        ins.push_back(g.data.data());
    }
    for (FieldGrid& g : out) outs.push_back(g.data.data());
    auto kv = k.c();
    fsx_stage_timings t = detail::to_c(st);
    check(fsx_solve_periodic_slabs((int64_t)slabs.size(), shapes.data(), ins.data(), &kv.k, T,
                                   cache ? cache->handle() : nullptr, outs.data(), nullptr, st ? &t : nullptr));
    detail::from_c(t, st);
    return out;
}

// fp32 storage mode (no reference counterpart: the reference is fp64 only):
// float cells in and out, fp64 arithmetic inside (fsx_solve_periodic_f32).
inline std::vector<float> solve_periodic_f32(const GridShape& shape, const std::vector<float>& a0,
                                             const StencilKernel& k, std::uint64_t T, StageTimings* st = nullptr) {
    std::vector<float> out(a0.size());
    const fsx_shape s = shape.c();
    auto kv = k.c();
    fsx_stage_timings t = detail::to_c(st);
    check(fsx_solve_periodic_f32(&s, a0.data(), &kv.k, T, out.data(), nullptr, st ? &t : nullptr));
    detail::from_c(t, st);
    return out;
}

// Direct-stepping verifier on the GPU (oracle.hpp:15-20: step_periodic,
// evolve_periodic_naive), bitwise equal to the reference loop.
inline FieldGrid evolve_periodic_naive(const FieldGrid& a0, const StencilKernel& k, std::uint64_t T) {
    FieldGrid out(a0.shape);
    const fsx_shape s = a0.shape.c();
    auto kv = k.c();
    check(fsx_evolve_periodic_naive(&s, a0.data.data(), &kv.k, T, out.data.data(), nullptr));
    return out;
}

inline FieldGrid step_periodic(const FieldGrid& a, const StencilKernel& k) { return evolve_periodic_naive(a, k, 1); }

}  // namespace fftstencil_b200
