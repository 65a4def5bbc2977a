// C++ caller of the drop-in header (include/fftstencil_b200.hpp) — the same
// calls the reference's own tests make (proj/tests/test_periodic.cpp:39-46,
// 57-62, 230-246), through libfsx.so.  Exit code 0 = all checks passed.
// Argument "gpu" also runs the solves that need a device.
#include <cmath>
#include <cstdio>
#include <cstring>

#include "fftstencil_b200.hpp"

using namespace fftstencil_b200;

static int failures = 0;
#define CHECK(c)                                                    \
    do {                                                            \
        if (!(c)) {                                                 \
            std::printf("FAIL %s:%d %s\n", __FILE__, __LINE__, #c); \
            ++failures;                                             \
        }                                                           \
    } while (0)

template <class E, class F>
static bool throws(F&& f) {
    try {
        f();
    } catch (const E&) {
        return true;
    } catch (...) {
        return false;
    }
    return false;
}

int main(int argc, char** argv) {
    const bool gpu = argc > 1 && std::strcmp(argv[1], "gpu") == 0;
    StencilKernel k(1);
    k.add_tap({-1}, -2.0);
    k.add_tap({0}, 1.0);
    k.add_tap({1}, 3.0);
    FieldGrid a(GridShape({4}));
    a.data = {1, 2, 3, 4};
    // T == 0 returns the input exactly (no device needed)
    CHECK(solve_periodic(a, k, 0).data == a.data);
    // SpecError paths (host validation, no device needed)
    StencilKernel far(1);
    far.add_tap({4}, 1.0);
    CHECK(throws<SpecError>([&] { solve_periodic(a, far, 1); }));
    CHECK(throws<SpecError>([&] { solve_periodic_vector(a, k, 1); }));
    CHECK(throws<SpecError>([&] { StencilKernel(1).add_tap({0}, NAN); }));
    CHECK(throws<SpecError>([&] { solve_periodic(a, StencilKernel(1), 1); }));
    // fp32 storage mode, T == 0: a bit-exact copy (no device)
    const std::vector<float> a32 = {1.f, 2.f, 3.f, 4.f};
    CHECK(solve_periodic_f32(GridShape({4}), a32, k, 0) == a32);
    if (gpu) {
        // the Appendix step matrix in fp32 storage: [1,2,3,4] -> [-1,9,11,1]
        const std::vector<float> o32 = solve_periodic_f32(GridShape({4}), a32, k, 1);
        const float w32[4] = {-1, 9, 11, 1};
        for (int i = 0; i < 4; ++i) CHECK(std::fabs(o32[i] - w32[i]) <= 1e-5f);
        const double want[4] = {-1, 9, 11, 1};
        FieldGrid out = solve_periodic(a, k, 1);
        for (int i = 0; i < 4; ++i) CHECK(std::fabs(out.data[i] - want[i]) <= 1e-12);
        StencilKernel blow(1);
        blow.add_tap({1}, 1e8);
        blow.add_tap({0}, 1e8);
        FieldGrid b(GridShape({16}));
        for (int i = 0; i < 16; ++i) b.data[i] = std::sin(i);
        CHECK(throws<NumericError>([&] { solve_periodic(b, blow, 1u << 20); }));
        StageTimings st;
        SpectrumCache cache;
        FieldGrid c = solve_periodic_cached(a, k, 1, cache, &st);
        for (int i = 0; i < 4; ++i) CHECK(std::fabs(c.data[i] - want[i]) <= 1e-12);
        CHECK(st.sum() > 0);
        // multi-GPU through the unchanged drop-in call: the process default
        // device list (two ranks emulated on device 0) slab-decomposes a 2D
        // and a 3D grid; the result matches the single-GPU solve
        StencilKernel k2(2), k3(3);
        for (int o = -1; o <= 1; ++o) {
            k2.add_tap({o, 0}, 0.2);
            k2.add_tap({0, o}, 0.2);
            k3.add_tap({o, 0, 0}, 0.1);
            k3.add_tap({0, o, 0}, 0.1);
            k3.add_tap({0, 0, o}, 0.1);
        }
        FieldGrid g2(GridShape({64, 128})), g3(GridShape({16, 8, 32}));
        for (size_t i = 0; i < g2.data.size(); ++i) g2.data[i] = std::cos(0.37 * i);
        for (size_t i = 0; i < g3.data.size(); ++i) g3.data[i] = std::sin(0.11 * i);
        const FieldGrid s2 = solve_periodic(g2, k2, 50), s3 = solve_periodic(g3, k3, 20);
        set_devices({0, 0});
        StageTimings mst;
        const FieldGrid m2 = solve_periodic(g2, k2, 50, &mst), m3 = solve_periodic(g3, k3, 20);
        set_devices({});
        CHECK(mst.sum() > 0);
        double e2 = 0, n2 = 0, e3 = 0, n3 = 0;
        for (size_t i = 0; i < s2.data.size(); ++i) {
            e2 += (m2.data[i] - s2.data[i]) * (m2.data[i] - s2.data[i]);
            n2 += s2.data[i] * s2.data[i];
        }
        for (size_t i = 0; i < s3.data.size(); ++i) {
            e3 += (m3.data[i] - s3.data[i]) * (m3.data[i] - s3.data[i]);
            n3 += s3.data[i] * s3.data[i];
        }
        CHECK(std::sqrt(e2 / n2) <= 1e-12);
        CHECK(std::sqrt(e3 / n3) <= 1e-12);
        // one recursion level's face slabs (different shapes) in one call =
        // the sequential solve_periodic_cached calls, bit for bit
        std::vector<FieldGrid> level;
        for (int ax = 0; ax < 2; ++ax)
            for (int side = 0; side < 2; ++side) {
                FieldGrid sl(GridShape(ax == 0 ? std::vector<Index>{12, 128} : std::vector<Index>{64, 12}));
                for (size_t i = 0; i < sl.data.size(); ++i) sl.data[i] = std::sin(0.3 * i + ax + 2 * side);
                level.push_back(sl);
            }
        SpectrumCache c1, c2;
        StageTimings bst;
        const std::vector<FieldGrid> batched = solve_periodic_slabs(level, k2, 7, &c1, &bst);
        CHECK(batched.size() == level.size());
        CHECK(bst.boundary_recursion > 0);
        for (size_t i = 0; i < level.size(); ++i) CHECK(batched[i].data == solve_periodic_cached(level[i], k2, 7, c2).data);
    }
    std::printf("%s: %d failure(s)\n", gpu ? "gpu" : "cpu", failures);
    return failures ? 1 : 0;
}
