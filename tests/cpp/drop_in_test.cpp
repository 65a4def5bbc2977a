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
    }
    std::printf("%s: %d failure(s)\n", gpu ? "gpu" : "cpu", failures);
    return failures ? 1 : 0;
}
