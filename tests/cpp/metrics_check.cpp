// metrics_check.cpp -- the verification harness (reference metrics.hpp:20-179)
// on deterministic planes, printed with full precision.  Written against the
// reference's headers only; tests/test_cpp_acceptance.py builds the SAME
// source against the reference and against the drop-in and requires
// identical output (host-side code, no device needed).
#include "sobel5/metrics.hpp"
#include "sobel5/synth.hpp"

#include <cmath>
#include <cstdio>
#include <optional>
#include <string>

using namespace sobel5;

namespace {

RealPlane real_of(const GrayPlane& img, double scale, double offset) {
    RealPlane r(img.width(), img.height());
    for (std::size_t i = 0; i < img.size(); ++i)
        r.data()[i] = std::sqrt(static_cast<double>(img.data()[i]) * scale) + offset;
    return r;
}

void print_ssim(const char* tag, const SsimStats& s) {
    std::printf("%s %.17g %.17g %.17g %.17g %.17g %.17g %.17g %.17g\n", tag, s.mu_x, s.mu_y, s.var_x,
                s.var_y, s.cov_xy, s.c1, s.c2, s.ssim);
}

template <typename E>
void expect_throw(const char* tag, E, auto&& fn) {
    try {
        fn();
        std::printf("%s no-throw\n", tag);
    } catch (const E& e) {
        std::printf("%s %s\n", tag, e.what());
    }
}

}  // namespace

int main() {
    const GrayPlane a = synth_random(97, 61, 3), b = synth_random(97, 61, 4);
    const RealPlane x = real_of(a, 3.0, 0.25), y = real_of(b, 2.0, -1.5), z = real_of(a, 3.0, 0.25);
    print_ssim("xy", ssim_global(x, y));
    print_ssim("xx", ssim_global(x, z));
    print_ssim("xy_range", ssim_global(x, y, 255.0));
    const RealPlane flat(8, 8);
    print_ssim("flat", ssim_global(flat, flat));
    const DiffStats d = diff_stats(a, b);
    std::printf("diff_u8 %.17g %.17g %lld\n", d.max_abs, d.mean_abs, static_cast<long long>(d.count_nonzero));
    const DiffStats dr = diff_stats(x, y);
    std::printf("diff_f64 %.17g %.17g %lld\n", dr.max_abs, dr.mean_abs, static_cast<long long>(dr.count_nonzero));
    expect_throw("dims", DimMismatch(""), [&] { ssim_global(x, RealPlane(5, 5)); });
    expect_throw("range", NonPositiveParam(""), [&] { ssim_global(x, y, -1.0); });
    expect_throw("empty", EmptyPlane(""), [&] { ssim_global(RealPlane(), RealPlane()); });
    expect_throw("diff_dims", DimMismatch(""), [&] { diff_stats(a, GrayPlane(3, 3)); });
    expect_throw("iters", NonPositiveParam(""), [&] { measure("m", 1, 1, 0, 1, [] {}); });
    expect_throw("workers", NonPositiveParam(""), [&] { measure("m", 1, 1, 1, 0, [] {}); });
    BenchReport r;
    r.label = "fast-5x5";
    r.width = 2048;
    r.height = 2048;
    r.iterations = 100;
    r.mean_s = 0.0123456789012;
    r.stddev_s = 0.000123456789;
    r.mps = 339.7312345;
    r.mps_per_core = 21.23321;
    std::printf("%s\n%s\n", BenchReport::csv_header().c_str(), r.csv_row().c_str());
    int calls = 0;
    const BenchReport m = measure("count", 10, 20, 5, 2, [&] { ++calls; });
    std::printf("measure calls %d iters %d %s %d %d\n", calls, m.iterations, m.label.c_str(), m.width, m.height);
    return 0;
}
