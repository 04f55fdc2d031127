// acceptance.cpp -- SPEC.md ACCEPTANCE 1-5, 7 and 8 as a
// caller of the reference library writes them: only the reference's headers
// ("sobel5/...") and its public API.  The SAME source builds against the
// reference (-I/root/reference/proj/include, CPU) and against this repo's
// drop-in (-I<repo>/include -lsobel5_b200, GPU); tests/test_cpp_acceptance.py
// runs both builds.  Prints one line per criterion and "acceptance: N
// failed"; exit status 1 if any check failed.
//
// usage: acceptance [n_images=200] [max_side=512]
#include "sobel5/filter_algebra.hpp"
#include "sobel5/metrics.hpp"
#include "sobel5/oracle.hpp"
#include "sobel5/pipeline.hpp"
#include "sobel5/strips.hpp"
#include "sobel5/synth.hpp"

#include <cmath>
#include <cstdint>
#include <cstdio>
#include <cstdlib>
#include <iostream>
#include <string>

using namespace sobel5;

namespace {

int g_failed = 0;

void report(const char* what, bool ok, const std::string& detail = "") {
    std::printf("%s: %s%s%s\n", what, ok ? "PASS" : "FAIL", detail.empty() ? "" : "  ",
                detail.c_str());
    if (!ok) ++g_failed;
}

bool same_within(const RealPlane& a, const RealPlane& b, double rel) {
    if (a.width() != b.width() || a.height() != b.height()) return false;
    for (std::size_t i = 0; i < a.size(); ++i) {
        const double x = a.data()[i], y = b.data()[i];
        if (std::fabs(x - y) > rel * std::max(std::fabs(x), std::fabs(y))) return false;
    }
    return true;
}

}  // namespace

int main(int argc, char** argv) {
    const int n_images = argc > 1 ? std::atoi(argv[1]) : 200;
    const int max_side = argc > 2 ? std::atoi(argv[2]) : 512;
    const FilterParams params;  // (1, 2, 6, 4)

    // 1 + 2: oracle equivalence and SSIM over seeded random images from 5x5
    // up to max_side, every lane width x prefetch setting in rotation
    std::uint64_t rng = 2023;
    int bad_int = 0, bad_g = 0, bad_ssim = 0, exact_g = 0;
    double min_ssim = 1.0;
    const int lanes_set[4] = {8, 16, 32, 64};
    for (int i = 0; i < n_images; ++i) {
        const int w = 5 + static_cast<int>(splitmix64(rng) % static_cast<std::uint64_t>(max_side - 4));
        const int h = 5 + static_cast<int>(splitmix64(rng) % static_cast<std::uint64_t>(max_side - 4));
        GrayPlane img = synth_random(w, h, splitmix64(rng));
        if (i % 3 == 1)  // low-amplitude images keep the edge map off saturation
            for (auto& v : img.data()) v &= 0x07;
        const int lanes = lanes_set[i % 4];
        const Prefetch pf = (i / 4) % 2 ? Prefetch::on : Prefetch::off;
        const StreamResult fast = run_stream(img, params, plan_strips(w, lanes, 2), pf, 1 + i % 3);
        const Sobel5Result ref = sobel5_4d(img, params);
        if (!(fast.gx == ref.gx && fast.gy == ref.gy && fast.gd == ref.gd && fast.gdt == ref.gdt))
            ++bad_int;
        if (!same_within(fast.g, ref.g, 1e-9)) ++bad_g;
        exact_g += fast.g == ref.g;
        const SsimStats s = ssim_global(fast.g, ref.g);
        min_ssim = std::min(min_ssim, s.ssim);
        if (s.ssim != 1.0) ++bad_ssim;
        const DiffStats d = diff_stats(fast.gd, ref.gd);
        if (d.count_nonzero != 0 || d.max_abs != 0) ++bad_int;
    }
    report("ACCEPTANCE-1 oracle equivalence (gx/gy/gd/gdt bit-identical, g within 1e-9)",
           bad_int == 0 && bad_g == 0,
           std::to_string(n_images) + " images, " + std::to_string(exact_g) +
               " with bit-identical g, int mismatches " + std::to_string(bad_int));
    report("ACCEPTANCE-2 SSIM == 1.0", bad_ssim == 0, "min " + std::to_string(min_ssim));

    // 3: the diagonal-transform identities and the Gd+- parity through the
    // sum/difference kernels
    {
        bool ok = true;
        std::uint64_t prng = 7;
        for (int t = 0; t < 1000 && ok; ++t) {
            FilterParams p;
            p.a = 1 + static_cast<std::int64_t>(splitmix64(prng) % 3);
            p.b = static_cast<std::int64_t>(1 + splitmix64(prng) % 6);
            p.m = static_cast<std::int64_t>(1 + splitmix64(prng) % 12);
            p.n = static_cast<std::int64_t>(1 + splitmix64(prng) % 12);
            try {
                validate_params(p);
            } catch (const Error&) {
                continue;
            }
            const KdSumDiff sd = make_kd_sum_diff(p);
            const Kernel5 kd = materialize(p, Direction::D), kdt = materialize(p, Direction::DT);
            const KdMinusDecomposition dec = decompose_kd_minus(p);
            const Kernel5 s1 = dec.deriv_term.outer(), s2 = dec.diff_term.outer();
            for (int i = 0; i < 5; ++i)
                for (int j = 0; j < 5; ++j) {
                    ok = ok && sd.plus.at(i, j) + sd.minus.at(i, j) == 2 * kd.at(i, j);
                    ok = ok && sd.plus.at(i, j) - sd.minus.at(i, j) == 2 * kdt.at(i, j);
                    ok = ok && s1.at(i, j) - s2.at(i, j) == sd.minus.at(i, j);
                }
        }
        std::uint64_t irng = 99;
        for (int i = 0; i < 100 && ok; ++i) {
            const GrayPlane img = synth_random(5 + static_cast<int>(splitmix64(irng) % 60),
                                               5 + static_cast<int>(splitmix64(irng) % 60), i + 1);
            const DiagPair dp = diag_via_sum_diff(img, params);  // throws ParityViolation if odd
            const Sobel5Result r = sobel5_4d(img, params);
            ok = ok && dp.gd == r.gd && dp.gdt == r.gdt;
        }
        report("ACCEPTANCE-3 Kd+- identities, Eq. 19, Gd+- parity", ok);
    }

    // 4: reuse budget on a 1024 x 1024 run (lanes 32): 3 k0/k1 row
    // convolutions per incremental row per strip vs 4 naive
    {
        const GrayPlane img = synth_random(1024, 1024, 1);
        const StripPlan plan = plan_strips(1024, 32, 2);
        const StreamResult r = run_stream(img, params, plan, Prefetch::on);
        // per strip: k0 = 2H - 8, k1 = H - 2 (priming excluded: 3 per incremental row)
        const std::uint64_t ns = plan.strips.size(), H = 1024;
        const double per_row = static_cast<double>(r.counters.row_conv5_k0 + r.counters.row_conv5_k1) /
                               (static_cast<double>(ns) * (H - 10.0 / 3.0));
        report("ACCEPTANCE-4 k0/k1 convolutions per incremental row per strip == 3 (naive 4)",
               r.counters.row_conv5_k0 == ns * (2 * H - 8) && r.counters.row_conv5_k1 == ns * (H - 2) &&
                   r.counters.row_conv5_f == r.counters.row_diff,
               "k0 " + std::to_string(r.counters.row_conv5_k0) + " k1 " +
                   std::to_string(r.counters.row_conv5_k1) + " per row " + std::to_string(per_row));
    }

    // 5: the speed comparison, in the reference's measure() CSV schema
    // (reported: the relative criterion is machine-local)
    {
        const GrayPlane img = synth_random(2048, 2048, 1);
        const StripPlan plan = plan_strips(2048, 32, 2);
        std::cout << BenchReport::csv_header() << "\n";
        const BenchReport fast = measure("fast-5x5", 2048, 2048, 3, 1,
                                         [&] { (void)run_stream(img, params, plan, Prefetch::on); });
        const BenchReport orc = measure("oracle-5x5", 2048, 2048, 3, 1, [&] { (void)sobel5_4d(img, params); });
        std::cout << fast.csv_row() << "\n" << orc.csv_row() << "\n";
        std::printf("ACCEPTANCE-5 speed: fast / oracle MPS = %.2f (reported)\n", fast.mps / orc.mps);
    }

    // 7: the 3x3 two-direction path against the Eq. 1-2 dense correlations
    {
        bool ok = true;
        std::uint64_t r3 = 5;
        for (int i = 0; i < 100 && ok; ++i) {
            const int w = 3 + static_cast<int>(splitmix64(r3) % 200), h = 3 + static_cast<int>(splitmix64(r3) % 120);
            const GrayPlane img = synth_random(w, h, 1000 + i);
            const Stream3Result s = run_stream_3x3(img, plan_strips(w, 16, 1), Prefetch::on);
            const SignedPlane gx = conv2d_valid(img, kernel3_x()), gy = conv2d_valid(img, kernel3_y());
            ok = ok && s.gx == gx && s.gy == gy;
            for (int y = 0; y < gx.height() && ok; ++y)
                for (int x = 0; x < gx.width(); ++x) {
                    const double a = gx.at(y, x), b = gy.at(y, x);
                    ok = ok && s.g.at(y, x) == std::sqrt(a * a + b * b);
                }
        }
        report("ACCEPTANCE-7 3x3 streaming path == dense Eq. 1-2", ok);
    }

    // 8: strip coverage for every width up to 4096 (r = 2, lanes 8..64)
    {
        bool ok = true;
        for (int lanes : lanes_set)
            for (int w = 5; w <= 4096 && ok; ++w) {
                const StripPlan p = plan_strips(w, lanes, 2);
                int next = 0;
                for (const Strip& s : p.strips) {
                    ok = ok && s.out_off == next && s.out_w > 0 && s.in_off == s.out_off;
                    next = s.out_off + s.out_w;
                }
                ok = ok && next == w - 4;
            }
        report("ACCEPTANCE-8 strip coverage", ok);
    }

    std::printf("acceptance: %d failed\n", g_failed);
    return g_failed ? 1 : 0;
}
