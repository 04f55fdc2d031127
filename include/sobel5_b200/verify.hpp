// sobel5_b200/verify.hpp -- the verification and measurement layer of the
// drop-in: the oracle's dense correlation (on the GPU) and the host-side
// statistics / timing harness a verify or bench flow uses
// (sobel5_cli.cpp:187-276).
//
// Same names, argument meaning, checks, check order and messages as the
// reference's oracle.hpp:19-49 (conv2d_valid) and metrics.hpp:20-179
// (SsimStats / ssim_global, DiffStats / diff_stats, BenchReport / measure);
// independent implementation.  conv2d_valid runs on the device through the
// C ABI (sobel5_conv2d_valid_host); the statistics are host reductions over
// host planes (they compare results that already live on the host).
#pragma once

#include <algorithm>
#include <chrono>
#include <cmath>
#include <cstdint>
#include <iomanip>
#include <optional>
#include <sstream>
#include <string>
#include <vector>

#include "sobel5_b200/core.hpp"
#include "sobel5_b200/params.hpp"
#include "sobel5_b200/stream.hpp"

namespace sobel5 {

// ---- oracle.hpp:19-49 ---------------------------------------------------------

namespace gpu {
template <std::size_t K>
inline SignedPlane conv2d(const GrayPlane& img, const std::array<std::array<std::int32_t, K>, K>& w) {
    const int k = static_cast<int>(K);
    if (img.width() < k || img.height() < k)
        throw ImageTooSmall("conv2d_valid needs at least " + std::to_string(k) + "x" + std::to_string(k) +
                            ", got " + std::to_string(img.width()) + "x" + std::to_string(img.height()));
    std::int32_t flat[K * K];
    for (std::size_t i = 0; i < K; ++i)
        for (std::size_t j = 0; j < K; ++j) flat[i * K + j] = w[i][j];
    SignedPlane out(img.width() - k + 1, img.height() - k + 1);
    sobel5_ctx* c = thread_context().get();
    const sobel5_status st = sobel5_conv2d_valid_host(c, img.data().data(), img.width(), img.height(), flat, k,
                                                      out.data().data());
    if (st != SOBEL5_OK) raise(st, std::string("conv2d_valid (") + sobel5_ctx_last_error(c) + ")");
    return out;
}
}  // namespace gpu

/// Valid-mode correlation with a 5x5 kernel (no flip): out(y, x) sums
/// k(i, j) * img(y + i, x + j); the int64 sum cast to int32.
inline SignedPlane conv2d_valid(const GrayPlane& img, const Kernel5& k) { return gpu::conv2d<5>(img, k.w); }
inline SignedPlane conv2d_valid(const GrayPlane& img, const Kernel3& k) { return gpu::conv2d<3>(img, k.w); }

// ---- metrics.hpp:20-88 -----------------------------------------------------------

/// Whole-image (global-statistics) SSIM terms, Eq. 22: population means,
/// variances and covariance over every pixel.
struct SsimStats {
    double mu_x = 0;
    double mu_y = 0;
    double var_x = 0;
    double var_y = 0;
    double cov_xy = 0;
    double c1 = 0;
    double c2 = 0;
    double ssim = 0;
};

namespace detail {
inline std::string dims(int w, int h) { return std::to_string(w) + "x" + std::to_string(h); }

template <typename A, typename B>
inline void require_same_nonempty(const A& a, const B& b, const char* who) {
    if (a.empty() || b.empty()) throw EmptyPlane(std::string(who) + " needs non-empty planes");
    if (a.width() != b.width() || a.height() != b.height())
        throw DimMismatch(std::string(who) + " dims differ: " + dims(a.width(), a.height()) + " vs " +
                          dims(b.width(), b.height()));
}
}  // namespace detail

/// data_range, when given, must be positive; by default it is the joint
/// value range of both planes (1.0 when that range is empty).
inline SsimStats ssim_global(const RealPlane& x, const RealPlane& y, std::optional<double> data_range = std::nullopt) {
    detail::require_same_nonempty(x, y, "ssim_global");
    if (data_range && *data_range <= 0)
        throw NonPositiveParam("data_range must be positive, got " + std::to_string(*data_range));
    const std::vector<double>& xs = x.data();
    const std::vector<double>& ys = y.data();
    const double n = static_cast<double>(xs.size());
    // pass 1: sums and the joint range; pass 2: centred second moments
    double sx = 0, sy = 0;
    double lo = xs.front(), hi = xs.front();
    for (std::size_t i = 0; i < xs.size(); ++i) {
        sx += xs[i];
        sy += ys[i];
        lo = std::min({lo, xs[i], ys[i]});
        hi = std::max({hi, xs[i], ys[i]});
    }
    SsimStats s;
    s.mu_x = sx / n;
    s.mu_y = sy / n;
    double vxx = 0, vyy = 0, vxy = 0;
    for (std::size_t i = 0; i < xs.size(); ++i) {
        const double ex = xs[i] - s.mu_x, ey = ys[i] - s.mu_y;
        vxx += ex * ex;
        vyy += ey * ey;
        vxy += ex * ey;
    }
    s.var_x = vxx / n;
    s.var_y = vyy / n;
    s.cov_xy = vxy / n;
    double range = data_range.value_or(hi - lo);
    if (range <= 0) range = 1.0;
    const double k1 = 0.01 * range, k2 = 0.03 * range;
    s.c1 = k1 * k1;
    s.c2 = k2 * k2;
    const double luminance = 2 * (s.mu_x * s.mu_y) + s.c1;
    const double structure = 2 * s.cov_xy + s.c2;
    const double norm_l = s.mu_x * s.mu_x + s.mu_y * s.mu_y + s.c1;
    const double norm_s = s.var_x + s.var_y + s.c2;
    s.ssim = (luminance * structure) / (norm_l * norm_s);
    return s;
}

// ---- metrics.hpp:90-115 ----------------------------------------------------------

struct DiffStats {
    double max_abs = 0;
    double mean_abs = 0;
    std::int64_t count_nonzero = 0;
};

/// Element-wise |a - b| statistics of two same-size planes.
template <typename T>
DiffStats diff_stats(const Plane<T>& a, const Plane<T>& b) {
    detail::require_same_nonempty(a, b, "diff_stats");
    DiffStats s;
    double total = 0;
    const auto& av = a.data();
    const auto& bv = b.data();
    for (std::size_t i = 0; i < av.size(); ++i) {
        const double d = std::fabs(static_cast<double>(av[i]) - static_cast<double>(bv[i]));
        total += d;
        if (d > s.max_abs) s.max_abs = d;
        if (d != 0) ++s.count_nonzero;
    }
    s.mean_abs = total / static_cast<double>(av.size());
    return s;
}

// ---- metrics.hpp:117-179 ---------------------------------------------------------

/// One measurement: mean and population stddev of the timed iterations
/// (one untimed warm-up first) and the derived megapixels per second.
struct BenchReport {
    std::string label;
    int width = 0;
    int height = 0;
    int iterations = 0;
    double mean_s = 0;
    double stddev_s = 0;
    double mps = 0;           // megapixels per second
    double mps_per_core = 0;  // mps / worker threads

    static std::string csv_header() { return "label,width,height,iters,mean_s,stddev_s,mps,mps_per_core"; }

    std::string csv_row() const {
        std::ostringstream row;
        row << label << ',' << width << ',' << height << ',' << iterations << ',';
        row << std::setprecision(9) << mean_s << ',' << stddev_s << ',';
        row << std::setprecision(6) << mps << ',' << mps_per_core;
        return row.str();
    }
};

/// Times fn(): one warm-up call, then `iterations` calls each timed with the
/// steady clock.  workers only scales mps_per_core.
template <typename Fn>
BenchReport measure(const std::string& label, int width, int height, int iterations, int workers, Fn&& fn) {
    if (iterations < 1) throw NonPositiveParam("iterations must be >= 1, got " + std::to_string(iterations));
    if (workers < 1) throw NonPositiveParam("workers must be >= 1, got " + std::to_string(workers));
    using clock = std::chrono::steady_clock;
    fn();
    std::vector<double> t(static_cast<std::size_t>(iterations));
    for (double& dt : t) {
        const auto start = clock::now();
        fn();
        dt = std::chrono::duration<double>(clock::now() - start).count();
    }
    double mean = 0;
    for (double dt : t) mean += dt;
    mean /= static_cast<double>(t.size());
    double m2 = 0;
    for (double dt : t) m2 += (dt - mean) * (dt - mean);
    BenchReport r;
    r.label = label;
    r.width = width;
    r.height = height;
    r.iterations = iterations;
    r.mean_s = mean;
    r.stddev_s = std::sqrt(m2 / static_cast<double>(t.size()));
    r.mps = static_cast<double>(width) * height / (mean * 1e6);
    r.mps_per_core = r.mps / workers;
    return r;
}

}  // namespace sobel5
