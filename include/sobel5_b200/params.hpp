// sobel5_b200/params.hpp -- the (a, b, m, n) filter family and the stream
// taps the kernels consume.  Host-only: this runs once per call.
//
// Same names, checks, check order and messages as the reference's
// filter_algebra.hpp:14-256 and pipeline.hpp:57-107 (make_stream_taps);
// independent implementation (weights are generated from one table of
// rational coefficients instead of per-direction literals).
#pragma once

#include <algorithm>
#include <array>
#include <cstdint>
#include <cstdlib>
#include <string>

#include "sobel5_b200/core.hpp"

namespace sobel5 {

struct Kernel5 {
    std::array<std::array<std::int32_t, 5>, 5> w{};
    std::int32_t at(int i, int j) const { return w[static_cast<std::size_t>(i)][static_cast<std::size_t>(j)]; }
    friend bool operator==(const Kernel5& a, const Kernel5& b) { return a.w == b.w; }
    friend bool operator!=(const Kernel5& a, const Kernel5& b) { return !(a == b); }
};

/// 3x3 integer kernel of the classic two-direction operator (reference
/// filter_algebra.hpp:25-39).
struct Kernel3 {
    std::array<std::array<std::int32_t, 3>, 3> w{};
    std::int32_t at(int i, int j) const { return w[static_cast<std::size_t>(i)][static_cast<std::size_t>(j)]; }
    friend bool operator==(const Kernel3& a, const Kernel3& b) { return a.w == b.w; }
};

namespace detail {
/// Eq. 1: the 3x3 Sobel pair is smoothing [1, 2, 1] across the derivative
/// [-1, 0, 1]; Gx differentiates along the row, Gy down the column.
inline Kernel3 sobel3_outer(bool along_row) {
    constexpr std::int32_t smooth[3] = {1, 2, 1}, deriv[3] = {-1, 0, 1};
    Kernel3 k;
    for (std::size_t i = 0; i < 3; ++i)
        for (std::size_t j = 0; j < 3; ++j)
            k.w[i][j] = along_row ? smooth[i] * deriv[j] : deriv[i] * smooth[j];
    return k;
}
}  // namespace detail

inline Kernel3 kernel3_x() { return detail::sobel3_outer(true); }
inline Kernel3 kernel3_y() { return detail::sobel3_outer(false); }

/// scale * (col outer row)
struct SeparablePair {
    std::array<std::int32_t, 5> col{};
    std::array<std::int32_t, 5> row{};
    std::int32_t scale = 1;
    Kernel5 outer() const {
        Kernel5 k;
        for (std::size_t i = 0; i < 5; ++i)
            for (std::size_t j = 0; j < 5; ++j) k.w[i][j] = scale * col[i] * row[j];
        return k;
    }
};

struct FilterParams {
    std::int64_t a = 1;
    Rational b{2};
    Rational m{6};
    Rational n{4};
};

enum class Direction { X, Y, D, DT };

inline const char* direction_name(Direction d) {
    constexpr const char* names[] = {"Kx", "Ky", "Kd", "Kdt"};
    return names[static_cast<int>(d)];
}

inline constexpr std::int64_t kMaxWeightMagnitude = std::int64_t{1} << 15;

namespace detail {

using RationalKernel = std::array<std::array<Rational, 5>, 5>;

// Symbols of the Eq. 5 weights: each entry is a signed product of a with one
// of {0, 1, b, m, n, mb, nb}.
enum Sym : int { Z, ONE, B, M, N, MB, NB };
// Kd and Kdt (PAPER Eq. 5) as (sign, symbol); Kx/Ky are separable.
constexpr int kKd[5][5][2] = {{{-1, M}, {-1, N}, {-1, ONE}, {-1, B}, {1, Z}},
                              {{-1, N}, {-1, MB}, {-1, NB}, {1, Z}, {1, B}},
                              {{-1, ONE}, {-1, NB}, {1, Z}, {1, NB}, {1, ONE}},
                              {{-1, B}, {1, Z}, {1, NB}, {1, MB}, {1, N}},
                              {{1, Z}, {1, B}, {1, ONE}, {1, N}, {1, M}}};

inline Rational sym_value(int s, const FilterParams& p) {
    switch (s) {
        case Z: return Rational{0};
        case ONE: return Rational{1};
        case B: return p.b;
        case M: return p.m;
        case N: return p.n;
        case MB: return p.m * p.b;
        default: return p.n * p.b;
    }
}

inline RationalKernel materialize_exact(const FilterParams& p, Direction dir) {
    const Rational a{p.a};
    RationalKernel k;
    const std::array<Rational, 5> smooth{Rational{1}, p.n, p.m, p.n, Rational{1}};
    const std::array<Rational, 5> deriv{Rational{-1}, -p.b, Rational{0}, p.b, Rational{1}};
    for (std::size_t i = 0; i < 5; ++i)
        for (std::size_t j = 0; j < 5; ++j) {
            switch (dir) {
                case Direction::X: k[i][j] = a * smooth[i] * deriv[j]; break;
                case Direction::Y: k[i][j] = a * deriv[i] * smooth[j]; break;
                case Direction::D:
                case Direction::DT: {
                    // Kdt is Kd mirrored left-right
                    const std::size_t jj = dir == Direction::D ? j : 4 - j;
                    const int sign = kKd[i][jj][0];
                    k[i][j] = a * Rational{sign} * sym_value(kKd[i][jj][1], p);
                    break;
                }
            }
        }
    return k;
}

inline std::int32_t narrow_weight(const Rational& r, const char* kernel, int i, int j) {
    if (!r.is_integer())
        throw NonIntegralWeight(std::string(kernel) + "(" + std::to_string(i) + "," +
                                std::to_string(j) + ") = " + r.str() + " is not an integer");
    return static_cast<std::int32_t>(r.numerator());
}

}  // namespace detail

/// filter_algebra.hpp:157-188: positivity, integral weights, integral b/m/n,
/// |weight| <= 2^15 -- in that order.
inline void validate_params(const FilterParams& p) {
    if (p.a < 1) throw NonPositiveParam("a = " + std::to_string(p.a) + " must be a positive integer");
    const std::pair<const char*, const Rational*> shape[] = {{"b", &p.b}, {"m", &p.m}, {"n", &p.n}};
    for (const auto& [name, v] : shape)
        if (*v <= Rational{0}) throw NonPositiveParam(std::string(name) + " = " + v->str() + " must be positive");
    std::int64_t largest = 0;
    for (Direction d : {Direction::X, Direction::Y, Direction::D, Direction::DT}) {
        const auto k = detail::materialize_exact(p, d);
        for (int i = 0; i < 5; ++i)
            for (int j = 0; j < 5; ++j) {
                const std::int64_t v = detail::narrow_weight(
                    k[static_cast<std::size_t>(i)][static_cast<std::size_t>(j)], direction_name(d), i, j);
                largest = std::max<std::int64_t>(largest, v < 0 ? -v : v);
            }
    }
    for (const auto& [name, v] : shape)
        if (!v->is_integer())
            throw NonIntegralWeight(std::string("parameter ") + name + " = " + v->str() +
                                    " must be an integer (streaming taps are integer vectors)");
    if (largest > kMaxWeightMagnitude)
        throw ParamOverflow("largest weight magnitude " + std::to_string(largest) + " exceeds " +
                            std::to_string(kMaxWeightMagnitude));
}

inline Kernel5 materialize(const FilterParams& p, Direction dir) {
    const auto exact = detail::materialize_exact(p, dir);
    Kernel5 k;
    for (int i = 0; i < 5; ++i)
        for (int j = 0; j < 5; ++j)
            k.w[static_cast<std::size_t>(i)][static_cast<std::size_t>(j)] = detail::narrow_weight(
                exact[static_cast<std::size_t>(i)][static_cast<std::size_t>(j)], direction_name(dir), i, j);
    return k;
}

struct KdSumDiff {
    Kernel5 plus;   // Kd + Kdt (Eq. 10)
    Kernel5 minus;  // Kd - Kdt
};

inline KdSumDiff make_kd_sum_diff(const FilterParams& p) {
    const Kernel5 d = materialize(p, Direction::D), t = materialize(p, Direction::DT);
    KdSumDiff r;
    for (std::size_t i = 0; i < 5; ++i)
        for (std::size_t j = 0; j < 5; ++j) {
            r.plus.w[i][j] = d.w[i][j] + t.w[i][j];
            r.minus.w[i][j] = d.w[i][j] - t.w[i][j];
        }
    return r;
}

/// Eq. 19: Kd- = deriv_term - diff_term, both rank 1.
struct KdMinusDecomposition {
    SeparablePair deriv_term;
    SeparablePair diff_term;
};

inline KdMinusDecomposition decompose_kd_minus(const FilterParams& p) {
    auto whole = [](const Rational& r, const char* what) {
        if (!r.is_integer()) throw NonIntegralWeight(std::string(what) + " = " + r.str() + " is not an integer");
        return static_cast<std::int32_t>(r.numerator());
    };
    const Rational& b = p.b;
    const std::int32_t m = whole(p.m, "m"), nb_ = whole(p.n + b, "n+b");
    const std::int32_t t = whole(p.m * b + b - p.n, "m*b+b-n");
    const std::int32_t u = whole(p.n * b + b * b - p.m * b, "n*b+b*b-m*b");
    const std::int32_t v = whole(Rational{2} * b - Rational{2} * p.n * b, "2b-2nb");
    KdMinusDecomposition r;
    r.deriv_term.scale = static_cast<std::int32_t>(p.a);
    r.deriv_term.col = {m, nb_, 2, nb_, m};
    r.deriv_term.row = {-1, whole(-b, "-b"), 0, whole(b, "b"), 1};
    r.diff_term.scale = static_cast<std::int32_t>(p.a);
    r.diff_term.col = {t, u, v, u, t};
    r.diff_term.row = {0, -1, 0, 1, 0};
    return r;
}

/// The per-stream integer taps (reference pipeline.hpp:57-73); layout-equal
/// to sobel5_taps of the C ABI.
struct StreamTaps {
    std::int32_t a = 1;
    std::array<std::int32_t, 5> f{};
    std::array<std::int32_t, 5> h{};
    std::array<std::int32_t, 5> k0{};
    std::array<std::int32_t, 5> k1{};
    std::array<std::int32_t, 5> gx_v{};
    std::array<std::int32_t, 5> gy_v{};
    std::array<std::int32_t, 5> gdm_f{};
    std::array<std::int32_t, 5> gdm_d{};
    bool wide_vagg = false;
};

inline StreamTaps make_stream_taps(const FilterParams& p) {
    validate_params(p);
    const std::int32_t a = static_cast<std::int32_t>(p.a);
    const std::int32_t b = static_cast<std::int32_t>(p.b.as_integer());
    const std::int32_t m = static_cast<std::int32_t>(p.m.as_integer());
    const std::int32_t n = static_cast<std::int32_t>(p.n.as_integer());
    auto sym = [](std::int32_t e0, std::int32_t e1, std::int32_t e2) {
        return std::array<std::int32_t, 5>{e0, e1, e2, e1, e0};
    };
    StreamTaps t;
    t.a = a;
    t.f = {-1, -b, 0, b, 1};
    t.h = sym(1, n, m);
    t.k0 = sym(-a * m, -a * (n + b), -2 * a);
    t.k1 = sym(a * (b - n), -a * m * b, -2 * a * n * b);
    t.gx_v = sym(a, a * n, a * m);
    t.gy_v = {-a, -a * b, 0, a * b, a};
    t.gdm_f = sym(a * m, a * (n + b), 2 * a);
    t.gdm_d = sym(a * (m * b + b - n), a * (n * b + b * b - m * b), a * (2 * b - 2 * n * b));
    // the reference's int64-vs-int32 aggregation switch (pipeline.hpp:94-105)
    auto l1 = [](const std::array<std::int32_t, 5>& v) {
        std::int64_t s = 0;
        for (auto x : v) s += x < 0 ? -std::int64_t{x} : std::int64_t{x};
        return s;
    };
    const std::int64_t fmax = 255 * l1(t.f), hmax = 255 * l1(t.h);
    const std::int64_t worst =
        std::max({l1(t.gx_v) * fmax, l1(t.gy_v) * hmax, l1(t.gdm_f) * fmax + l1(t.gdm_d) * 510});
    t.wide_vagg = worst > INT32_MAX;
    return t;
}

}  // namespace sobel5
