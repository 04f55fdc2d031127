// sobel5_b200/core.hpp -- value types of the drop-in API: the exception
// family, row-major planes and exact rationals.
//
// Mirrors the names and semantics of the reference's errors.hpp:9-32,
// plane.hpp:14-72 and rational.hpp:17-152 so code written against the
// reference compiles unchanged; the implementation is independent.
#pragma once

#include <cstdint>
#include <numeric>
#include <optional>
#include <span>
#include <stdexcept>
#include <string>
#include <string_view>
#include <utility>
#include <vector>

namespace sobel5 {

// ---- errors (reference errors.hpp:9-32) -------------------------------------

struct Error : std::runtime_error {
    explicit Error(const std::string& what) : std::runtime_error(what) {}
};

#define SOBEL5_B200_ERROR(Name) \
    struct Name : Error {       \
        using Error::Error;     \
    }
SOBEL5_B200_ERROR(NonPositiveParam);
SOBEL5_B200_ERROR(NonIntegralWeight);
SOBEL5_B200_ERROR(ParamOverflow);
SOBEL5_B200_ERROR(ImageTooSmall);
SOBEL5_B200_ERROR(RowTooShort);
SOBEL5_B200_ERROR(MissingRow);
SOBEL5_B200_ERROR(VariantMismatch);
SOBEL5_B200_ERROR(ParityViolation);
SOBEL5_B200_ERROR(LaneTooNarrow);
SOBEL5_B200_ERROR(DimMismatch);
SOBEL5_B200_ERROR(EmptyPlane);
SOBEL5_B200_ERROR(UnsupportedFormat);
SOBEL5_B200_ERROR(CorruptFile);
SOBEL5_B200_ERROR(IoError);
SOBEL5_B200_ERROR(UnsupportedExtension);
// Not in the reference: the device path failed (CUDA error, no device, OOM).
SOBEL5_B200_ERROR(DeviceError);
#undef SOBEL5_B200_ERROR

// ---- planes (reference plane.hpp:14-72) --------------------------------------

/// Row-major, tightly packed 2-D buffer owning its pixels.
template <typename T>
class Plane {
public:
    Plane() = default;

    Plane(int width, int height) : w_(width), h_(height) {
        require_positive(width, height);
        px_.assign(static_cast<std::size_t>(width) * static_cast<std::size_t>(height), T{});
    }

    Plane(int width, int height, std::vector<T> pixels)
        : w_(width), h_(height), px_(std::move(pixels)) {
        require_positive(width, height);
        const std::size_t want = static_cast<std::size_t>(width) * static_cast<std::size_t>(height);
        if (px_.size() != want)
            throw DimMismatch("plane data length " + std::to_string(px_.size()) +
                              " does not match " + std::to_string(width) + "x" +
                              std::to_string(height));
    }

    int width() const { return w_; }
    int height() const { return h_; }
    bool empty() const { return px_.empty(); }
    std::size_t size() const { return px_.size(); }

    T& at(int y, int x) { return px_[index(y, x)]; }
    const T& at(int y, int x) const { return px_[index(y, x)]; }

    std::span<T> row(int y) { return {px_.data() + index(y, 0), static_cast<std::size_t>(w_)}; }
    std::span<const T> row(int y) const {
        return {px_.data() + index(y, 0), static_cast<std::size_t>(w_)};
    }

    std::vector<T>& data() { return px_; }
    const std::vector<T>& data() const { return px_; }

    friend bool operator==(const Plane& a, const Plane& b) {
        return a.w_ == b.w_ && a.h_ == b.h_ && a.px_ == b.px_;
    }

private:
    std::size_t index(int y, int x) const {
        return static_cast<std::size_t>(y) * static_cast<std::size_t>(w_) +
               static_cast<std::size_t>(x);
    }
    static void require_positive(int width, int height) {
        if (width > 0 && height > 0) return;
        throw DimMismatch("plane dimensions must be positive, got " + std::to_string(width) +
                          "x" + std::to_string(height));
    }

    int w_ = 0;
    int h_ = 0;
    std::vector<T> px_;
};

using GrayPlane = Plane<std::uint8_t>;
using SignedPlane = Plane<std::int32_t>;
using RealPlane = Plane<double>;

// ---- exact rationals (reference rational.hpp:17-152) ---------------------------

/// num/den over int64 with 128-bit intermediates, always reduced with den > 0.
class Rational {
public:
    constexpr Rational() = default;
    constexpr Rational(std::int64_t v) : n_(v), d_(1) {}  // NOLINT: implicit like the reference
    Rational(std::int64_t num, std::int64_t den) {
        if (den == 0) throw NonPositiveParam("rational denominator is zero");
        *this = reduce(num, den);
    }

    std::int64_t numerator() const { return n_; }
    std::int64_t denominator() const { return d_; }
    bool is_integer() const { return d_ == 1; }
    std::int64_t as_integer() const {
        if (d_ != 1) throw NonIntegralWeight("rational " + str() + " is not an integer");
        return n_;
    }
    double to_double() const { return static_cast<double>(n_) / static_cast<double>(d_); }
    std::string str() const {
        return d_ == 1 ? std::to_string(n_) : std::to_string(n_) + "/" + std::to_string(d_);
    }

    friend Rational operator+(const Rational& a, const Rational& b) {
        return reduce(W(a.n_) * b.d_ + W(b.n_) * a.d_, W(a.d_) * b.d_);
    }
    friend Rational operator-(const Rational& a, const Rational& b) {
        return reduce(W(a.n_) * b.d_ - W(b.n_) * a.d_, W(a.d_) * b.d_);
    }
    friend Rational operator*(const Rational& a, const Rational& b) {
        return reduce(W(a.n_) * b.n_, W(a.d_) * b.d_);
    }
    friend Rational operator-(const Rational& a) { return reduce(-W(a.n_), a.d_); }
    friend bool operator==(const Rational& a, const Rational& b) {
        return a.n_ == b.n_ && a.d_ == b.d_;
    }
    friend bool operator!=(const Rational& a, const Rational& b) { return !(a == b); }
    friend bool operator<(const Rational& a, const Rational& b) {
        return W(a.n_) * b.d_ < W(b.n_) * a.d_;
    }
    friend bool operator>(const Rational& a, const Rational& b) { return b < a; }
    friend bool operator<=(const Rational& a, const Rational& b) { return !(b < a); }
    friend bool operator>=(const Rational& a, const Rational& b) { return !(a < b); }

    /// "7", "-2", "3/2", "0.25"; nullopt when malformed (reference
    /// rational.hpp parse()).
    static std::optional<Rational> parse(std::string_view text) {
        if (text.empty()) return std::nullopt;
        std::size_t i = 0;
        bool negative = false;
        if (text[0] == '+' || text[0] == '-') {
            negative = text[0] == '-';
            i = 1;
        }
        std::int64_t digits = 0, scale = 1;
        bool seen_digit = false, fraction = false;
        for (; i < text.size(); ++i) {
            const char c = text[i];
            if (c >= '0' && c <= '9') {
                if (digits > (INT64_MAX - 9) / 10) return std::nullopt;
                digits = digits * 10 + (c - '0');
                seen_digit = true;
                if (fraction) {
                    if (scale > INT64_MAX / 10) return std::nullopt;
                    scale *= 10;
                }
            } else if (c == '.' && !fraction && scale == 1) {
                fraction = true;
            } else if (c == '/' && !fraction && seen_digit && i + 1 < text.size()) {
                const auto rhs = parse(text.substr(i + 1));
                if (!rhs || rhs->n_ <= 0) return std::nullopt;
                return reduce(negative ? -W(digits) : W(digits), 1) * Rational(rhs->d_, rhs->n_);
            } else {
                return std::nullopt;
            }
        }
        if (!seen_digit) return std::nullopt;
        return reduce(negative ? -W(digits) : W(digits), scale);
    }

private:
    using W = __int128;
    static Rational reduce(W num, W den) {
        if (den < 0) {
            num = -num;
            den = -den;
        }
        W a = num < 0 ? -num : num, b = den;
        while (b != 0) {
            const W t = a % b;
            a = b;
            b = t;
        }
        if (a > 1) {
            num /= a;
            den /= a;
        }
        if (num > INT64_MAX || num < INT64_MIN || den > INT64_MAX)
            throw ParamOverflow("rational arithmetic overflow");
        Rational r;
        r.n_ = static_cast<std::int64_t>(num);
        r.d_ = static_cast<std::int64_t>(den);
        return r;
    }

    std::int64_t n_ = 0;
    std::int64_t d_ = 1;
};

}  // namespace sobel5
