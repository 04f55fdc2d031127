// sobel5_wire.cpp -- host side of the int16 D2H wire (sobel5_ctx.cu).
//
// With default taps every gradient of the packed kernel lies in
// [-2^15, 2^15), so the host path ships gx, gy, gd, gdt as int16 over PCIe
// (16 instead of 24 B/px with g) and the host sign-extends each row chunk
// into the caller's int32 planes while later chunks are still on the wire.
// This is the widening: AVX2 sign extension with non-temporal stores (the
// destination planes are written once and not re-read here), scalar
// elsewhere.  The values are copied, never computed: the result is the
// int32 plane the device would have written.
//
// The magnitude plane g is a function of the four gradients alone
// (pipeline.hpp:401-407: the left-to-right double sum of their squares, then
// sqrt), so by default it does not cross PCIe at all (8 instead of 16 B/px):
// the host rebuilds it from the int16 rows it is widening.  With default
// taps every square is < 2^30 and the sum < 2^32, so each partial sum is an
// exact double whatever the order and the IEEE square root (vsqrtpd, like
// the device's __dsqrt_rn of the exact integer sum) gives the same bits the
// reference computes.
#include <cmath>
#include <cstddef>
#include <cstdint>
#include <cstdlib>
#include <cstring>

#if defined(__x86_64__) || defined(__i386__)
#include <immintrin.h>
#define SOBEL5_WIRE_X86 1
#endif

namespace sobel5_b200 {

namespace {

void widen_scalar(int32_t* dst, const int16_t* src, size_t n) {
    for (size_t i = 0; i < n; ++i) dst[i] = src[i];
}

#ifdef SOBEL5_WIRE_X86
__attribute__((target("avx2"))) void widen_avx2(int32_t* dst, const int16_t* src, size_t n) {
    size_t i = 0;
    // scalar head until dst is 32-byte aligned (streaming stores need it)
    while (i < n && (reinterpret_cast<uintptr_t>(dst + i) & 31u) != 0) {
        dst[i] = src[i];
        ++i;
    }
    for (; i + 16 <= n; i += 16) {
        const __m256i a = _mm256_loadu_si256(reinterpret_cast<const __m256i*>(src + i));
        _mm256_stream_si256(reinterpret_cast<__m256i*>(dst + i),
                            _mm256_cvtepi16_epi32(_mm256_castsi256_si128(a)));
        _mm256_stream_si256(reinterpret_cast<__m256i*>(dst + i + 8),
                            _mm256_cvtepi16_epi32(_mm256_extracti128_si256(a, 1)));
    }
    for (; i < n; ++i) dst[i] = src[i];
    _mm_sfence();  // order the streaming stores before the caller's handoff
}
#endif

void magnitude_scalar(double* g, const int16_t* const* src, int np, size_t n) {
    for (size_t i = 0; i < n; ++i) {
        double acc = 0.0;
        for (int p = 0; p < np; ++p) {
            const double v = src[p][i];
            acc = acc + v * v;
        }
        g[i] = std::sqrt(acc);
    }
}

#ifdef SOBEL5_WIRE_X86
template <int NP>
__attribute__((target("avx512f"))) void magnitude_avx512(double* g, const int16_t* const* src,
                                                         size_t n) {
    size_t i = 0;
    // scalar head until g is 64-byte aligned (streaming stores need it)
    for (; i < n && (reinterpret_cast<uintptr_t>(g + i) & 63u) != 0; ++i) {
        double acc = 0.0;
        for (int p = 0; p < NP; ++p) acc = acc + static_cast<double>(src[p][i]) * src[p][i];
        g[i] = std::sqrt(acc);
    }
    for (; i + 16 <= n; i += 16) {
        __m512d lo = _mm512_setzero_pd(), hi = _mm512_setzero_pd();
#pragma GCC unroll 4
        for (int p = 0; p < NP; ++p) {
            const __m512i v = _mm512_cvtepi16_epi32(
                _mm256_loadu_si256(reinterpret_cast<const __m256i*>(src[p] + i)));
            const __m512d a = _mm512_cvtepi32_pd(_mm512_castsi512_si256(v));
            const __m512d b = _mm512_cvtepi32_pd(_mm512_extracti64x4_epi64(v, 1));
            lo = _mm512_fmadd_pd(a, a, lo);  // exact: every partial sum < 2^53
            hi = _mm512_fmadd_pd(b, b, hi);
        }
        _mm512_stream_pd(g + i, _mm512_sqrt_pd(lo));
        _mm512_stream_pd(g + i + 8, _mm512_sqrt_pd(hi));
    }
    for (; i < n; ++i) {
        double acc = 0.0;
        for (int p = 0; p < NP; ++p) acc = acc + static_cast<double>(src[p][i]) * src[p][i];
        g[i] = std::sqrt(acc);
    }
    _mm_sfence();
}

template <int NP>
__attribute__((target("avx2,fma"))) void magnitude_avx2(double* g, const int16_t* const* src,
                                                        size_t n) {
    size_t i = 0;
    for (; i < n && (reinterpret_cast<uintptr_t>(g + i) & 31u) != 0; ++i) {
        double acc = 0.0;
        for (int p = 0; p < NP; ++p) acc = acc + static_cast<double>(src[p][i]) * src[p][i];
        g[i] = std::sqrt(acc);
    }
    for (; i + 8 <= n; i += 8) {
        __m256d lo = _mm256_setzero_pd(), hi = _mm256_setzero_pd();
        for (int p = 0; p < NP; ++p) {
            const __m256i v = _mm256_cvtepi16_epi32(
                _mm_loadu_si128(reinterpret_cast<const __m128i*>(src[p] + i)));
            const __m256d a = _mm256_cvtepi32_pd(_mm256_castsi256_si128(v));
            const __m256d b = _mm256_cvtepi32_pd(_mm256_extracti128_si256(v, 1));
            lo = _mm256_fmadd_pd(a, a, lo);
            hi = _mm256_fmadd_pd(b, b, hi);
        }
        _mm256_stream_pd(g + i, _mm256_sqrt_pd(lo));
        _mm256_stream_pd(g + i + 4, _mm256_sqrt_pd(hi));
    }
    for (; i < n; ++i) {
        double acc = 0.0;
        for (int p = 0; p < NP; ++p) acc = acc + static_cast<double>(src[p][i]) * src[p][i];
        g[i] = std::sqrt(acc);
    }
    _mm_sfence();
}

// One row in ONE pass (AVX-512): per 16 pixels the np int16 rows are loaded
// once, sign-extended and streamed to the int32 planes, and g is built from
// the same registers -- 1.5x the single-core rate of widen-then-magnitude
// (the host path is bound by per-core store throughput).  Needs a column
// where every destination is 64-byte aligned at once; the caller falls back
// to the two-pass form otherwise.
template <int NP>
__attribute__((target("avx512f"))) void decode_fused_avx512(int32_t* const* dst, double* g,
                                                            const int16_t* const* src, size_t i0,
                                                            size_t n) {
    auto scalar = [&](size_t i) {
        double acc = 0.0;
        for (int p = 0; p < NP; ++p) {
            dst[p][i] = src[p][i];
            acc = acc + static_cast<double>(src[p][i]) * src[p][i];
        }
        g[i] = std::sqrt(acc);
    };
    size_t i = 0;
    for (; i < i0 && i < n; ++i) scalar(i);
    for (; i + 16 <= n; i += 16) {
        __m512d lo = _mm512_setzero_pd(), hi = _mm512_setzero_pd();
#pragma GCC unroll 4
        for (int p = 0; p < NP; ++p) {
            const __m512i v = _mm512_cvtepi16_epi32(
                _mm256_loadu_si256(reinterpret_cast<const __m256i*>(src[p] + i)));
            _mm512_stream_si512(reinterpret_cast<__m512i*>(dst[p] + i), v);
            const __m512d a = _mm512_cvtepi32_pd(_mm512_castsi512_si256(v));
            const __m512d b = _mm512_cvtepi32_pd(_mm512_extracti64x4_epi64(v, 1));
            lo = _mm512_fmadd_pd(a, a, lo);  // exact: every partial sum < 2^53
            hi = _mm512_fmadd_pd(b, b, hi);
        }
        _mm512_stream_pd(g + i, _mm512_sqrt_pd(lo));
        _mm512_stream_pd(g + i + 8, _mm512_sqrt_pd(hi));
    }
    for (; i < n; ++i) scalar(i);
    _mm_sfence();
}
#endif

}  // namespace

void widen_i16(int32_t* dst, const int16_t* src, size_t n);
void magnitude_i16(double* g, const int16_t* const* src, int np, size_t n);

namespace {
// 2: AVX-512, 1: AVX2 + FMA, 0: scalar; SOBEL5_WIRE_ISA=avx2 / scalar
// narrows the choice (tests)
int wire_isa() {
#ifdef SOBEL5_WIRE_X86
    static const int isa = [] {
        const char* v = std::getenv("SOBEL5_WIRE_ISA");
        const bool scalar = v && std::strcmp(v, "scalar") == 0;
        const bool narrow2 = v && std::strcmp(v, "avx2") == 0;
        if (scalar) return 0;
        if (!narrow2 && __builtin_cpu_supports("avx512f")) return 2;
        return __builtin_cpu_supports("avx2") && __builtin_cpu_supports("fma") ? 1 : 0;
    }();
    return isa;
#else
    return 0;
#endif
}
}  // namespace

void decode_row_i16(int32_t* const* dst, double* g, const int16_t* const* src, int np, size_t n) {
#ifdef SOBEL5_WIRE_X86
    bool all = g != nullptr && (np == 2 || np == 4) && n >= 64 && wire_isa() == 2;
    for (int p = 0; p < np && all; ++p) all = dst[p] != nullptr;
    if (all) {
        // the first column where every destination is 64-byte aligned: the
        // int32 planes must agree mod 64, g must be aligned there too
        const uintptr_t a0 = reinterpret_cast<uintptr_t>(dst[0]);
        bool ok = (a0 & 3u) == 0;
        for (int p = 1; p < np && ok; ++p) ok = ((reinterpret_cast<uintptr_t>(dst[p]) - a0) & 63u) == 0;
        const size_t i0 = ((64 - (a0 & 63u)) & 63u) / 4;
        ok = ok && (reinterpret_cast<uintptr_t>(g + i0) & 63u) == 0;
        if (ok) {
            np == 4 ? decode_fused_avx512<4>(dst, g, src, i0, n)
                    : decode_fused_avx512<2>(dst, g, src, i0, n);
            return;
        }
    }
#endif
    for (int p = 0; p < np; ++p)
        if (dst[p]) widen_i16(dst[p], src[p], n);
    if (g) magnitude_i16(g, src, np, n);
}

void magnitude_i16(double* g, const int16_t* const* src, int np, size_t n) {
#ifdef SOBEL5_WIRE_X86
    const int isa = wire_isa();
    if ((np == 2 || np == 4) && isa > 0) {
        if (isa == 2) {
            np == 4 ? magnitude_avx512<4>(g, src, n) : magnitude_avx512<2>(g, src, n);
        } else {
            np == 4 ? magnitude_avx2<4>(g, src, n) : magnitude_avx2<2>(g, src, n);
        }
        return;
    }
#endif
    magnitude_scalar(g, src, np, n);
}

void widen_i16(int32_t* dst, const int16_t* src, size_t n) {
#ifdef SOBEL5_WIRE_X86
    static const bool avx2 = __builtin_cpu_supports("avx2");
    if (avx2) {
        widen_avx2(dst, src, n);
        return;
    }
#endif
    widen_scalar(dst, src, n);
}

}  // namespace sobel5_b200
