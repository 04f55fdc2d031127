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
#include <cstddef>
#include <cstdint>

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

}  // namespace

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
