// decode_probe.cpp -- host side of the int16 wire alone on the GPU box's CPU:
// the 8K frame's decode (4 int16 planes -> 4 int32 planes + g) with T
// threads, the same without g (widening only), and plain non-temporal
// writes of the 795 MB result (the host memory write ceiling).  Tells
// whether the e2e host path is bound by the square roots, by the widening or
// by host memory.  Build: g++ -O2 -std=c++17 -pthread tools/probes/decode_probe.cpp
//   paper_2305_00515_b200/csrc/sobel5_wire.cpp -o build/decode_probe
#include <immintrin.h>

#include <chrono>
#include <cstdint>
#include <cstdio>
#include <cstring>
#include <thread>
#include <vector>

namespace sobel5_b200 {
void decode_row_i16(int32_t* const* dst, double* g, const int16_t* const* src, int np, size_t n);
}

using clk = std::chrono::steady_clock;

template <class F>
static double par_ms(int T, F&& f) {
    const auto t0 = clk::now();
    std::vector<std::thread> th;
    for (int t = 0; t < T; ++t) th.emplace_back([&, t] { f(t, T); });
    for (auto& x : th) x.join();
    return std::chrono::duration<double, std::milli>(clk::now() - t0).count();
}

__attribute__((target("avx512f"))) static void nt_fill(void* p, size_t bytes) {
    __m512i z = _mm512_set1_epi32(1);
    auto* q = static_cast<__m512i*>(p);
    for (size_t i = 0; i < bytes / 64; ++i) _mm512_stream_si512(q + i, z);
    _mm_sfence();
}

int main() {
    const int W = 7676, H = 4316;
    const size_t n = size_t(W) * H;
    std::vector<int16_t> src[4];
    for (int p = 0; p < 4; ++p) {
        src[p].resize(n);
        for (size_t i = 0; i < n; ++i) src[p][i] = int16_t((i * 2654435761u + p * 977) >> 17);
    }
    int32_t* dst[4];
    for (int p = 0; p < 4; ++p) dst[p] = static_cast<int32_t*>(aligned_alloc(64, n * 4));
    double* g = static_cast<double*>(aligned_alloc(64, n * 8));
    for (int p = 0; p < 4; ++p) std::memset(dst[p], 0, n * 4);
    std::memset(g, 0, n * 8);
    for (int T : {1, 4, 8, 16}) {
        for (int with_g = 1; with_g >= 0; --with_g) {
            double best = 1e9;
            for (int rep = 0; rep < 3; ++rep)
                best = std::min(best, par_ms(T, [&](int t, int TT) {
                    const int r0 = H * t / TT, r1 = H * (t + 1) / TT;
                    for (int r = r0; r < r1; ++r) {
                        const size_t o = size_t(r) * W;
                        int32_t* d[4] = {dst[0] + o, dst[1] + o, dst[2] + o, dst[3] + o};
                        const int16_t* s[4] = {src[0].data() + o, src[1].data() + o, src[2].data() + o,
                                               src[3].data() + o};
                        sobel5_b200::decode_row_i16(d, with_g ? g + o : nullptr, s, 4, W);
                    }
                }));
            std::printf("decode T=%2d %s: %6.2f ms\n", T, with_g ? "widen+g " : "widen   ", best);
        }
        double best = 1e9;
        for (int rep = 0; rep < 3; ++rep)
            best = std::min(best, par_ms(T, [&](int t, int TT) {
                for (int p = 0; p < 5; ++p) {
                    char* b = p < 4 ? reinterpret_cast<char*>(dst[p]) : reinterpret_cast<char*>(g);
                    const size_t bytes = (p < 4 ? n * 4 : n * 8) & ~size_t(63);
                    const size_t a = bytes / 64 * t / TT * 64, e = bytes / 64 * (t + 1) / TT * 64;
                    nt_fill(b + a, e - a);
                }
            }));
        std::printf("nt-write 795 MB T=%2d: %6.2f ms (%.1f GB/s)\n", T, best, n * 24 / best / 1e6);
    }
    return 0;
}
