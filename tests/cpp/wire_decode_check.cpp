// wire_decode_check.cpp -- host side of the int16 D2H wire (sobel5_wire.cpp)
// without a GPU: widen_i16 and the rebuilt magnitude plane (magnitude_i16,
// AVX-512 / AVX2 / scalar) against the reference's formula
// (pipeline.hpp:401-407 / oracle.hpp:89-96: the left-to-right double sum of
// the squares, then sqrt), bit for bit, for random and extreme gradients,
// every destination alignment and ragged lengths.  Prints "ok" or the first
// mismatch; exit status 0 / 1.
#include <cmath>
#include <cstdint>
#include <cstdio>
#include <cstring>
#include <random>
#include <vector>

namespace sobel5_b200 {
void widen_i16(int32_t* dst, const int16_t* src, size_t n);
void magnitude_i16(double* g, const int16_t* const* src, int np, size_t n);
void decode_row_i16(int32_t* const* dst, double* g, const int16_t* const* src, int np, size_t n);
}  // namespace sobel5_b200

int main() {
    std::mt19937_64 rng(42);
    const int16_t extremes[] = {-32768, 32767, -12240, 12240, 0, 1, -1, 24480, -24480};
    int cases = 0;
    for (int np : {2, 4}) {
        for (size_t n : {size_t{0}, size_t{1}, size_t{7}, size_t{15}, size_t{16}, size_t{17},
                         size_t{63}, size_t{1000}, size_t{7676}}) {
            for (int mis = 0; mis < 8; ++mis) {  // g destination offset (elements)
                std::vector<int16_t> src[4];
                const int16_t* rows[4] = {};
                for (int p = 0; p < np; ++p) {
                    src[p].resize(n + 1);
                    for (size_t i = 0; i < n; ++i)
                        src[p][i] = (rng() & 3) == 0 ? extremes[rng() % 9]
                                                     : static_cast<int16_t>(rng() & 0xffff);
                    rows[p] = src[p].data() + (mis & 1);  // unaligned sources too
                }
                std::vector<double> g(n + 16, -1.0);
                double* gd = g.data() + mis;
                sobel5_b200::magnitude_i16(gd, rows, np, n);
                for (size_t i = 0; i < n; ++i) {
                    double s = 0.0;
                    for (int p = 0; p < np; ++p) {
                        const double v = rows[p][i];
                        s = s + v * v;
                    }
                    const double want = std::sqrt(s);
                    if (std::memcmp(&want, &gd[i], 8) != 0) {
                        std::printf("magnitude mismatch np %d n %zu mis %d i %zu: %.17g vs %.17g\n", np,
                                    n, mis, i, gd[i], want);
                        return 1;
                    }
                }
                if (g[mis + n] != -1.0 || (mis > 0 && g[mis - 1] != -1.0)) {
                    std::printf("magnitude wrote outside its row (np %d n %zu mis %d)\n", np, n, mis);
                    return 1;
                }
                std::vector<int32_t> w(n + 16, 7);
                sobel5_b200::widen_i16(w.data() + mis, rows[0], n);
                for (size_t i = 0; i < n; ++i)
                    if (w[mis + i] != rows[0][i]) {
                        std::printf("widen mismatch n %zu mis %d i %zu\n", n, mis, i);
                        return 1;
                    }
                if (w[mis + n] != 7) {
                    std::printf("widen wrote outside its row\n");
                    return 1;
                }
                ++cases;
            }
        }
    }
    // decode_row_i16: one pass when every destination can be 64-byte aligned
    // at one column (same offset mod 16 for the int32 planes, g matching),
    // two passes otherwise; either way the reference's values
    for (int np : {2, 4}) {
        for (size_t n : {size_t{1}, size_t{63}, size_t{64}, size_t{100}, size_t{1000}, size_t{7676}}) {
            for (int layout = 0; layout < 6; ++layout) {
                // layout 0..2: aligned-compatible offsets; 3: int32 planes
                // disagree; 4: g misaligned; 5: some planes skipped, no g
                std::vector<int16_t> src[4];
                const int16_t* rows[4] = {};
                for (int p = 0; p < np; ++p) {
                    src[p].resize(n);
                    for (auto& v : src[p])
                        v = (rng() & 7) == 0 ? extremes[rng() % 9] : static_cast<int16_t>(rng() & 0xffff);
                    rows[p] = src[p].data();
                }
                const int off = layout < 3 ? layout * 4 : 3;
                std::vector<std::vector<int32_t>> w32(np, std::vector<int32_t>(n + 64, 7));
                std::vector<double> g(n + 64, -1.0);
                int32_t* dst[4] = {};
                auto aligned = [](void* p) {
                    return reinterpret_cast<uintptr_t>(p) & ~uintptr_t{63};
                };
                for (int p = 0; p < np; ++p) {
                    char* base = reinterpret_cast<char*>(aligned(w32[p].data() + 16));
                    dst[p] = reinterpret_cast<int32_t*>(base) + off + (layout == 3 && p == 1 ? 1 : 0);
                    if (layout == 5 && p == 1) dst[p] = nullptr;
                }
                double* gb = reinterpret_cast<double*>(aligned(g.data() + 8)) + off % 8;  // matches the int32 planes
                if (layout == 4) gb += 1;
                if (layout == 5) gb = nullptr;
                sobel5_b200::decode_row_i16(dst, gb, rows, np, n);
                for (size_t i = 0; i < n; ++i) {
                    double acc = 0.0;
                    for (int p = 0; p < np; ++p) {
                        if (dst[p] && dst[p][i] != rows[p][i]) {
                            std::printf("decode int mismatch np %d n %zu layout %d p %d i %zu\n", np, n,
                                        layout, p, i);
                            return 1;
                        }
                        acc = acc + static_cast<double>(rows[p][i]) * rows[p][i];
                    }
                    const double want = std::sqrt(acc);
                    if (gb && std::memcmp(&want, &gb[i], 8) != 0) {
                        std::printf("decode g mismatch np %d n %zu layout %d i %zu\n", np, n, layout, i);
                        return 1;
                    }
                }
                ++cases;
            }
        }
    }
    std::printf("ok %d cases\n", cases);
    return 0;
}
