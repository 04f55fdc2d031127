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
    std::printf("ok %d cases\n", cases);
    return 0;
}
