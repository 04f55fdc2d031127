// Host side of the C++ run_stream at 8K without the GPU: five threads each
// build one result plane by appending 8 row chunks from a resident source
// (the pinned staging stand-in), with / without MADV_HUGEPAGE.
#include <sys/mman.h>
#include <chrono>
#include <cstdint>
#include <cstdio>
#include <cstring>
#include <thread>
#include <vector>
using clk = std::chrono::steady_clock;
static double ms(clk::time_point a) { return std::chrono::duration<double, std::milli>(clk::now() - a).count(); }
template <class T>
static void build(std::vector<T>& v, const T* src, size_t n, bool huge, int chunks, double* t_res, double* t_all) {
    auto t0 = clk::now();
    v.reserve(n);
    if (huge) {
        const uintptr_t p = reinterpret_cast<uintptr_t>(v.data()), H = 2u << 20;
        const uintptr_t a = (p + H - 1) & ~(H - 1), e = (p + n * sizeof(T)) & ~(H - 1);
        if (e > a) madvise(reinterpret_cast<void*>(a), e - a, MADV_HUGEPAGE);
    }
    *t_res = ms(t0);
    const size_t per = (n + chunks - 1) / chunks;
    for (size_t o = 0; o < n; o += per) v.insert(v.end(), src + o, src + std::min(n, o + per));
    *t_all = ms(t0);
}
int main() {
    const size_t n = size_t(7676) * 4316;
    std::vector<int32_t> si(n, 3);
    std::vector<double> sd(n, 1.5);
    for (int huge = 0; huge < 2; ++huge)
        for (int it = 0; it < 3; ++it) {
            std::vector<int32_t> a[4];
            std::vector<double> g;
            double r[5], t[5];
            auto t0 = clk::now();
            std::thread th[4];
            for (int i = 0; i < 4; ++i) th[i] = std::thread([&, i] { build(a[i], si.data(), n, huge, 8, &r[i], &t[i]); });
            build(g, sd.data(), n, huge, 8, &r[4], &t[4]);
            for (auto& x : th) x.join();
            double tot = ms(t0);
            std::printf("huge=%d it=%d total %.1f ms | g %.1f ms | ints %.1f %.1f %.1f %.1f ms\n", huge, it, tot, t[4], t[0], t[1], t[2], t[3]);
        }
    // g alone
    for (int huge = 0; huge < 2; ++huge) {
        std::vector<double> g; double r, t;
        build(g, sd.data(), n, huge, 8, &r, &t);
        std::printf("g alone huge=%d: %.1f ms\n", huge, t);
    }
}
