// As append_probe, plus MADV_POPULATE_WRITE of the reserved capacity split
// over P threads before the appends (kernel pre-faults, no user-space touch).
#include <sys/mman.h>
#include <sys/utsname.h>
#include <chrono>
#include <cerrno>
#include <cstdint>
#include <cstdio>
#include <cstring>
#include <thread>
#include <vector>
#ifndef MADV_POPULATE_WRITE
#define MADV_POPULATE_WRITE 23
#endif
using clk = std::chrono::steady_clock;
static double ms(clk::time_point a) { return std::chrono::duration<double, std::milli>(clk::now() - a).count(); }
struct Range { uintptr_t a, e; };
template <class T> static Range reserve_huge(std::vector<T>& v, size_t n) {
    v.reserve(n);
    const uintptr_t p = reinterpret_cast<uintptr_t>(v.data()), H = 2u << 20;
    const uintptr_t a = (p + H - 1) & ~(H - 1), e = (p + n * sizeof(T)) & ~(H - 1);
    if (e > a) madvise(reinterpret_cast<void*>(a), e - a, MADV_HUGEPAGE);
    const uintptr_t pa = p & ~uintptr_t(4095), pe = (p + n * sizeof(T) + 4095) & ~uintptr_t(4095);
    return {pa, pe};
}
int main() {
    utsname u; uname(&u); std::printf("kernel %s\n", u.release);
    const size_t n = size_t(7676) * 4316;
    std::vector<int32_t> si(n, 3);
    std::vector<double> sd(n, 1.5);
    for (int P : {4, 8, 16})
        for (int it = 0; it < 3; ++it) {
            std::vector<int32_t> a[4];
            std::vector<double> g;
            auto t0 = clk::now();
            Range r[5];
            for (int i = 0; i < 4; ++i) r[i] = reserve_huge(a[i], n);
            r[4] = reserve_huge(g, n);
            // split all ranges into P equal byte slices (2 MB granules)
            std::vector<Range> pieces;
            for (auto& x : r)
                for (uintptr_t o = x.a; o < x.e; o += (8u << 20)) pieces.push_back({o, std::min(x.e, o + (8u << 20))});
            std::vector<std::thread> th;
            std::atomic<size_t> next{0};
            int err = 0;
            for (int t = 0; t < P; ++t)
                th.emplace_back([&] {
                    for (size_t i; (i = next.fetch_add(1)) < pieces.size();)
                        if (madvise(reinterpret_cast<void*>(pieces[i].a), pieces[i].e - pieces[i].a, MADV_POPULATE_WRITE)) err = errno;
                });
            for (auto& x : th) x.join();
            double t_pop = ms(t0);
            std::thread ts[4];
            for (int i = 0; i < 4; ++i) ts[i] = std::thread([&, i] {
                const size_t per = (n + 7) / 8;
                for (size_t o = 0; o < n; o += per) a[i].insert(a[i].end(), si.data() + o, si.data() + std::min(n, o + per));
            });
            {
                const size_t per = (n + 7) / 8;
                for (size_t o = 0; o < n; o += per) g.insert(g.end(), sd.data() + o, sd.data() + std::min(n, o + per));
            }
            double t_g = ms(t0);
            for (auto& x : ts) x.join();
            std::printf("P=%2d it=%d populate %.1f ms, g done %.1f ms, total %.1f ms (err %d)\n", P, it, t_pop, t_g, ms(t0), err);
        }
}
