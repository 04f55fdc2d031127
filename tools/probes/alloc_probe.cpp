// Host-side cost of value-initialised result planes (4 x int32 + f64 at 8K =
// 795 MB), and what madvise(MADV_HUGEPAGE) on the reserved capacity and
// threading do to it.  Run on the GPU box's host.
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
static void make(std::vector<T>& v, size_t n, bool huge) {
    v.reserve(n);
    if (huge) {
        const uintptr_t p = reinterpret_cast<uintptr_t>(v.data());
        const uintptr_t a = (p + (2u << 20) - 1) & ~uintptr_t((2u << 20) - 1);
        const uintptr_t e = (p + n * sizeof(T)) & ~uintptr_t((2u << 20) - 1);
        if (e > a) madvise(reinterpret_cast<void*>(a), e - a, MADV_HUGEPAGE);
    }
    v.resize(n);
}
int main() {
    const size_t n = size_t(7676) * 4316;
    for (int huge = 0; huge < 2; ++huge)
        for (int it = 0; it < 3; ++it) {
            auto t0 = clk::now();
            {
                std::vector<int32_t> a, b, c, d; std::vector<double> g;
                make(a, n, huge); make(b, n, huge); make(c, n, huge); make(d, n, huge); make(g, n, huge);
            }
            double serial = ms(t0);
            t0 = clk::now();
            {
                std::vector<int32_t> a, b, c, d; std::vector<double> g;
                std::thread t1([&] { make(a, n, huge); }), t2([&] { make(b, n, huge); }),
                    t3([&] { make(c, n, huge); }), t4([&] { make(d, n, huge); }), t5([&] { make(g, n, huge); });
                t1.join(); t2.join(); t3.join(); t4.join(); t5.join();
            }
            std::printf("huge=%d iter %d: serial %.1f ms, 5 threads %.1f ms\n", huge, it, serial, ms(t0));
        }
    std::vector<char> s(n * 8, 1), t(n * 8, 0);
    for (int th : {1, 4, 8, 16}) {
        auto t0 = clk::now();
        std::vector<std::thread> ts;
        const size_t per = s.size() / th;
        for (int k = 0; k < th; ++k)
            ts.emplace_back([&, k] { std::memcpy(t.data() + k * per, s.data() + k * per, per); });
        for (auto& x : ts) x.join();
        double m = ms(t0);
        std::printf("memcpy 265MB resident, %2d threads: %.1f ms (%.1f GB/s)\n", th, m, s.size() / m / 1e6);
    }
    FILE* f = std::fopen("/sys/kernel/mm/transparent_hugepage/enabled", "r");
    char buf[256] = {};
    if (f) { if (!std::fgets(buf, sizeof buf, f)) buf[0] = 0; std::fclose(f); }
    std::printf("THP: %s", buf);
}
