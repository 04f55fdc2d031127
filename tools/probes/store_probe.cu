// Store-pattern probe: the packed kernel's exact grid/CTA geometry and store
// sequence (4 x st.global.cs.v4.s32 + 2 x st.global.cs.v2.f64 per lane per
// output row), with the arithmetic removed.  Measures the write ceiling of
// the access pattern itself (tools/probes/run_probes.py).
#include <cstdint>
extern "C" __global__ void __launch_bounds__(128) store_probe(int32_t* gx, int32_t* gy, int32_t* gd,
                                                              int32_t* gdt, double* g, int64_t pitch,
                                                              int out_w, int out_h, int band, int cs) {
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    const int x0 = (blockIdx.x * 4 + warp) * 128 + lane * 4;
    if (x0 >= out_w) return;
    const int oy0 = blockIdx.y * band;
    const int n = min(band, out_h - oy0);
    for (int v = 0; v < n; ++v) {
        const int64_t o = static_cast<int64_t>(oy0 + v) * pitch + x0;
        const int a = v + x0;
        if (cs) {
            asm volatile("st.global.cs.v4.s32 [%0], {%1,%1,%1,%1};" ::"l"(gx + o), "r"(a) : "memory");
            asm volatile("st.global.cs.v4.s32 [%0], {%1,%1,%1,%1};" ::"l"(gy + o), "r"(a) : "memory");
            asm volatile("st.global.cs.v4.s32 [%0], {%1,%1,%1,%1};" ::"l"(gd + o), "r"(a) : "memory");
            asm volatile("st.global.cs.v4.s32 [%0], {%1,%1,%1,%1};" ::"l"(gdt + o), "r"(a) : "memory");
            const double d = a;
            asm volatile("st.global.cs.v2.f64 [%0], {%1,%1};" ::"l"(g + o), "d"(d) : "memory");
            asm volatile("st.global.cs.v2.f64 [%0], {%1,%1};" ::"l"(g + o + 2), "d"(d) : "memory");
        } else {
            reinterpret_cast<int4*>(gx + o)[0] = make_int4(a, a, a, a);
            reinterpret_cast<int4*>(gy + o)[0] = make_int4(a, a, a, a);
            reinterpret_cast<int4*>(gd + o)[0] = make_int4(a, a, a, a);
            reinterpret_cast<int4*>(gdt + o)[0] = make_int4(a, a, a, a);
            const double d = a;
            reinterpret_cast<double2*>(g + o)[0] = make_double2(d, d);
            reinterpret_cast<double2*>(g + o + 2)[0] = make_double2(d, d);
        }
    }
}

// Same bytes written plane-major by a trivially parallel grid (one 16-byte
// store per thread): the best case for DRAM page locality.
extern "C" __global__ void flat_probe(int4* p, int64_t n16) {
    for (int64_t i = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; i < n16;
         i += static_cast<int64_t>(gridDim.x) * blockDim.x)
        __stcs(p + i, make_int4(1, 2, 3, 4));
}
