// Write-bandwidth probes for B200 store patterns (see run_probes2.py).
#include <cstdint>
// flat: one contiguous buffer, VEC-byte stores per thread, grid-stride
template <int VEC, int HINT>
__device__ __forceinline__ void st(void* p, uint32_t a) {
    if (VEC == 16) {
        if (HINT == 1) asm volatile("st.global.cs.v4.b32 [%0], {%1,%1,%1,%1};" ::"l"(p), "r"(a) : "memory");
        else if (HINT == 2) asm volatile("st.global.L1::no_allocate.v4.b32 [%0], {%1,%1,%1,%1};" ::"l"(p), "r"(a) : "memory");
        else asm volatile("st.global.v4.b32 [%0], {%1,%1,%1,%1};" ::"l"(p), "r"(a) : "memory");
    } else {
        if (HINT == 1) asm volatile("st.global.cs.v8.b32 [%0], {%1,%1,%1,%1,%1,%1,%1,%1};" ::"l"(p), "r"(a) : "memory");
        else if (HINT == 2) asm volatile("st.global.L1::no_allocate.v8.b32 [%0], {%1,%1,%1,%1,%1,%1,%1,%1};" ::"l"(p), "r"(a) : "memory");
        else asm volatile("st.global.v8.b32 [%0], {%1,%1,%1,%1,%1,%1,%1,%1};" ::"l"(p), "r"(a) : "memory");
    }
}
template <int VEC, int HINT>
__global__ void flat(char* p, int64_t n) {
    for (int64_t i = (blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x) * VEC; i < n;
         i += static_cast<int64_t>(gridDim.x) * blockDim.x * VEC)
        st<VEC, HINT>(p + i, static_cast<uint32_t>(i));
}
// planes: the kernel's geometry, PX pixels per lane (4 or 8), 6 planes
// (4 x int32 + 1 x f64 as two int32-planes' worth), VEC-byte stores
template <int PX, int VEC, int HINT>
__global__ void __launch_bounds__(128) planes(char* gx, char* gy, char* gd, char* gdt, char* g,
                                              int64_t pitch, int out_w, int out_h, int band) {
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    const int x0 = (blockIdx.x * 4 + warp) * (32 * PX) + lane * PX;
    if (x0 >= out_w) return;
    const int oy0 = blockIdx.y * band;
    const int n = min(band, out_h - oy0);
    for (int v = 0; v < n; ++v) {
        const int64_t o = static_cast<int64_t>(oy0 + v) * pitch + x0;
        const uint32_t a = v + x0;
#pragma unroll
        for (int b = 0; b < PX * 4; b += VEC) {
            st<VEC, HINT>(gx + o * 4 + b, a);
            st<VEC, HINT>(gy + o * 4 + b, a);
            st<VEC, HINT>(gd + o * 4 + b, a);
            st<VEC, HINT>(gdt + o * 4 + b, a);
        }
#pragma unroll
        for (int b = 0; b < PX * 8; b += VEC) st<VEC, HINT>(g + o * 8 + b, a);
    }
}
#define INST_FLAT(V, H) template __global__ void flat<V, H>(char*, int64_t);
INST_FLAT(16, 0) INST_FLAT(16, 1) INST_FLAT(16, 2) INST_FLAT(32, 0) INST_FLAT(32, 1) INST_FLAT(32, 2)
#define INST_PL(P, V, H) template __global__ void planes<P, V, H>(char*, char*, char*, char*, char*, int64_t, int, int, int);
INST_PL(4, 16, 0) INST_PL(4, 16, 1) INST_PL(8, 16, 0) INST_PL(8, 16, 1) INST_PL(8, 32, 0) INST_PL(8, 32, 1) INST_PL(4, 16, 2) INST_PL(8, 32, 2)
