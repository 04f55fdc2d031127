// Store-path probe 4: does a wider per-lane store (8 px per lane: one 256-bit
// STG per int plane, two per g) raise the SR write pattern above the 4-px
// pattern (128-bit int stores)?  Store-only kernels at the 8K SR geometry.
#include <cstdint>
__device__ __forceinline__ void st4(void* p, uint32_t a) {
    asm volatile("st.global.cs.v4.b32 [%0], {%1,%1,%1,%1};" ::"l"(p), "r"(a) : "memory");
}
__device__ __forceinline__ void st8(void* p, uint32_t a) {
    asm volatile("st.global.cs.v8.b32 [%0], {%1,%1,%1,%1,%1,%1,%1,%1};" ::"l"(p), "r"(a) : "memory");
}
template <int PX>  // pixels per lane: 4 or 8
__global__ void __launch_bounds__(128) reg_px(char* gx, char* gy, char* gd, char* gdt, char* g,
                                              int64_t pitch, int out_w, int out_h, int band) {
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    const int x0 = (blockIdx.x * 4 + warp) * (32 * PX) + lane * PX;
    if (x0 >= out_w) return;
    const int oy0 = blockIdx.y * band;
    const int n = min(band, out_h - oy0);
    for (int v = 0; v < n; ++v) {
        const int64_t o = static_cast<int64_t>(oy0 + v) * pitch + x0;
        const uint32_t a = v + x0;
        if (PX == 4) {
            st4(gx + o * 4, a); st4(gy + o * 4, a); st4(gd + o * 4, a); st4(gdt + o * 4, a);
            st8(g + o * 8, a);
        } else {
            st8(gx + o * 4, a); st8(gy + o * 4, a); st8(gd + o * 4, a); st8(gdt + o * 4, a);
            st8(g + o * 8, a); st8(g + o * 8 + 32, a);
        }
    }
}
template __global__ void reg_px<4>(char*, char*, char*, char*, char*, int64_t, int, int, int);
template __global__ void reg_px<8>(char*, char*, char*, char*, char*, int64_t, int, int, int);

// 4 px per lane for compute, but lane pairs exchange halves so that even
// lanes store gx and gy as 8-px (256-bit) rows and odd lanes gd and gdt;
// every lane stores its own 4 doubles of g (256-bit): 3 STG per lane-row.
__global__ void __launch_bounds__(128) reg_pair(char* gx, char* gy, char* gd, char* gdt, char* g,
                                                int64_t pitch, int out_w, int out_h, int band) {
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    const int x0 = (blockIdx.x * 4 + warp) * 128 + lane * 4;
    const int xp = x0 & ~7;  // the pair's 8-px block
    if (x0 >= out_w) return;
    const int oy0 = blockIdx.y * band;
    const int n = min(band, out_h - oy0);
    const bool odd = lane & 1;
    for (int v = 0; v < n; ++v) {
        const int64_t o = static_cast<int64_t>(oy0 + v) * pitch;
        const uint32_t a = v + x0;
        const uint32_t b = __shfl_xor_sync(0xffffffffu, a, 1);
        st8((odd ? gd : gx) + (o + xp) * 4, a ^ b);
        st8((odd ? gdt : gy) + (o + xp) * 4, a ^ b);
        st8(g + (o + x0) * 8, a);
    }
}
