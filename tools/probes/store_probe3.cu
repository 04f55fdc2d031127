// Store-path probes for the SR contract (24 B/px over 5 planes) on B200:
// register stores (the kernel's pattern) vs TMA bulk stores (smem staging +
// cp.async.bulk.global.shared::cta) per warp and per CTA.  run_probes3.py.
#include <cstdint>

__device__ __forceinline__ void stcs4(void* p, uint32_t a) {
    asm volatile("st.global.cs.v4.b32 [%0], {%1,%1,%1,%1};" ::"l"(p), "r"(a) : "memory");
}
__device__ __forceinline__ void stcs8(void* p, uint32_t a) {
    asm volatile("st.global.cs.v8.b32 [%0], {%1,%1,%1,%1,%1,%1,%1,%1};" ::"l"(p), "r"(a) : "memory");
}
__device__ __forceinline__ uint32_t smem_u32(const void* p) {
    return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}
__device__ __forceinline__ void bulk_store(void* g, const void* s, uint32_t bytes) {
    asm volatile("cp.async.bulk.global.shared::cta.bulk_group [%0], [%1], %2;" ::"l"(g),
                 "r"(smem_u32(s)), "r"(bytes) : "memory");
}
__device__ __forceinline__ void bulk_commit() { asm volatile("cp.async.bulk.commit_group;" ::: "memory"); }
template <int N>
__device__ __forceinline__ void bulk_wait_read() {
    asm volatile("cp.async.bulk.wait_group.read %0;" ::"n"(N) : "memory");
}
__device__ __forceinline__ void fence_async_smem() {
    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
}

// baseline: the SR kernel's stores (4 px per lane, v4 int stores, v8 g store)
__global__ void __launch_bounds__(128) reg_planes(char* gx, char* gy, char* gd, char* gdt, char* g,
                                                  int64_t pitch, int out_w, int out_h, int band) {
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    const int x0 = (blockIdx.x * 4 + warp) * 128 + lane * 4;
    if (x0 >= out_w) return;
    const int oy0 = blockIdx.y * band;
    const int n = min(band, out_h - oy0);
    for (int v = 0; v < n; ++v) {
        const int64_t o = static_cast<int64_t>(oy0 + v) * pitch + x0;
        const uint32_t a = v + x0;
        stcs4(gx + o * 4, a);
        stcs4(gy + o * 4, a);
        stcs4(gd + o * 4, a);
        stcs4(gdt + o * 4, a);
        stcs8(g + o * 8, a);
    }
}

// per-warp TMA: each warp stages its row (4 x 512 B + 1 KB) in smem, lane 0
// issues five bulk stores; double buffered.
__global__ void __launch_bounds__(128) tma_warp(char* gx, char* gy, char* gd, char* gdt, char* g,
                                                int64_t pitch, int out_w, int out_h, int band) {
    __shared__ __align__(128) uint32_t stage[4][2][768];  // [warp][buf][3 KB]
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    const int wx0 = (blockIdx.x * 4 + warp) * 128;
    if (wx0 >= out_w) return;
    const int oy0 = blockIdx.y * band;
    const int n = min(band, out_h - oy0);
    for (int v = 0; v < n; ++v) {
        uint32_t* s = stage[warp][v & 1];
        if (v >= 2) {
            if (lane == 0) bulk_wait_read<1>();
            __syncwarp();
        }
        const uint32_t a = v + wx0 + lane;
        reinterpret_cast<uint4*>(s)[lane] = make_uint4(a, a, a, a);             // gx 512 B
        reinterpret_cast<uint4*>(s + 128)[lane] = make_uint4(a, a, a, a);       // gy
        reinterpret_cast<uint4*>(s + 256)[lane] = make_uint4(a, a, a, a);       // gd
        reinterpret_cast<uint4*>(s + 384)[lane] = make_uint4(a, a, a, a);       // gdt
        reinterpret_cast<uint4*>(s + 512)[2 * lane] = make_uint4(a, a, a, a);   // g 1 KB
        reinterpret_cast<uint4*>(s + 512)[2 * lane + 1] = make_uint4(a, a, a, a);
        fence_async_smem();
        __syncwarp();
        if (lane == 0) {
            const int64_t o = static_cast<int64_t>(oy0 + v) * pitch + wx0;
            bulk_store(gx + o * 4, s, 512);
            bulk_store(gy + o * 4, s + 128, 512);
            bulk_store(gd + o * 4, s + 256, 512);
            bulk_store(gdt + o * 4, s + 384, 512);
            bulk_store(g + o * 8, s + 512, 1024);
            bulk_commit();
        }
    }
    if (lane == 0) bulk_wait_read<0>();
}

// per-CTA TMA: the CTA stages 512 columns (4 x 2 KB + 4 KB) and one thread
// issues five bulk stores per row; double buffered, one barrier per row.
__global__ void __launch_bounds__(128) tma_cta(char* gx, char* gy, char* gd, char* gdt, char* g,
                                               int64_t pitch, int out_w, int out_h, int band) {
    __shared__ __align__(128) uint32_t stage[2][3072];  // [buf][12 KB]
    const int t = threadIdx.x;
    const int cx0 = blockIdx.x * 512;
    const int oy0 = blockIdx.y * band;
    const int n = min(band, out_h - oy0);
    for (int v = 0; v < n; ++v) {
        uint32_t* s = stage[v & 1];
        if (v >= 2 && t == 0) bulk_wait_read<1>();
        __syncthreads();
        const uint32_t a = v + cx0 + t;
        reinterpret_cast<uint4*>(s)[t] = make_uint4(a, a, a, a);
        reinterpret_cast<uint4*>(s + 512)[t] = make_uint4(a, a, a, a);
        reinterpret_cast<uint4*>(s + 1024)[t] = make_uint4(a, a, a, a);
        reinterpret_cast<uint4*>(s + 1536)[t] = make_uint4(a, a, a, a);
        reinterpret_cast<uint4*>(s + 2048)[2 * t] = make_uint4(a, a, a, a);
        reinterpret_cast<uint4*>(s + 2048)[2 * t + 1] = make_uint4(a, a, a, a);
        fence_async_smem();
        __syncthreads();
        if (t == 0) {
            const int64_t o = static_cast<int64_t>(oy0 + v) * pitch + cx0;
            const uint32_t cols = static_cast<uint32_t>(min(512, out_w - cx0)) & ~3u;
            bulk_store(gx + o * 4, s, cols * 4);
            bulk_store(gy + o * 4, s + 512, cols * 4);
            bulk_store(gd + o * 4, s + 1024, cols * 4);
            bulk_store(gdt + o * 4, s + 1536, cols * 4);
            bulk_store(g + o * 8, s + 2048, cols * 8);
            bulk_commit();
        }
    }
    if (t == 0) bulk_wait_read<0>();
}

// register stores with a configurable CTA width (WARPS warps side by side)
template <int WARPS>
__global__ void __launch_bounds__(32 * WARPS) reg_planes_w(char* gx, char* gy, char* gd, char* gdt,
                                                          char* g, int64_t pitch, int out_w,
                                                          int out_h, int band) {
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    const int x0 = (blockIdx.x * WARPS + warp) * 128 + lane * 4;
    if (x0 >= out_w) return;
    const int oy0 = blockIdx.y * band;
    const int n = min(band, out_h - oy0);
    for (int v = 0; v < n; ++v) {
        const int64_t o = static_cast<int64_t>(oy0 + v) * pitch + x0;
        const uint32_t a = v + x0;
        stcs4(gx + o * 4, a);
        stcs4(gy + o * 4, a);
        stcs4(gd + o * 4, a);
        stcs4(gdt + o * 4, a);
        stcs8(g + o * 8, a);
    }
}
template __global__ void reg_planes_w<1>(char*, char*, char*, char*, char*, int64_t, int, int, int);
template __global__ void reg_planes_w<2>(char*, char*, char*, char*, char*, int64_t, int, int, int);
template __global__ void reg_planes_w<8>(char*, char*, char*, char*, char*, int64_t, int, int, int);
template __global__ void reg_planes_w<16>(char*, char*, char*, char*, char*, int64_t, int, int, int);
