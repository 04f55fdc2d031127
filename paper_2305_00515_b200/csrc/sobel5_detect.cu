// sobel5_detect.cu -- the CLI detect path on the device (SURVEY.md 8f rows
// 1-2): optional replicate padding fused into the stencil's loads, then the
// edge-map export of g (image_io.hpp:233-256) in either SaveMode, plus the
// standalone quantize of a device plane (save_plane, image_io.hpp:258-268).
//
// Reference flow (sobel5_cli.cpp:127-189): img = pad_replicate(img, r)
// (:133) -> run_stream (:160-167) -> save_plane(g, normalize) (:177).
// Here: normalize needs the frame's min/max of g before any pixel can be
// mapped, so it takes two passes:
//   init   : minmax keys <- (+inf, -inf)
//   pass 1 : stencil, optional planes, per-frame min/max of g (warp reduce +
//            one atomic per warp) and, for integer magnitudes, the exact
//            S = g^2 plane (u32, L2-resident where it fits)
//   table  : per frame, the exact threshold table of S -> u8 (256 threads)
//   pass 2 : memory-bound map of the S plane through the table (integer
//            magnitudes), or the stencil again with the double formula
#include <cuda_runtime.h>

#include <algorithm>
#include <cmath>
#include <cstdint>
#include <cstdlib>

#include "sobel5_gpu.h"
#include "sobel5_internal.h"
#include "sobel5_packed.cuh"

using namespace sobel5_b200;

namespace {

constexpr size_t kAlign = 256;

size_t align_up(size_t v) { return (v + kAlign - 1) / kAlign * kAlign; }

// Scratch layout: [minmax x frames][norm_table x frames][S plane (u32, the
// output planes' pitch and frame stride)].
size_t head_bytes(int frames) {
    return align_up(align_up(sizeof(sobel5_minmax) * frames) + sizeof(sobel5_norm_table) * frames);
}
sobel5_minmax* scratch_minmax(void* s) { return static_cast<sobel5_minmax*>(s); }
sobel5_norm_table* scratch_table(void* s, int frames) {
    return reinterpret_cast<sobel5_norm_table*>(static_cast<char*>(s) +
                                                align_up(sizeof(sobel5_minmax) * frames));
}
uint32_t* scratch_s32(void* s, int frames) {
    return reinterpret_cast<uint32_t*>(static_cast<char*>(s) + head_bytes(frames));
}

// The detect path's small kernels start with pdl_enter() and are launched
// with launch_pdl: each one's launch overlaps its predecessor's tail (pass 1
// -> table -> map), and each waits for that predecessor before any access.
__global__ void minmax_init_kernel(sobel5_minmax* mm, int frames) {
    pdl_enter();
    const int i = blockIdx.x * blockDim.x + threadIdx.x;
    if (i < frames) {
        mm[i].lo_key = ~0ull;
        mm[i].hi_key = 0ull;
    }
}

// One block per frame.  lo / hi from the keys; for integer sums of squares
// (exact_s) thread k in 1..255 binary-searches the smallest S in
// [S_lo, S_hi] whose normalized value is >= k (the map is monotone).
__global__ void norm_table_kernel(const sobel5_minmax* mm, sobel5_norm_table* tab, int exact_s,
                                  int allow_one_step) {
    pdl_enter();
    const sobel5_minmax m = mm[blockIdx.x];
    sobel5_norm_table* t = tab + blockIdx.x;
    const bool any = m.lo_key <= m.hi_key;
    const double lo = any ? dkey_value(m.lo_key) : 0.0;
    const double hi = any ? dkey_value(m.hi_key) : 0.0;
    const double span = hi - lo;  // image_io.hpp:248
    const int k = threadIdx.x;
    if (k == 0) {
        t->lo = lo;
        t->span = span;
        t->lo_f = static_cast<float>(lo);
        t->scale_f = span > 0.0 ? static_cast<float>(255.0 / span) : 0.0f;
        t->exact_s = static_cast<uint32_t>(exact_s);
        // the map's float estimate y * scale - lo * scale of m = (g - lo) *
        // 255 / span errs by a few ulps of max(hi * scale, lo * scale), so
        // it is within 1/4 of m whenever hi * 255 / span <= 2^16 (lo <= hi)
        t->one_step = (allow_one_step && exact_s && any && span > 0.0 && hi * (255.0 / span) <= 65536.0) ? 1u : 0u;
        t->thr[0] = 0u;
        t->thr[256] = 0xffffffffu;
    }
    if (k >= 1 && k <= 255) {
        uint32_t thr = 0xffffffffu;
        if (exact_s && any) {
            // g = sqrt(S) correctly rounded and S < 2^31: S = rint(g * g)
            const uint32_t s_lo = static_cast<uint32_t>(llrint(lo * lo));
            const uint32_t s_hi = static_cast<uint32_t>(llrint(hi * hi));
            auto u_of = [&](uint32_t S) { return normalize_u8(sqrt_u30(S), lo, span); };
            if (u_of(s_hi) >= static_cast<uint32_t>(k)) {
                // lround(m) >= k  <=>  m >= k - 1/2 (m >= 0): the real-valued
                // threshold seeds a short walk on the exact double map
                const double g = lo + (k - 0.5) * span / 255.0;
                double seed = ceil(g * g);
                seed = fmin(fmax(seed, static_cast<double>(s_lo)), static_cast<double>(s_hi));
                uint32_t a = static_cast<uint32_t>(seed);
                while (a > s_lo && u_of(a - 1) >= static_cast<uint32_t>(k)) --a;
                while (u_of(a) < static_cast<uint32_t>(k)) ++a;  // terminates: u(s_hi) >= k
                thr = a;
            }
        }
        t->thr[k] = thr;
    }
}

// Normalize pass 2 of the detect path (integer magnitudes): u8 from the S
// plane written by pass 1, 4 pixels per thread per row (16-byte load, 4-byte
// store), kRows rows in flight per thread.  u(S) = max{k : thr[k] <= S};
// a float estimate of (sqrt(S) - lo) * 255 / span picks k, one 8-byte
// shared load of (thr[k], thr[k+1]) confirms it -- the check is exact, so
// any estimate is safe -- and a binary search decides the rare misses
// (tiny spans, estimates off by more than one step).
__device__ __forceinline__ bool norm_check(uint32_t S, uint32_t e, const uint2* pr) {
    const uint2 t = pr[e];
    return t.x <= S && S < t.y;
}
__device__ __noinline__ uint32_t norm_search(uint32_t S, const uint32_t* thr) {
    uint32_t k = 0;
#pragma unroll
    for (uint32_t step = 128; step >= 1; step >>= 1)
        if (thr[k + step] <= S) k += step;
    return k;
}
// est -> clamp(rint(est), ., 255) via the 1.5 * 2^23 mantissa trick; a
// negative or huge estimate just lands on an entry whose check fails
__device__ __forceinline__ uint32_t est_index(float m) {
    return min(__float_as_uint(m) - 0x4B400000u, 255u);
}

// One-compare form (table one_step): with the estimate m' within 1/4 of m,
// j = round(m' + 1/2) lies in [0, 256] and leaves u(S) in {j - 1, j}, and
// u(S) >= j <=> S >= thr[j] (thr[j] is the smallest S with u >= j; thr[0] = 0
// and thr[256] = UINT32_MAX close both ends), so u = j - 1 + [S >= thr[j]]:
// I2F, MUFU.SQRT, FFMA, FADD, one 4-byte shared load and one compare per
// pixel, no clamp, no search (the unsigned min only keeps a broken estimate
// inside the table).
__device__ __forceinline__ uint32_t norm_one_step(uint32_t S, float scale, float off, const uint32_t* thr) {
    float y;
    asm("sqrt.approx.ftz.f32 %0, %1;" : "=f"(y) : "f"(__uint2float_rn(S)));
    const float m = __fadd_rn(__fmaf_rn(y, scale, off), 12582912.0f);  // off carries the + 1/2
    const uint32_t j = min(__float_as_uint(m) - 0x4B400000u, 256u);
    return j - (S < thr[j] ? 1u : 0u);
}

// One thread's 4-column slice in the one-compare form, rows y, y + step, ...
// (top to bottom: reading the S plane bottom-up to catch pass 1's last rows
// in L2 measured slower, 90.8 vs 88.2 us for the 8K detect).  FULL: all 4
// columns inside the plane (one 4-byte store per row).
template <bool FULL>
__device__ __forceinline__ void norm_one_step_rows(const uint32_t* __restrict__ s, uint8_t* __restrict__ o,
                                                   int64_t pitch, int y, int out_h, int step, int ncols,
                                                   float sc, float off, const uint32_t* thr) {
    constexpr int kRows = 4;
    for (; y < out_h; y += step) {
        uint4 S[kRows];
#pragma unroll
        for (int k = 0; k < kRows; ++k)
            if (y + k < out_h) S[k] = __ldcs(reinterpret_cast<const uint4*>(s + static_cast<int64_t>(y + k) * pitch));
#pragma unroll
        for (int k = 0; k < kRows; ++k) {
            if (y + k >= out_h) break;
            const uint32_t u0 = norm_one_step(S[k].x, sc, off, thr);
            const uint32_t u1 = norm_one_step(S[k].y, sc, off, thr);
            const uint32_t u2 = norm_one_step(S[k].z, sc, off, thr);
            const uint32_t u3 = norm_one_step(S[k].w, sc, off, thr);
            uint8_t* q = o + static_cast<int64_t>(y + k) * pitch;
            if (FULL) {
                st_cs_u32(q, pack_u8x4(u0, u1, u2, u3));
            } else {
                const uint32_t u[4] = {u0, u1, u2, u3};
                for (int j = 0; j < ncols; ++j) q[j] = static_cast<uint8_t>(u[j]);
            }
        }
    }
}

__global__ void norm_map_kernel(const uint32_t* __restrict__ s32, int64_t pitch,
                                int64_t frame_stride, int out_w, int out_h,
                                const sobel5_norm_table* __restrict__ tab, uint8_t* __restrict__ u8) {
    pdl_enter();
    __shared__ uint32_t s_thr[257];
    __shared__ uint2 s_pair[256];
    const sobel5_norm_table* t = tab + blockIdx.z;
    const bool one_step = t->one_step != 0;  // uniform per frame
    for (int i = threadIdx.x; i < 257; i += blockDim.x) s_thr[i] = t->thr[i];
    __syncthreads();
    if (!one_step)  // the search form's (thr[k], thr[k+1]) pairs
        for (int i = threadIdx.x; i < 256; i += blockDim.x) s_pair[i] = make_uint2(s_thr[i], s_thr[i + 1]);
    const float2 scale2 = make_float2(t->scale_f, t->scale_f);
    const float nlo = -t->lo_f * t->scale_f;
    const float2 off2 = make_float2(nlo, nlo);
    const float2 magic2 = make_float2(12582912.0f, 12582912.0f);
    __syncthreads();
    const int x = (blockIdx.x * blockDim.x + threadIdx.x) * 4;
    if (x >= out_w) return;
    const int64_t base = static_cast<int64_t>(blockIdx.z) * frame_stride + x;
    // kRows rows per iteration: their loads are in flight together (one
    // 16-B load per thread per row would leave HBM latency exposed)
    constexpr int kRows = 4;
    if (one_step) {
        const float sc = t->scale_f;
        const float off = __fadd_rn(-t->lo_f * sc, 0.5f);
        const int y0 = blockIdx.y * kRows, step = gridDim.y * kRows;
        if (x + 3 < out_w)
            norm_one_step_rows<true>(s32 + base, u8 + base, pitch, y0, out_h, step, 4, sc, off, s_thr);
        else
            norm_one_step_rows<false>(s32 + base, u8 + base, pitch, y0, out_h, step, out_w - x, sc, off, s_thr);
        return;
    }
    for (int y0 = blockIdx.y * kRows; y0 < out_h; y0 += gridDim.y * kRows) {
        uint4 S[kRows];
#pragma unroll
        for (int k = 0; k < kRows; ++k)
            if (y0 + k < out_h)
                S[k] = __ldcs(reinterpret_cast<const uint4*>(s32 + base + static_cast<int64_t>(y0 + k) * pitch));
#pragma unroll
        for (int k = 0; k < kRows; ++k) {
            if (y0 + k >= out_h) break;
            const int64_t o = base + static_cast<int64_t>(y0 + k) * pitch;
            const uint4 v = S[k];
            const float2 fa = make_float2(__uint2float_rn(v.x), __uint2float_rn(v.y));
            const float2 fb = make_float2(__uint2float_rn(v.z), __uint2float_rn(v.w));
            const float2 ra = make_float2(rsqrt_approx(fmaxf(fa.x, 1.0f)), rsqrt_approx(fmaxf(fa.y, 1.0f)));
            const float2 rb = make_float2(rsqrt_approx(fmaxf(fb.x, 1.0f)), rsqrt_approx(fmaxf(fb.y, 1.0f)));
            const float2 ma = __fadd2_rn(__ffma2_rn(__fmul2_rn(fa, ra), scale2, off2), magic2);
            const float2 mb = __fadd2_rn(__ffma2_rn(__fmul2_rn(fb, rb), scale2, off2), magic2);
            uint32_t u0 = est_index(ma.x), u1 = est_index(ma.y);
            uint32_t u2 = est_index(mb.x), u3 = est_index(mb.y);
            const bool k0 = norm_check(v.x, u0, s_pair), k1 = norm_check(v.y, u1, s_pair);
            const bool k2 = norm_check(v.z, u2, s_pair), k3 = norm_check(v.w, u3, s_pair);
            if (!(k0 && k1 && k2 && k3)) {  // rare: one branch per 4 pixels
                if (!k0) u0 = norm_search(v.x, s_thr);
                if (!k1) u1 = norm_search(v.y, s_thr);
                if (!k2) u2 = norm_search(v.z, s_thr);
                if (!k3) u3 = norm_search(v.w, s_thr);
            }
            if (x + 3 < out_w) {
                st_cs_u32(u8 + o, pack_u8x4(u0, u1, u2, u3));
            } else {
                const uint32_t u[4] = {u0, u1, u2, u3};
                for (int j = 0; j < 4 && x + j < out_w; ++j) u8[o + j] = static_cast<uint8_t>(u[j]);
            }
        }
    }
}

// ---- standalone quantize of a device plane (detail::quantize) ------------

template <class T>
__device__ __forceinline__ double as_double(T v) {
    return static_cast<double>(v);
}

template <class T>
__global__ void plane_minmax_kernel(const T* plane, int64_t pitch, int width, int height,
                                    sobel5_minmax* mm) {
    unsigned long long lo = ~0ull, hi = 0ull;
    // 2-D grid-stride (rows over blockIdx.y, columns over x): no per-element
    // 64-bit division
    constexpr int kU = 4;  // loads in flight per thread
    for (int y = blockIdx.y; y < height; y += gridDim.y) {
        const T* row = plane + static_cast<int64_t>(y) * pitch;
        const int stride = gridDim.x * blockDim.x;
        for (int x = blockIdx.x * blockDim.x + threadIdx.x; x < width; x += kU * stride) {
            T vals[kU];
#pragma unroll
            for (int k = 0; k < kU; ++k)
                if (x + k * stride < width) vals[k] = __ldcs(row + x + k * stride);
#pragma unroll
            for (int k = 0; k < kU; ++k) {
                if (x + k * stride >= width) break;
                const double v = as_double(vals[k]);
                if (v != v) continue;  // NaN never occurs for Sobel planes
                const unsigned long long key = dkey(v);
                lo = min(lo, key);
                hi = max(hi, key);
            }
        }
    }
    for (int o = 16; o > 0; o >>= 1) {
        lo = min(lo, __shfl_xor_sync(0xffffffffu, lo, o));
        hi = max(hi, __shfl_xor_sync(0xffffffffu, hi, o));
    }
    if ((threadIdx.x & 31) == 0 && lo <= hi) {
        atomicMin(reinterpret_cast<unsigned long long*>(&mm->lo_key), lo);
        atomicMax(reinterpret_cast<unsigned long long*>(&mm->hi_key), hi);
    }
}

// clamp_abs (image_io.hpp:235-240) or normalize (:242-255), per element.
template <class T>
__global__ void plane_map_kernel(const T* plane, int64_t pitch, int width, int height, int mode,
                                 const sobel5_norm_table* tab, uint8_t* out, int64_t out_pitch) {
    const double lo = mode ? tab->lo : 0.0, span = mode ? tab->span : 0.0;
    constexpr int kU = 4;  // loads in flight per thread
    for (int y = blockIdx.y; y < height; y += gridDim.y) {
        const T* row = plane + static_cast<int64_t>(y) * pitch;
        uint8_t* orow = out + static_cast<int64_t>(y) * out_pitch;
        const int stride = gridDim.x * blockDim.x;
        for (int x = blockIdx.x * blockDim.x + threadIdx.x; x < width; x += kU * stride) {
            T vals[kU];
#pragma unroll
            for (int k = 0; k < kU; ++k)
                if (x + k * stride < width) vals[k] = __ldcs(row + x + k * stride);
#pragma unroll
            for (int k = 0; k < kU; ++k) {
                if (x + k * stride >= width) break;
                const double v = as_double(vals[k]);
                uint32_t u;
                if (mode) {
                    u = normalize_u8(v, lo, span);
                } else {
                    const double r = round(fabs(v));
                    u = r < 255.0 ? static_cast<uint32_t>(r) : 255u;
                }
                orow[x + k * stride] = static_cast<uint8_t>(u);
            }
        }
    }
}

// SOBEL5_NORM_ONE_STEP=0 keeps every frame on the estimate-check-search map
// (tests compare both forms)
int norm_one_step_allowed() {
    const char* v = std::getenv("SOBEL5_NORM_ONE_STEP");
    return (v && std::atoi(v) == 0) ? 0 : 1;
}

sobel5_status run_init(sobel5_minmax* mm, int frames, cudaStream_t s) {
    const cudaError_t e = launch_pdl(minmax_init_kernel, dim3((frames + 127) / 128), dim3(128), s, mm, frames);
    count_launch();
    return map_cuda(e);
}

// normalize export (image_io.hpp:242-255) around a stencil launcher:
//   exact (integer S): init, pass 1 = stencil + planes + S plane + min/max,
//     table, pass 2 = S plane -> u8 (memory-bound map, no stencil rerun);
//   otherwise: init, pass 1 = stencil + planes + min/max, table (lo, span),
//     pass 2 = stencil again with the direct double formula.
template <class Launch>
sobel5_status detect_normalize(void* scratch, int frames, bool exact, const sobel5_planes* d_out,
                               int64_t out_frame_stride, void* stream, Launch&& launch,
                               const LaunchExtra& ex, sobel5_diag* d_diag, int out_w, int out_h) {
    if (out_w < 1 || out_h < 1) {
        // let the launcher report the reference's error for the size
        sobel5_planes none = *d_out;
        return launch(&none, ex, d_diag);
    }
    cudaStream_t s = static_cast<cudaStream_t>(stream);
    sobel5_minmax* mm = scratch_minmax(scratch);
    sobel5_norm_table* tab = scratch_table(scratch, frames);
    sobel5_planes p1 = *d_out;
    p1.u8 = nullptr;
    sobel5_planes p2{};
    p2.u8 = d_out->u8;
    p2.pitch = d_out->pitch;
    if (sobel5_status st = run_init(mm, frames, s); st != SOBEL5_OK) return st;
    LaunchExtra e1 = ex;
    e1.minmax = mm;
    if (exact) e1.s32 = scratch_s32(scratch, frames);
    if (sobel5_status st = launch(&p1, e1, d_diag); st != SOBEL5_OK) return st;
    if (cudaError_t e = launch_pdl(norm_table_kernel, dim3(frames), dim3(256), s, mm, tab, exact ? 1 : 0,
                                   norm_one_step_allowed());
        e != cudaSuccess)
        return map_cuda(e);
    count_launch();
    if (exact) {
        // a few thousand CTAs that loop over rows: every CTA first stages the
        // 257-entry threshold table in shared memory, so one CTA per row
        // (the first version) spent more loads on tables than on pixels
        const unsigned gx = static_cast<unsigned>((out_w + 4 * 128 - 1) / (4 * 128));
        const unsigned gy = static_cast<unsigned>(std::max(
            1, std::min((out_h + 3) / 4, static_cast<int>(148u * 16u / (gx * frames)) + 1)));
        const dim3 grid(gx, gy, static_cast<unsigned>(frames));
        const cudaError_t e = launch_pdl(norm_map_kernel, grid, dim3(128), s, e1.s32, d_out->pitch,
                                         out_frame_stride, out_w, out_h, tab, d_out->u8);
        count_launch();
        return map_cuda(e);
    }
    LaunchExtra e2 = ex;
    e2.norm = tab;
    e2.u8_norm = 1;
    return launch(&p2, e2, nullptr);
}

}  // namespace

extern "C" {

sobel5_status sobel5_launch_ex(const uint8_t* d_in, int64_t in_pitch, int64_t in_frame_stride,
                               int width, int height, int n_frames, const sobel5_taps* taps,
                               int prefetch, int pad, const sobel5_planes* d_out,
                               int64_t out_frame_stride, sobel5_diag* d_diag, void* stream) {
    LaunchExtra ex;
    ex.pad = pad ? 1 : 0;
    return launch_common(nullptr, d_in, nullptr, in_pitch, in_frame_stride, width, height,
                         n_frames, taps, prefetch, d_out, out_frame_stride, d_diag, stream, ex);
}

size_t sobel5_detect_scratch_bytes(int out_h, int64_t pitch, int64_t out_frame_stride,
                                   int n_frames) {
    if (n_frames < 1 || out_h < 0 || pitch < 0) return 0;
    const int64_t plane = (n_frames - 1) * out_frame_stride + static_cast<int64_t>(out_h) * pitch;
    return head_bytes(n_frames) + static_cast<size_t>(plane) * sizeof(uint32_t);
}

sobel5_status sobel5_detect(const uint8_t* d_in, int64_t in_pitch, int64_t in_frame_stride,
                            int width, int height, int n_frames, const sobel5_taps* taps,
                            int prefetch, int pad, int save_mode, const sobel5_planes* d_out,
                            int64_t out_frame_stride, void* d_scratch, sobel5_diag* d_diag,
                            void* stream) {
    if (!d_out || !d_out->u8 || (save_mode != 0 && save_mode != 1) || n_frames < 1)
        return SOBEL5_INVALID_ARG;
    LaunchExtra ex;
    ex.pad = pad ? 1 : 0;
    if (save_mode == 0)  // clamp_abs: one fused launch
        return launch_common(nullptr, d_in, nullptr, in_pitch, in_frame_stride, width, height,
                             n_frames, taps, prefetch, d_out, out_frame_stride, d_diag, stream, ex);
    if (!d_scratch || reinterpret_cast<uintptr_t>(d_scratch) % 256 != 0) return SOBEL5_INVALID_ARG;
    const bool exact = taps && taps_packed(taps);
    return detect_normalize(
        d_scratch, n_frames, exact, d_out, out_frame_stride, stream,
        [&](const sobel5_planes* planes, const LaunchExtra& e, sobel5_diag* dg) {
            return launch_common(nullptr, d_in, nullptr, in_pitch, in_frame_stride, width, height,
                                 n_frames, taps, prefetch, planes, out_frame_stride, dg, stream, e);
        },
        ex, d_diag, pad ? width : width - 4, pad ? height : height - 4);
}

sobel5_status sobel3_detect(const uint8_t* d_in, int64_t in_pitch, int64_t in_frame_stride,
                            int width, int height, int n_frames, int prefetch, int pad,
                            int save_mode, const sobel5_planes* d_out, int64_t out_frame_stride,
                            void* d_scratch, void* stream) {
    if (!d_out || !d_out->u8 || (save_mode != 0 && save_mode != 1) || n_frames < 1)
        return SOBEL5_INVALID_ARG;
    LaunchExtra ex;
    ex.pad = pad ? 1 : 0;
    if (save_mode == 0)
        return sobel3_common(d_in, in_pitch, in_frame_stride, width, height, n_frames, prefetch,
                             d_out, out_frame_stride, stream, ex);
    if (!d_scratch || reinterpret_cast<uintptr_t>(d_scratch) % 256 != 0) return SOBEL5_INVALID_ARG;
    return detect_normalize(
        d_scratch, n_frames, true, d_out, out_frame_stride, stream,
        [&](const sobel5_planes* planes, const LaunchExtra& e, sobel5_diag*) {
            return sobel3_common(d_in, in_pitch, in_frame_stride, width, height, n_frames,
                                 prefetch, planes, out_frame_stride, stream, e);
        },
        ex, nullptr, pad ? width : width - 2, pad ? height : height - 2);
}

sobel5_status sobel5_quantize_plane(const void* d_plane, int kind, int64_t pitch, int width,
                                    int height, int save_mode, uint8_t* d_u8, int64_t u8_pitch,
                                    void* d_scratch, void* stream) {
    // save_plane (image_io.hpp:258-268): an empty plane throws EmptyPlane
    if (width < 1 || height < 1) return SOBEL5_EMPTY_PLANE;
    if (!d_plane || !d_u8 || kind < 0 || kind > 2 || (save_mode != 0 && save_mode != 1) ||
        pitch < width || u8_pitch < width)
        return SOBEL5_INVALID_ARG;
    cudaStream_t s = static_cast<cudaStream_t>(stream);
    const unsigned bx = static_cast<unsigned>(std::min((width + 1023) / 1024, 148 * 8));
    const dim3 blocks(bx, static_cast<unsigned>(std::max(1, std::min(height, static_cast<int>(148u * 8u / bx)))));
    sobel5_norm_table* tab = nullptr;
    if (save_mode == 1) {
        if (!d_scratch || reinterpret_cast<uintptr_t>(d_scratch) % 16 != 0)
            return SOBEL5_INVALID_ARG;
        sobel5_minmax* mm = scratch_minmax(d_scratch);
        tab = scratch_table(d_scratch, 1);
        if (sobel5_status st = run_init(mm, 1, s); st != SOBEL5_OK) return st;
        if (kind == 0)
            plane_minmax_kernel<<<blocks, 256, 0, s>>>(static_cast<const double*>(d_plane), pitch,
                                                       width, height, mm);
        else if (kind == 1)
            plane_minmax_kernel<<<blocks, 256, 0, s>>>(static_cast<const int32_t*>(d_plane), pitch,
                                                       width, height, mm);
        else
            plane_minmax_kernel<<<blocks, 256, 0, s>>>(static_cast<const uint8_t*>(d_plane), pitch,
                                                       width, height, mm);
        norm_table_kernel<<<1, 256, 0, s>>>(mm, tab, 0, 0);
        count_launch(2);
        if (cudaError_t e = cudaGetLastError(); e != cudaSuccess) return map_cuda(e);
    }
    if (kind == 0)
        plane_map_kernel<<<blocks, 256, 0, s>>>(static_cast<const double*>(d_plane), pitch, width,
                                                height, save_mode, tab, d_u8, u8_pitch);
    else if (kind == 1)
        plane_map_kernel<<<blocks, 256, 0, s>>>(static_cast<const int32_t*>(d_plane), pitch, width,
                                                height, save_mode, tab, d_u8, u8_pitch);
    else
        plane_map_kernel<<<blocks, 256, 0, s>>>(static_cast<const uint8_t*>(d_plane), pitch, width,
                                                height, save_mode, tab, d_u8, u8_pitch);
    count_launch();
    return map_cuda(cudaGetLastError());
}

}  // extern "C"
