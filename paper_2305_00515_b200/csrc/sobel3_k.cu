// sobel3_k.cu -- the 3x3 operator's launches and C ABI:
// run_stream_3x3 (reference pipeline.hpp:551-573) and the detect path with
// --op sobel3_2d (sobel5_cli.cpp:128-149, pad radius 1).
#include <cuda_runtime.h>

#include <cstdint>
#include <cstdlib>
#include <cstring>

#include "sobel3_packed.cuh"
#include "sobel5_gpu.h"
#include "sobel5_internal.h"

namespace sobel5_b200 {

namespace {

constexpr int kOut3 = kOutGx | kOutGy | kOutG;  // Stream3Result

template <int PF, bool PAD, int OUTS>
cudaError_t go(const KernelParams& kp, dim3 grid, cudaStream_t s) {
    if (PF > 0 && kp.tma_load)  // band rows by TMA (sobel3_common decides)
        return launch_kp(sobel3_packed_kernel<0, PAD, OUTS, true>, grid, kCtaThreads, 0, s, kp);
    return launch_kp(sobel3_packed_kernel<PF, PAD, OUTS>, grid, kCtaThreads, 0, s, kp);
}

template <int PF, bool PAD>
cudaError_t outs(const KernelParams& kp, dim3 grid, cudaStream_t s) {
    switch (packed_out_set(kp)) {
        case kOut3: return go<PF, PAD, kOut3>(kp, grid, s);
        case kOut3 | kOutN16: return go<PF, PAD, kOut3 | kOutN16>(kp, grid, s);
        case kOutGx | kOutGy | kOutN16: return go<PF, PAD, kOutGx | kOutGy | kOutN16>(kp, grid, s);
        case kOutU8: return go<PF, PAD, kOutU8>(kp, grid, s);
        case kOutMinMax: return go<PF, PAD, kOutMinMax>(kp, grid, s);
        case kOutMinMax | kOutS32: return go<PF, PAD, kOutMinMax | kOutS32>(kp, grid, s);
        case kOutU8 | kOutNorm: return go<PF, PAD, kOutU8 | kOutNorm>(kp, grid, s);
        default: return go<PF, PAD, kOutRuntime>(kp, grid, s);
    }
}

}  // namespace

sobel5_status sobel3_common(const uint8_t* d_in, int64_t in_pitch, int64_t in_frame_stride,
                            int width, int height, int frames, int prefetch,
                            const sobel5_planes* out, int64_t out_frame_stride, void* stream,
                            const LaunchExtra& ex) {
    if (ex.pad) {
        if (width < 1 || height < 1) return SOBEL5_EMPTY_PLANE;  // image_io.hpp:280
    } else if (width < 3 || height < 3) {
        return SOBEL5_IMAGE_TOO_SMALL;  // pipeline.hpp:553-556
    }
    if (!d_in || frames < 1 || frames > 65535) return SOBEL5_INVALID_ARG;
    if (in_pitch < (width + 3) / 4 * 4 || in_pitch % 16 != 0 ||
        reinterpret_cast<uintptr_t>(d_in) % 16 != 0)
        return SOBEL5_INVALID_ARG;
    if (frames > 1 && (in_frame_stride % 16 != 0 || out_frame_stride % 4 != 0))
        return SOBEL5_INVALID_ARG;
    const int out_w = ex.pad ? width : width - 2;
    const int out_h = ex.pad ? height : height - 2;
    if (sobel5_status st = check_planes(out, out_w); st != SOBEL5_OK) return st;
    if (out->gd || out->gdt) return SOBEL5_INVALID_ARG;  // the 3x3 operator has no diagonals
    if (ex.n16 && (ex.pad || !out->gx || !out->gy || out->g32 || out->u8 || ex.minmax ||
                   ex.norm || ex.u8_norm || ex.s32))
        return SOBEL5_INVALID_ARG;  // the int16 wire: gx, gy (+ g), valid mode
    if (ex.u8_norm && (!ex.norm || !out->u8)) return SOBEL5_INVALID_ARG;

    KernelParams kp{};
    kp.mid = d_in;
    kp.in_pitch = in_pitch;
    kp.in_frame_stride = in_frame_stride;
    kp.mid_rows = height;
    kp.width = width;
    kp.out_w = out_w;
    kp.out_h = out_h;
    kp.band = choose_band(out_w, out_h, frames, !(out->gx || out->gy || out->g || out->g32));
    kp.gx = out->gx;
    kp.gy = out->gy;
    kp.g = out->g;
    kp.g32 = out->g32;
    kp.u8 = out->u8;
    kp.pitch = out->pitch;
    kp.out_frame_stride = out_frame_stride;
    kp.pad = ex.pad;
    kp.minmax = ex.minmax;
    kp.norm = ex.norm;
    kp.u8_norm = ex.u8_norm;
    kp.s32 = ex.s32;
    kp.n16 = ex.n16;
    // the write-bound Stream3Result contract reads its band rows by TMA, as the
    // 5x5 kernel does, with 4-row bands (8K: 89.6 vs 91.3 us at 8; 2r = 2 halo
    // rows per band), SOBEL5_TMA_LOAD=0 disables it
    const bool wide = out->gx || out->gy || out->g || out->g32;
    const char* tv = std::getenv("SOBEL5_TMA_LOAD");
    const char* bv = std::getenv("SOBEL5_BAND");
    const char* tp = std::getenv("SOBEL5_TMA_PAD");
    const bool tma_on = !(tv && *tv && std::atoi(tv) == 0);
    kp.tma_load = (prefetch && !ex.pad && wide && !ex.norm && tma_on) ? 1 : 0;
    if (kp.tma_load && !(bv && *bv && std::atoi(bv) > 0)) {
        const int64_t cols = (out_w + kCtaCols - 1) / kCtaCols;  // many waves only
        if (cols * frames * ((out_h + 7) / 8) >= 148 * 4 * 8) kp.band = 4;
        else kp.tma_load = 0;
    }
    unsigned gy = static_cast<unsigned>((out_h + kp.band - 1) / kp.band);
    if (gy > 65535u) {
        kp.band = (out_h + 65534) / 65535;
        gy = static_cast<unsigned>((out_h + kp.band - 1) / kp.band);
    }
    // replicate padding (detect --op sobel3_2d): clamped rows by TMA for the
    // wide planes and the narrow passes, as in the 5x5 kernel
    if (prefetch && ex.pad && tma_on && !(tp && *tp && std::atoi(tp) == 0) && !ex.norm &&
        (wide || (out->u8 && !ex.u8_norm) || (ex.minmax && ex.s32)))
        kp.tma_load = 1;
    if (kp.band > 32) kp.tma_load = 0;  // the shared-memory band holds 34 rows
    // the clamp_abs edge map alone: its own kernel (sobel3_u8.cuh: TMA band
    // rows, 8 px per lane as packed pairs, float epilogue); SOBEL5_U8_FAST=0
    // keeps kernel C (ablation)
    const char* fv = std::getenv("SOBEL5_U8_FAST");
    if (prefetch && out->u8 && !wide && !ex.minmax && !ex.norm && !ex.u8_norm && !ex.s32 &&
        out->pitch % 8 == 0 && reinterpret_cast<uintptr_t>(out->u8) % 8 == 0 &&
        (frames == 1 || out_frame_stride % 8 == 0) && !(fv && *fv && std::atoi(fv) == 0)) {
        const U8Plan up = u3_fast_plan(out_w, out_h, frames);
        if ((out_h + up.band - 1) / up.band <= 65535) {
            kp.band = up.band;
            kp.tma_load = 1;
            count_launch();
            return map_cuda(launch_u3_fast(kp, frames, up, static_cast<cudaStream_t>(stream)));
        }
    }
    const dim3 grid(static_cast<unsigned>((out_w + kCtaCols - 1) / kCtaCols), gy,
                    static_cast<unsigned>(frames));
    count_launch();
    cudaStream_t s = static_cast<cudaStream_t>(stream);
    cudaError_t e;
    if (ex.pad) e = prefetch ? outs<1, true>(kp, grid, s) : outs<0, true>(kp, grid, s);
    else e = prefetch ? outs<1, false>(kp, grid, s) : outs<0, false>(kp, grid, s);
    return map_cuda(e);
}

}  // namespace sobel5_b200

using namespace sobel5_b200;

extern "C" {

sobel5_status sobel3_launch(const uint8_t* d_in, int64_t in_pitch, int64_t in_frame_stride,
                            int width, int height, int n_frames, int prefetch, int pad,
                            const sobel5_planes* d_out, int64_t out_frame_stride, void* stream) {
    LaunchExtra ex;
    ex.pad = pad ? 1 : 0;
    return sobel3_common(d_in, in_pitch, in_frame_stride, width, height, n_frames, prefetch, d_out,
                         out_frame_stride, stream, ex);
}

sobel5_status sobel3_plan_counters(int height, const int* strip_out_w, int n_strips, int prefetch,
                                   sobel5_counters* out) {
    if (!out || (n_strips > 0 && !strip_out_w) || height < 3) return SOBEL5_INVALID_ARG;
    // run_strip_3x3 tallies (pipeline.hpp:488-547): per strip one hpass per
    // input row (3 primed + one per later centre, either prefetch mode) and
    // 5 MACs per output pixel for the hpass plus 5 per centre.
    (void)prefetch;
    uint64_t width_sum = 0;
    for (int i = 0; i < n_strips; ++i) {
        if (strip_out_w[i] <= 0) return SOBEL5_INVALID_ARG;
        width_sum += static_cast<uint64_t>(strip_out_w[i]);
    }
    const uint64_t H = static_cast<uint64_t>(height), S = static_cast<uint64_t>(n_strips);
    std::memset(out, 0, sizeof *out);
    out->row_conv3_f = H * S;
    out->row_conv3_h = H * S;
    out->mac = 5 * (H + (H - 2)) * width_sum;
    return SOBEL5_OK;
}

}  // extern "C"
