// sobel5_abi.cu -- the extern "C" boundary (include/sobel5_gpu.h): argument
// validation in the reference's order, kernel selection, device launch
// entry points, and the host-buffer path with chunked copy/compute overlap.
//
// Reference interface replaced: sobel5::run_stream (pipeline.hpp:452-477).
// No CPU fallback exists: without a device every compute entry point returns
// SOBEL5_NO_DEVICE / SOBEL5_CUDA_ERROR.
#include <cuda_runtime.h>

#include <algorithm>
#include <atomic>
#include <cstdint>
#include <cstdlib>
#include <cstring>
#include <string>
#include <vector>

#include "sobel5_gpu.h"
#include "sobel5_packed.cuh"
#include "sobel5_u8.cuh"
#include <algorithm>
#include "sobel5_internal.h"
#include "sobel5_stream.cuh"

using namespace sobel5_b200;

namespace {

std::atomic<uint64_t> g_launches{0};
thread_local sobel5_launch_info t_last_launch{};

constexpr int64_t kMaxWeight = int64_t{1} << 15;  // filter_algebra.hpp:148

int64_t round_up(int64_t v, int64_t m) { return (v + m - 1) / m * m; }

// ---- taps analysis ---------------------------------------------------------

bool taps_are_default(const sobel5_taps& t) {
    const DefaultTaps d;
    (void)d;
    for (int i = 0; i < 5; ++i) {
        if (t.f[i] != DefaultTaps::f[i] || t.h[i] != DefaultTaps::h[i] ||
            t.k0[i] != DefaultTaps::k0[i] || t.k1[i] != DefaultTaps::k1[i] ||
            t.gx_v[i] != DefaultTaps::gx_v[i] || t.gy_v[i] != DefaultTaps::gy_v[i] ||
            t.gdm_f[i] != DefaultTaps::gdm_f[i] || t.gdm_d[i] != DefaultTaps::gdm_d[i])
            return false;
    }
    return true;
}

// 255 * max(sum of positive weights, sum of |negative weights|): the largest
// |response| of a 5x5 integer kernel over uint8 input.
int64_t response_bound(const int64_t k[25]) {
    int64_t pos = 0, neg = 0;
    for (int i = 0; i < 25; ++i) (k[i] > 0 ? pos : neg) += k[i] > 0 ? k[i] : -k[i];
    return 255 * std::max(pos, neg);
}

// The effective 5x5 kernels of the streaming schedule for arbitrary taps,
// and from them whether the exact integer sum of squares fits uint32 (then
// double(S) and the reference's double sum are the same number).
MagMode choose_mag(const sobel5_taps& t) {
    int64_t kx[25], ky[25], kp[25], km[25];
    const int64_t dd[5] = {0, -1, 0, 1, 0};
    for (int i = 0; i < 5; ++i)
        for (int j = 0; j < 5; ++j) {
            kx[i * 5 + j] = int64_t{t.gx_v[i]} * t.f[j];
            ky[i * 5 + j] = int64_t{t.gy_v[i]} * t.h[j];
            km[i * 5 + j] = int64_t{t.gdm_f[i]} * t.f[j] - int64_t{t.gdm_d[i]} * dd[j];
            const int64_t kpr[5] = {t.k0[j], t.k1[j], 0, -int64_t{t.k1[j]}, -int64_t{t.k0[j]}};
            kp[i * 5 + j] = kpr[i];
        }
    const int64_t bx = response_bound(kx), by = response_bound(ky);
    const int64_t bp = response_bound(kp), bm = response_bound(km);
    const int64_t lim = int64_t{1} << 31;
    if (bx >= lim || by >= lim || bp + bm >= lim) return kMagF64;
    const int64_t bd = (bp + bm) / 2;
    const unsigned __int128 S = (unsigned __int128)(bx * bx) + (unsigned __int128)(by * by) +
                                2 * (unsigned __int128)(bd * bd);
    return S < ((unsigned __int128)1 << 32) ? kMagU32 : kMagF64;
}

// The packed (two pixels per register) kernel is exact for ANY taps whose
// extracted quantities -- gx, gy and the P / M diagonal sums -- stay within
// int16 for every uint8 input: all arithmetic before the extraction is mod
// 2^32 (a ring homomorphism), so only the final values must fit a lane.
bool taps_fit_packed(const sobel5_taps& t) {
    int64_t kx[25], ky[25], kp[25], km[25];
    const int64_t dd[5] = {0, -1, 0, 1, 0};
    for (int i = 0; i < 5; ++i)
        for (int j = 0; j < 5; ++j) {
            kx[i * 5 + j] = int64_t{t.gx_v[i]} * t.f[j];
            ky[i * 5 + j] = int64_t{t.gy_v[i]} * t.h[j];
            km[i * 5 + j] = int64_t{t.gdm_f[i]} * t.f[j] - int64_t{t.gdm_d[i]} * dd[j];
            const int64_t kpr[5] = {t.k0[j], t.k1[j], 0, -int64_t{t.k1[j]}, -int64_t{t.k0[j]}};
            kp[i * 5 + j] = kpr[i];
        }
    constexpr int64_t lim = 32767;
    return response_bound(kx) <= lim && response_bound(ky) <= lim && response_bound(kp) <= lim &&
           response_bound(km) <= lim;
}

// The packed-FP32 kernel (sobel5_f32x2.cuh) is exact for taps whose every
// partial sum stays an integer below 2^24 and whose final gx, gy, P, M and
// P +- M fit the 1.5 * 2^23 conversion (< 2^22): bounded by 255 times the
// absolute tap sums of each stage.  Every tap must itself be exact in FP32.
bool taps_fit_f32(const sobel5_taps& t) {
    auto abs_sum = [](const int32_t* v) {
        int64_t s = 0;
        for (int i = 0; i < 5; ++i) s += v[i] < 0 ? -int64_t{v[i]} : int64_t{v[i]};
        return s;
    };
    const int32_t* all[8] = {t.f, t.h, t.k0, t.k1, t.gx_v, t.gy_v, t.gdm_f, t.gdm_d};
    for (const int32_t* v : all)
        for (int i = 0; i < 5; ++i)
            if (v[i] >= (1 << 24) || v[i] <= -(1 << 24)) return false;
    const int64_t sf = abs_sum(t.f), sh = abs_sum(t.h), s0 = abs_sum(t.k0), s1 = abs_sum(t.k1);
    const int64_t bx = 255 * abs_sum(t.gx_v) * sf;
    const int64_t by = 255 * abs_sum(t.gy_v) * sh;
    const int64_t bm = 255 * (abs_sum(t.gdm_f) * sf + abs_sum(t.gdm_d));
    const int64_t bp = 255 * 2 * (s0 + s1);
    constexpr int64_t lim = int64_t{1} << 22;
    return bx < lim && by < lim && bp + bm < lim;
}

int env_int(const char* name, int dflt) {
    const char* v = std::getenv(name);
    return v && *v ? std::atoi(v) : dflt;
}

// Output rows per CTA band.  Small bands cost 4/band extra halo rows of
// horizontal work; large ones leave too few CTAs to fill 148 SMs.
int choose_band_impl(int out_w, int out_h, int frames, bool narrow_only) {
    const int forced = env_int("SOBEL5_BAND", 0);
    if (forced > 0) return forced;
    const int64_t cols = (out_w + kCtaCols - 1) / kCtaCols;
    auto ctas = [&](int band) { return cols * frames * ((out_h + band - 1) / band); };
    if (!narrow_only) {
        // Wide planes (the write-bound contracts): 16-row bands.  Shorter
        // bands help the bare HBM write pattern (store-only probe: band 4 /
        // 8 / 16 = 122 / 125 / 134 us at 8K) and the plain default-taps SR
        // kernel by ~1% at band 8, but cost 3-10% on every issue-bound
        // variant (generic taps, pad, prefetch off, SR32); taller bands lose
        // 2-6% (256x1080p, 32768^2: profiles/r1/band_sweep.txt).  Images too
        // small to fill one wave of CTAs get shorter bands.
        int band = 16;
        while (band > 4 && ctas(band) < 148 * 4) band /= 2;
        return band;
    }
    // u8-only / detect passes are issue-bound and prefer taller bands (the
    // 4 halo rows are 4/band of the row work): 8K u8 57.5 us at 32 vs 59.7
    // at 16 and 64; keep >= ~16 CTAs per SM for the last partial wave.
    int band = 64;
    while (band > 32 && ctas(band) < 148 * 16) band /= 2;
    // images too small for one wave of CTAs (~5 u8 CTAs per SM): shorter
    // bands until it is filled (1080p u8: band 32 -> 6, 9.7 -> 6.1 us; 4K:
    // 32 -> 24, 17.5 -> 16.1 us; profiles/r1/u8_band_sweep.txt)
    if (ctas(band) < 148 * 5) {
        const int64_t per_col = (148 * 5 + cols * frames - 1) / (cols * frames);  // bands wanted
        band = static_cast<int>(std::max<int64_t>(4, (out_h + per_col - 1) / per_col));
    }
    return band;
}

void fill_taps(KernelParams& kp, const sobel5_taps& t) {
    std::memcpy(kp.f, t.f, sizeof kp.f);
    std::memcpy(kp.h, t.h, sizeof kp.h);
    std::memcpy(kp.k0, t.k0, sizeof kp.k0);
    std::memcpy(kp.k1, t.k1, sizeof kp.k1);
    std::memcpy(kp.gx_v, t.gx_v, sizeof kp.gx_v);
    std::memcpy(kp.gy_v, t.gy_v, sizeof kp.gy_v);
    std::memcpy(kp.gdm_f, t.gdm_f, sizeof kp.gdm_f);
    std::memcpy(kp.gdm_d, t.gdm_d, sizeof kp.gdm_d);
    const int32_t* src[8] = {t.f, t.h, t.k0, t.k1, t.gx_v, t.gy_v, t.gdm_f, t.gdm_d};
    for (int q = 0; q < 8; ++q)
        for (int i = 0; i < 5; ++i)
            kp.tf[q][i] = static_cast<float>(q == 7 ? -static_cast<int64_t>(src[q][i]) : src[q][i]);
}

bool aligned(const void* p, uintptr_t a) { return (reinterpret_cast<uintptr_t>(p) % a) == 0; }

sobel5_status check_planes_impl(const sobel5_planes* o, int out_w) {
    if (!o) return SOBEL5_INVALID_ARG;
    if (o->pitch < out_w || o->pitch % 4 != 0) return SOBEL5_INVALID_ARG;
    const void* ps[7] = {o->gx, o->gy, o->gd, o->gdt, o->g, o->g32, o->u8};
    for (const void* q : ps)
        if (q && !aligned(q, 32)) return SOBEL5_INVALID_ARG;
    return SOBEL5_OK;
}

bool taps_fit_packed_p(const KernelParams& kp) {
    sobel5_taps t{};
    std::memcpy(t.f, kp.f, sizeof t.f);
    std::memcpy(t.h, kp.h, sizeof t.h);
    std::memcpy(t.k0, kp.k0, sizeof t.k0);
    std::memcpy(t.k1, kp.k1, sizeof t.k1);
    std::memcpy(t.gx_v, kp.gx_v, sizeof t.gx_v);
    std::memcpy(t.gy_v, kp.gy_v, sizeof t.gy_v);
    std::memcpy(t.gdm_f, kp.gdm_f, sizeof t.gdm_f);
    std::memcpy(t.gdm_d, kp.gdm_d, sizeof t.gdm_d);
    return taps_fit_packed(t);
}

bool taps_fit_f32_p(const KernelParams& kp) {
    sobel5_taps t{};
    std::memcpy(t.f, kp.f, sizeof t.f);
    std::memcpy(t.h, kp.h, sizeof t.h);
    std::memcpy(t.k0, kp.k0, sizeof t.k0);
    std::memcpy(t.k1, kp.k1, sizeof t.k1);
    std::memcpy(t.gx_v, kp.gx_v, sizeof t.gx_v);
    std::memcpy(t.gy_v, kp.gy_v, sizeof t.gy_v);
    std::memcpy(t.gdm_f, kp.gdm_f, sizeof t.gdm_f);
    std::memcpy(t.gdm_d, kp.gdm_d, sizeof t.gdm_d);
    return taps_fit_f32(t);
}

cudaError_t dispatch(const KernelParams& kp, dim3 grid, int prefetch, bool dflt, MagMode mag,
                     cudaStream_t s) {
    g_launches.fetch_add(1, std::memory_order_relaxed);
    if (dflt && env_int("SOBEL5_DENSE", 0) != 0 && !kp.pad && kp.top_rows == 0 && !kp.bot &&
        grid.z == 1 && (packed_out_set(kp) == kOutSR || packed_out_set(kp) == kOutU8)) {
        // ablation only: four dense 5x5 correlations, no operator
        // transformation (sobel5_k_dense.cu)
        return launch_dense_ablation(kp, grid, s);
    }
    if (dflt && env_int("SOBEL5_GENERIC", 0) == 0) {
        // default taps: packed two-pixels-per-register kernel (sobel5_packed.cuh)
        if (kp.pad) return launch_packed_pad(kp, grid, prefetch, s);
        const bool seg = kp.top_rows > 0 || kp.bot != nullptr;
        return seg ? launch_packed_seg(kp, grid, prefetch, s)
                   : launch_packed_plain(kp, grid, prefetch, s);
    }
    if (env_int("SOBEL5_GENERIC", 0) == 0 && taps_fit_packed_p(kp)) {
        // any other taps within the int16 bound: packed kernel, runtime taps
        if (kp.pad) return launch_packed_rt_pad(kp, grid, prefetch, s);
        const bool seg = kp.top_rows > 0 || kp.bot != nullptr;
        return seg ? launch_packed_rt_seg(kp, grid, prefetch, s)
                   : launch_packed_rt_plain(kp, grid, prefetch, s);
    }
    if (env_int("SOBEL5_GENERIC", 0) == 0 && taps_fit_f32_p(kp)) {
        // taps beyond the int16 lanes but within 2^22: packed FP32
        return launch_f32(kp, grid, prefetch, mag, s);
    }
    return launch_generic(kp, grid, prefetch, dflt, mag, s);
}

}  // namespace

namespace sobel5_b200 {

bool pdl_enabled() {
    static const bool on = env_int("SOBEL5_PDL", 1) != 0;
    return on;
}

bool taps_default(const sobel5_taps* t) { return taps_are_default(*t); }
bool n16_wire_ok(const sobel5_taps* t) {
    return t && taps_are_default(*t) && env_int("SOBEL5_WIRE16", 1) != 0 &&
           env_int("SOBEL5_GENERIC", 0) == 0 && env_int("SOBEL5_DENSE", 0) == 0;
}
bool taps_packed(const sobel5_taps* t) {
    return env_int("SOBEL5_GENERIC", 0) == 0 && (taps_are_default(*t) || taps_fit_packed(*t));
}
int choose_band(int out_w, int out_h, int frames, bool narrow_only) {
    return choose_band_impl(out_w, out_h, frames, narrow_only);
}
sobel5_status check_planes(const sobel5_planes* o, int out_w) { return check_planes_impl(o, out_w); }

void count_launch(int n) { g_launches.fetch_add(static_cast<uint64_t>(n), std::memory_order_relaxed); }

sobel5_status map_cuda(cudaError_t e) {
    if (e == cudaSuccess) return SOBEL5_OK;
    if (e == cudaErrorMemoryAllocation) return SOBEL5_OUT_OF_MEMORY;
    if (e == cudaErrorNoDevice || e == cudaErrorInsufficientDriver) return SOBEL5_NO_DEVICE;
    return SOBEL5_CUDA_ERROR;
}

// Common launch path for plain, batched, band and detect launches.
sobel5_status launch_common(const uint8_t* top, const uint8_t* mid, const uint8_t* bot,
                            int64_t in_pitch, int64_t in_frame_stride, int width, int mid_rows,
                            int frames, const sobel5_taps* taps, int prefetch,
                            const sobel5_planes* out, int64_t out_frame_stride,
                            sobel5_diag* diag, void* stream, const LaunchExtra& ex) {
    const int top_rows = top ? 2 : 0, bot_rows = bot ? 2 : 0;
    const int64_t rows = int64_t{top_rows} + mid_rows + bot_rows;
    if (ex.pad) {
        // pad_replicate(img, 2) (image_io.hpp:279-281): empty input throws
        // EmptyPlane; the padded image is then >= 5x5
        if (width < 1 || mid_rows < 1) return SOBEL5_EMPTY_PLANE;
        if (top || bot) return SOBEL5_INVALID_ARG;
    } else if (width < 5 || rows < 5) {
        // run_stream validation order: size first (pipeline.hpp:454-456)
        return SOBEL5_IMAGE_TOO_SMALL;
    }
    if (!taps || !mid || frames < 1) return SOBEL5_INVALID_ARG;
    if (diag && !aligned(diag, 16)) return SOBEL5_INVALID_ARG;  // 16-byte CAS word
    if (in_pitch < round_up(width, 4) || in_pitch % 16 != 0) return SOBEL5_INVALID_ARG;
    if (!aligned(mid, 16) || (top && !aligned(top, 16)) || (bot && !aligned(bot, 16)))
        return SOBEL5_INVALID_ARG;
    if (frames > 1 && (in_frame_stride % 16 != 0 || out_frame_stride % 4 != 0))
        return SOBEL5_INVALID_ARG;
    const int out_w = ex.pad ? width : width - 4;
    const int out_h = static_cast<int>(ex.pad ? rows : rows - 4);
    if (sobel5_status st = check_planes(out, out_w); st != SOBEL5_OK) return st;
    if (ex.u8_norm && (!ex.norm || !out->u8)) return SOBEL5_INVALID_ARG;
    // the S plane exists only for the packed kernels (exact integer S)
    if (ex.s32 && !taps_packed(taps)) return SOBEL5_INVALID_ARG;
    if (rows > (int64_t{1} << 30) || frames > 65535) return SOBEL5_INVALID_ARG;
    if (ex.n16 && (top || bot || ex.pad || !n16_wire_ok(taps) || !out->gx || !out->gy ||
                   !out->gd || !out->gdt || out->g32 || out->u8 || ex.minmax ||
                   ex.norm || ex.u8_norm || ex.s32))
        return SOBEL5_INVALID_ARG;

    KernelParams kp{};
    kp.top = top;
    kp.mid = mid;
    kp.bot = bot;
    kp.in_pitch = in_pitch;
    kp.in_frame_stride = in_frame_stride;
    kp.top_rows = top_rows;
    kp.mid_rows = mid_rows;
    kp.width = width;
    kp.frames = frames;
    kp.out_w = out_w;
    kp.out_h = out_h;
    const bool wide = out->gx || out->gy || out->gd || out->gdt || out->g || out->g32;
    kp.band = choose_band(out_w, out_h, frames, !wide);
    // Write-bound contracts of the default-taps kernel on plain images: the
    // CTA's band rows come in by TMA bulk copies (kGeomPlainTma), with short
    // bands (8K SR: 142.2 us register ring, band 16 -> 137.1 us TMA, band 8;
    // with the rows read from shared memory when consumed SR32 gains too
    // (117.3 vs 119.1 us); the u8-only contract stays 4-8% faster on the
    // register ring, and so
    // does the runtime-taps packed kernel (171 vs 150 us at 8-row bands);
    // profiles/r1/tma_load.txt).  SOBEL5_TMA_LOAD=0 disables it.
    // Stacked bands (C5, halos possibly in a peer GPU's memory): only the CTAs
    // whose rows are all in `mid` bulk-copy them (kGeomSegTma).
    // (opt-in SOBEL5_F32_TMA=1: kernel F, the packed-FP32 kernel of larger
    // taps, with TMA band rows on plain images -- measured slower at every
    // band, 8K (2,3,5,7) SR 182.8 us at 16 rows vs 168.5 on the register
    // ring: it is bound by its FFMA2 chains, not by the row loads;
    // profiles/r2/f32_tma.txt)
    const bool f32_tma = !taps_are_default(*taps) && !taps_fit_packed(*taps) && taps_fit_f32(*taps) &&
                         !ex.pad && !top && !bot && env_int("SOBEL5_F32_TMA", 0) != 0;
    kp.tma_load = (prefetch && (!ex.pad || env_int("SOBEL5_TMA_PAD", 1) != 0) &&
                   ((!top && !bot) || env_int("SOBEL5_TMA_SEG", 1) != 0) &&
                   (out->g || out->g32) && (taps_are_default(*taps) || f32_tma) &&
                   env_int("SOBEL5_TMA_LOAD", 1) != 0 && env_int("SOBEL5_GENERIC", 0) == 0 &&
                   env_int("SOBEL5_DENSE", 0) == 0 && !(ex.u8_norm || ex.norm))
                      ? 1
                      : 0;
    if (kp.tma_load && env_int("SOBEL5_BAND", 0) <= 0) {
        // worth it with many waves of 8-row CTAs (8K: 8100 CTAs); a 4K image
        // (2160) is faster on the register ring with 16-row bands
        // (39.3 vs 41.3 us, profiles/r1/tma_load.txt)
        const int64_t cols = (out_w + kCtaCols - 1) / kCtaCols;
        // bands of 6 rows for the plain StreamResult up to ~300 M output px
        // (8K bench.py interleaved: 134.9 vs 135.9 us at 8), 8 above (C4
        // 256 x 1080p: 238 vs 226 Gpx/s, C5 32K: 246 vs 235 -- long launches
        // run into the power cap, and the shorter bands' extra halo reads
        // cost more there), 8 padded (133.7 vs 135.8 at 6), 10 for SR32
        // (113.1 vs 117.4 us at 8), 12 for big SR32 (C4: 269.8 vs 265 / 261
        // Gpx/s at 10 / 8; profiles/r1/tma_load.txt)
        const bool big = int64_t{out_w} * out_h * frames > (int64_t{300} << 20);
        if (cols * frames * ((out_h + 7) / 8) >= 148 * 4 * 8)
            kp.band = !out->g ? (big ? 12 : 10) : (ex.pad || big) ? 8 : 6;
        else kp.tma_load = 0;
    }
    // The detect path's padded narrow passes (clamp_abs u8 map; normalize
    // pass 1 = min/max + S plane) read their clamped rows by TMA too, at
    // their own band: 8K pad clamp_abs 68.4 -> 59.6 us, pad normalize
    // 113.3 -> 103.1 us (the plain u8 map stays on the register ring:
    // 53.4 vs 51.1 us; profiles/r1/tma_load.txt).
    if (!kp.tma_load && ex.pad && prefetch && !wide && env_int("SOBEL5_TMA_LOAD", 1) != 0 &&
        env_int("SOBEL5_TMA_PAD", 1) != 0 &&
        ((out->u8 && !(ex.u8_norm || ex.norm)) || (ex.minmax && ex.s32)) && taps_are_default(*taps))
        kp.tma_load = 1;
    if (kp.band > 32) kp.tma_load = 0;  // the shared-memory band holds 36 rows
    // Opt-in (SOBEL5_TS=1 per-CTA boxes, 2 per-warp boxes): the plain
    // StreamResult with TMA band rows written by TMA tensor stores (two staged
    // rows per box) instead of register stores.  Measured slower at every band
    // (8K: 142.4 / 142.8 us at band 8 vs 131.7 us; 32768 x 8192: 1096 vs
    // 1069 us; profiles/r2/tma_store.txt): the staging round trip and the
    // per-CTA store drain cost more than the write pattern gains, so register
    // stores stay the default.
    const bool sr_only = out->gx && out->gy && out->gd && out->gdt && out->g && !out->g32 &&
                         !out->u8 && !ex.minmax && !ex.s32 && !ex.norm && !ex.u8_norm && !ex.n16;
    kp.gx = out->gx;
    kp.gy = out->gy;
    kp.gd = out->gd;
    kp.gdt = out->gdt;
    kp.g = out->g;
    kp.g32 = out->g32;
    kp.u8 = out->u8;
    kp.pitch = out->pitch;
    kp.out_frame_stride = out_frame_stride;
    kp.diag = diag;
    kp.need_mag = (out->g || out->g32 || out->u8 || ex.minmax) ? 1 : 0;
    kp.pad = ex.pad;
    kp.minmax = ex.minmax;
    kp.norm = ex.norm;
    kp.u8_norm = ex.u8_norm;
    kp.s32 = ex.s32;
    kp.n16 = ex.n16;
    kp.diag_frame0 = ex.frame0;
    kp.diag_row0 = ex.row0;
    fill_taps(kp, *taps);
    kp.tstore = 0;
    if (kp.tma_load && sr_only && !ex.pad && !top && !bot && env_int("SOBEL5_TS", 0) != 0) {
        if (env_int("SOBEL5_BAND", 0) <= 0) kp.band = env_int("SOBEL5_TS_BAND", 8);
        const int mode = env_int("SOBEL5_TS", 0);  // 1: CTA boxes, 2: per-warp boxes
        if (kp.band <= kTsBandRows - 4 && kp.band % kTsRows == 0 &&
            build_store_maps(kp, frames, kTsRows, mode == 2 ? kWarpCols : kTsBoxCols))
            kp.tstore = mode;
    }

    const dim3 grid(static_cast<unsigned>((out_w + kCtaCols - 1) / kCtaCols),
                    static_cast<unsigned>((out_h + kp.band - 1) / kp.band),
                    static_cast<unsigned>(frames));
    if (grid.y > 65535u) {
        // very tall images: grow the band until the grid fits
        kp.band = (out_h + 65534) / 65535;
        if (kp.band > 32) kp.tma_load = 0;  // the shared-memory band holds 36 rows
        if (kp.band > kTsBandRows - 4 || kp.band % kTsRows != 0) kp.tstore = 0;
    }
    const dim3 grid2(grid.x, static_cast<unsigned>((out_h + kp.band - 1) / kp.band), grid.z);
    // The u8-only clamp_abs edge map with default taps (plain / batch /
    // replicate-padded): the issue-bound contract has its own kernel
    // (sobel5_u8.cuh: packed pairs, ring vertical pass, TMA band rows).  SOBEL5_U8_FAST=0 keeps
    // the general packed kernel (ablation).
    // The normalize export's pass 1 (the exact S plane + the frame's min / max,
    // nothing else) runs on the same kernel in its S mode.
    const bool u8_only = out->u8 && !ex.minmax && !ex.norm && !ex.u8_norm && !ex.s32 &&
                         aligned(out->u8, 8);
    const bool s_pass = !out->u8 && ex.minmax && ex.s32 && !ex.norm && !ex.u8_norm &&
                        aligned(ex.s32, 32);
    if (prefetch && !top && !bot && !wide && (u8_only || s_pass) && taps_are_default(*taps) &&
        out->pitch % 8 == 0 && (frames == 1 || out_frame_stride % 8 == 0) &&
        env_int("SOBEL5_U8_FAST", 1) != 0 && env_int("SOBEL5_GENERIC", 0) == 0 &&
        env_int("SOBEL5_DENSE", 0) == 0) {
        const U8Plan u8p = u8_fast_plan(out_w, out_h, frames);
        kp.band = u8p.band;
        const int gy = (out_h + kp.band - 1) / kp.band;
        if (gy <= 65535) {
            kp.tma_load = 1;
            t_last_launch = sobel5_launch_info{kp.band, 1, sobel5_kernel_for_taps(taps),
                                               (out_w + u8p.cta_cols - 1) / u8p.cta_cols, gy, frames};
            count_launch();
            return map_cuda(launch_u8_fast(kp, frames, u8p, static_cast<cudaStream_t>(stream)));
        }
    }
    t_last_launch = sobel5_launch_info{kp.band, kp.tma_load, sobel5_kernel_for_taps(taps),
                                       static_cast<int>(grid2.x), static_cast<int>(grid2.y),
                                       static_cast<int>(grid2.z)};
    const cudaError_t e = dispatch(kp, grid2, prefetch, taps_are_default(*taps), choose_mag(*taps),
                                   static_cast<cudaStream_t>(stream));
    return map_cuda(e);
}

}  // namespace sobel5_b200

namespace {

// Device-side synth_random (synth.hpp:11-35), random-access form:
// pixel i = byte (i mod 8) of splitmix64 output word floor(i/8), where word
// k is mix(seed + (k+1) * 0x9E3779B97F4A7C15).
__device__ __forceinline__ uint64_t splitmix64_mix(uint64_t z) {
    z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ULL;
    z = (z ^ (z >> 27)) * 0x94D049BB133111EBULL;
    return z ^ (z >> 31);
}

__global__ void synth_random_kernel(uint8_t* img, int64_t pitch, int width, int height,
                                    int64_t row_offset, uint64_t seed, uint8_t mask) {
    const int64_t x = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
    const int y = blockIdx.y;
    if (x >= width || y >= height) return;
    const uint64_t i = static_cast<uint64_t>(row_offset + y) * static_cast<uint64_t>(width) +
                       static_cast<uint64_t>(x);
    const uint64_t word = splitmix64_mix(seed + (i / 8 + 1) * 0x9E3779B97F4A7C15ULL);
    img[static_cast<int64_t>(y) * pitch + x] =
        static_cast<uint8_t>((word >> (8 * (i % 8))) & 0xff) & mask;
}


__global__ void selftest_kernel(int which, uint32_t lo, uint32_t hi,
                                unsigned long long* count) {
    unsigned long long bad = 0;
    for (uint64_t s = lo + static_cast<uint64_t>(blockIdx.x) * blockDim.x + threadIdx.x; s < hi;
         s += static_cast<uint64_t>(gridDim.x) * blockDim.x) {
        const uint32_t S = static_cast<uint32_t>(s);
        if (which == 0) {
            const double a = sqrt_u30(S), b = __dsqrt_rn(static_cast<double>(S));
            bad += __double_as_longlong(a) != __double_as_longlong(b);
        } else if (which == 1) {
            const double g = __dsqrt_rn(static_cast<double>(S));
            const double r = round(g);
            const uint32_t want = r < 255.0 ? static_cast<uint32_t>(r) : 255u;
            bad += u8_from_s(S) != want;
        } else if (which == 2) {
            // packed-float u8 epilogue on exact integer sums S <= 65280
            if (S > 65280u) continue;
            const double r = round(__dsqrt_rn(static_cast<double>(S)));
            const uint32_t want = r < 255.0 ? static_cast<uint32_t>(r) : 255u;
            uint32_t a, b;
            u8_from_sf2(make_float2(static_cast<float>(S), static_cast<float>(S)), a, b);
            bad += (a != want) + (b != want);
        } else if (which == 4) {
            // the u8-only kernel's sqrt + saturating round (sobel5_u8.cuh) on
            // every exact integer sum S <= 65280
            if (S > 65280u) continue;
            const double r = round(__dsqrt_rn(static_cast<double>(S)));
            const uint32_t want = r < 255.0 ? static_cast<uint32_t>(r) : 255u;
            bad += (u8_round_sqrt(static_cast<float>(S)) & 0xffu) != want;
        } else if (which == 5) {
            // ... and on every float sum >= 65281 (S = float bit pattern)
            const float f = __uint_as_float(S);
            if (!(f >= 65281.0f) || isinf(f)) continue;
            bad += (u8_round_sqrt(f) & 0xffu) != 255u;
        } else {
            // ... and on every float sum >= 65281 (S = float bit pattern)
            const float f = __uint_as_float(S);
            if (!(f >= 65281.0f) || isinf(f)) continue;
            uint32_t a, b;
            u8_from_sf2(make_float2(f, f), a, b);
            bad += (a != 255u) + (b != 255u);
        }
    }
    if (bad) atomicAdd(count, bad);
}

}  // namespace

// ============================================================================
extern "C" {

int sobel5_abi_version(void) { return SOBEL5_GPU_ABI_VERSION; }

uint64_t sobel5_launch_count(void) { return g_launches.load(); }

sobel5_status sobel5_last_launch(sobel5_launch_info* out) {
    if (!out) return SOBEL5_INVALID_ARG;
    *out = t_last_launch;
    return SOBEL5_OK;
}

const char* sobel5_status_string(int status) {
    switch (status) {
        case SOBEL5_OK: return "ok";
        case SOBEL5_IMAGE_TOO_SMALL: return "image too small (need at least 5x5)";
        case SOBEL5_DIM_MISMATCH: return "dimension mismatch";
        case SOBEL5_PARITY_VIOLATION: return "odd sum/difference pair";
        case SOBEL5_INVALID_ARG: return "invalid argument";
        case SOBEL5_CUDA_ERROR: return "CUDA error";
        case SOBEL5_OUT_OF_MEMORY: return "out of memory";
        case SOBEL5_NON_POSITIVE_PARAM: return "non-positive filter parameter";
        case SOBEL5_PARAM_OVERFLOW: return "filter weight magnitude exceeds 2^15";
        case SOBEL5_LANE_TOO_NARROW: return "lane width too narrow";
        case SOBEL5_NO_DEVICE: return "no CUDA device";
        case SOBEL5_EMPTY_PLANE: return "cannot pad an empty image";
        default: return "unknown status";
    }
}

sobel5_status sobel5_make_taps(int64_t a, int64_t b, int64_t m, int64_t n, sobel5_taps* t) {
    if (!t) return SOBEL5_INVALID_ARG;
    // validate_params order (filter_algebra.hpp:158-165): a, then b, m, n
    if (a < 1 || b <= 0 || m <= 0 || n <= 0) return SOBEL5_NON_POSITIVE_PARAM;
    // every materialized weight is a*{1, b, m, n, mb, nb} (filter_algebra.hpp:82-134)
    if (a > kMaxWeight || b > kMaxWeight || m > kMaxWeight || n > kMaxWeight)
        return SOBEL5_PARAM_OVERFLOW;
    const int64_t mag = a * std::max({int64_t{1}, b, m, n, m * b, n * b});
    if (mag > kMaxWeight) return SOBEL5_PARAM_OVERFLOW;
    const int32_t A = static_cast<int32_t>(a), B = static_cast<int32_t>(b),
                  M = static_cast<int32_t>(m), N = static_cast<int32_t>(n);
    // make_stream_taps (pipeline.hpp:82-92)
    const int32_t f[5] = {-1, -B, 0, B, 1};
    const int32_t h[5] = {1, N, M, N, 1};
    const int32_t k0[5] = {-A * M, -A * (N + B), -2 * A, -A * (N + B), -A * M};
    const int32_t k1[5] = {A * (B - N), -A * M * B, -2 * A * N * B, -A * M * B, A * (B - N)};
    const int32_t gx_v[5] = {A, A * N, A * M, A * N, A};
    const int32_t gy_v[5] = {-A, -A * B, 0, A * B, A};
    const int32_t gdm_f[5] = {A * M, A * (N + B), 2 * A, A * (N + B), A * M};
    const int32_t t0 = A * (M * B + B - N), t1 = A * (N * B + B * B - M * B),
                  t2 = A * (2 * B - 2 * N * B);
    const int32_t gdm_d[5] = {t0, t1, t2, t1, t0};
    t->a = A;
    std::memcpy(t->f, f, sizeof f);
    std::memcpy(t->h, h, sizeof h);
    std::memcpy(t->k0, k0, sizeof k0);
    std::memcpy(t->k1, k1, sizeof k1);
    std::memcpy(t->gx_v, gx_v, sizeof gx_v);
    std::memcpy(t->gy_v, gy_v, sizeof gy_v);
    std::memcpy(t->gdm_f, gdm_f, sizeof gdm_f);
    std::memcpy(t->gdm_d, gdm_d, sizeof gdm_d);
    // wide_vagg (pipeline.hpp:94-105)
    auto abs_sum = [](const int32_t* v) {
        int64_t s = 0;
        for (int i = 0; i < 5; ++i) s += v[i] < 0 ? -int64_t{v[i]} : int64_t{v[i]};
        return s;
    };
    const int64_t mf = 255 * abs_sum(f), mh = 255 * abs_sum(h);
    const int64_t bound = std::max({abs_sum(gx_v) * mf, abs_sum(gy_v) * mh,
                                    abs_sum(gdm_f) * mf + abs_sum(gdm_d) * 510});
    t->wide_vagg = bound > INT32_MAX ? 1 : 0;
    return SOBEL5_OK;
}

sobel5_status sobel5_plan_counters(int height, const int* strip_out_w, int n_strips,
                                   const sobel5_taps* t, int prefetch, sobel5_counters* out) {
    if (!t || !out || (n_strips > 0 && !strip_out_w) || height < 5) return SOBEL5_INVALID_ARG;
    auto nz = [](const int32_t* v) {
        uint64_t c = 0;
        for (int i = 0; i < 5; ++i) c += v[i] != 0;
        return c;
    };
    // Closed form of run_strip's tallies (pipeline.hpp:330-343, 347-352,
    // 357-411) for one strip over H rows:
    //   hpass rows: 5 primed + one per later centre  -> H   (both modes)
    //   k0: 2 primed + (H-5) new rows + (H-5) recomputed -> 2H-8
    //   k1: 3 primed + (H-5) switches                 -> H-2
    const uint64_t H = static_cast<uint64_t>(height);
    const uint64_t rows = H, k0 = 2 * H - 8, k1 = H - 2, centres = H - 4;
    (void)prefetch;  // the prefetch schedule reorders but does not change counts
    uint64_t width_sum = 0;
    for (int i = 0; i < n_strips; ++i) {
        if (strip_out_w[i] <= 0) return SOBEL5_INVALID_ARG;
        width_sum += static_cast<uint64_t>(strip_out_w[i]);
    }
    const uint64_t S = static_cast<uint64_t>(n_strips);
    out->row_conv5_f = rows * S;
    out->row_conv5_h = rows * S;
    out->row_diff = rows * S;
    out->row_conv5_k0 = k0 * S;
    out->row_conv5_k1 = k1 * S;
    out->row_conv3_f = 0;
    out->row_conv3_h = 0;
    const uint64_t per_w = (nz(t->f) + nz(t->h) + 2) * rows + nz(t->k0) * k0 + nz(t->k1) * k1 +
                           (nz(t->gx_v) + nz(t->gy_v) + 4 + nz(t->gdm_f) + nz(t->gdm_d)) * centres;
    out->mac = per_w * width_sum;
    return SOBEL5_OK;
}

sobel5_status sobel5_launch(const uint8_t* d_in, int64_t in_pitch, int width, int height,
                            const sobel5_taps* taps, int prefetch, const sobel5_planes* d_out,
                            sobel5_diag* d_diag, void* stream) {
    return launch_common(nullptr, d_in, nullptr, in_pitch, 0, width, height, 1, taps, prefetch,
                         d_out, 0, d_diag, stream, LaunchExtra{});
}

sobel5_status sobel5_launch_batch(const uint8_t* d_in, int64_t in_pitch, int64_t in_frame_stride,
                                  int width, int height, int n_frames, const sobel5_taps* taps,
                                  int prefetch, const sobel5_planes* d_out,
                                  int64_t out_frame_stride, sobel5_diag* d_diag, void* stream) {
    return launch_common(nullptr, d_in, nullptr, in_pitch, in_frame_stride, width, height,
                         n_frames, taps, prefetch, d_out, out_frame_stride, d_diag, stream,
                         LaunchExtra{});
}

sobel5_status sobel5_launch_band(const uint8_t* d_top, const uint8_t* d_in, const uint8_t* d_bot,
                                 int64_t in_pitch, int width, int band_rows,
                                 const sobel5_taps* taps, int prefetch,
                                 const sobel5_planes* d_out, sobel5_diag* d_diag, void* stream) {
    return launch_common(d_top, d_in, d_bot, in_pitch, 0, width, band_rows, 1, taps, prefetch,
                         d_out, 0, d_diag, stream, LaunchExtra{});
}

int sobel5_kernel_for_taps(const sobel5_taps* t) {
    if (!t) return -1;
    if (env_int("SOBEL5_GENERIC", 0) != 0) return 3;
    if (taps_are_default(*t)) return 0;
    if (taps_fit_packed(*t)) return 1;
    if (taps_fit_f32(*t)) return 2;
    return 3;
}

sobel5_status sobel5_selftest(int which, uint32_t lo, uint32_t hi, uint64_t* d_count,
                              void* stream) {
    if (!d_count || hi < lo || which < 0 || which > 5) return SOBEL5_INVALID_ARG;
    if (which == 0 && hi > (1u << 30)) return SOBEL5_INVALID_ARG;
    selftest_kernel<<<148 * 8, 256, 0, static_cast<cudaStream_t>(stream)>>>(
        which, lo, hi, reinterpret_cast<unsigned long long*>(d_count));
    return map_cuda(cudaGetLastError());
}

sobel5_status sobel5_synth_random_device(uint8_t* d_img, int64_t pitch, int width, int height,
                                         int64_t row_offset, uint64_t seed, uint8_t mask,
                                         void* stream) {
    if (!d_img || width < 1 || height < 1 || pitch < width || height > 65535 * 1024)
        return SOBEL5_INVALID_ARG;
    // grid.y is limited to 65535: generate in slabs
    for (int y0 = 0; y0 < height; y0 += 65535) {
        const int hh = std::min(65535, height - y0);
        const dim3 grid(static_cast<unsigned>((width + 255) / 256), static_cast<unsigned>(hh));
        synth_random_kernel<<<grid, 256, 0, static_cast<cudaStream_t>(stream)>>>(
            d_img + static_cast<int64_t>(y0) * pitch, pitch, width, hh, row_offset + y0, seed,
            mask);
        g_launches.fetch_add(1, std::memory_order_relaxed);
        if (cudaError_t e = cudaGetLastError(); e != cudaSuccess) return map_cuda(e);
    }
    return SOBEL5_OK;
}

}  // extern "C"
namespace sobel5_b200 {
sobel5_status launch_band_at(const uint8_t* d_top, const uint8_t* d_in, const uint8_t* d_bot,
                             int64_t in_pitch, int width, int band_rows, const sobel5_taps* taps,
                             int prefetch, const sobel5_planes* d_out, sobel5_diag* d_diag,
                             void* stream, int row0) {
    LaunchExtra ex;
    ex.row0 = row0;
    return launch_common(d_top, d_in, d_bot, in_pitch, 0, width, band_rows, 1, taps, prefetch,
                         d_out, 0, d_diag, stream, ex);
}
}  // namespace sobel5_b200
