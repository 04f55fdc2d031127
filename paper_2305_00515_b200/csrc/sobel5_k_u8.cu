// sobel5_k_u8.cu -- instantiations and launcher of the u8-only clamp_abs
// kernel (sobel5_u8.cuh): plain images / batches and fused replicate padding.
#include <algorithm>
#include <cstdint>
#include <cstdlib>

#include "sobel5_internal.h"
#include "sobel5_u8.cuh"

namespace sobel5_b200 {

namespace {
int env_or(const char* name, int dflt) {
    const char* v = std::getenv(name);
    return v && *v ? std::atoi(v) : dflt;
}
template <int NP, int W>
cudaError_t go(const KernelParams& kp, int frames, cudaStream_t s) {
    using G = U8Geom<NP, W>;
    const dim3 grid(static_cast<unsigned>((kp.out_w + G::kCtaCols - 1) / G::kCtaCols),
                    static_cast<unsigned>((kp.out_h + kp.band - 1) / kp.band),
                    static_cast<unsigned>(frames));
    if (kp.s32) {  // normalize pass 1: exact S plane + min / max (MODE 1)
        if (kp.pad)
            return launch_kp(sobel5_u8_kernel<NP, true, W, 1>, grid, G::kThreads, 0, s, kp);
        return launch_kp(sobel5_u8_kernel<NP, false, W, 1>, grid, G::kThreads, 0, s, kp);
    }
    if (kp.pad)
        return launch_kp(sobel5_u8_kernel<NP, true, W>, grid, G::kThreads, 0, s, kp);
    return launch_kp(sobel5_u8_kernel<NP, false, W>, grid, G::kThreads, 0, s, kp);
}

template <int NP>
cudaError_t go_w(const KernelParams& kp, int frames, int warps, cudaStream_t s) {
    switch (warps) {
        case 1: return go<NP, 1>(kp, frames, s);
        case 2: return go<NP, 2>(kp, frames, s);
        default: return go<NP, 4>(kp, frames, s);
    }
}
}  // namespace

// Pairs per lane, warps per CTA and output rows per CTA of a launch
// (profiles/r2/u8_warps.txt: W x band sweep at 1080p / 4K / 8K / 16K).
//   NP: 4 (8 columns per lane, 128 registers) by default; 2 (4 columns, 79
//   registers) issues 18% more instructions at a higher issue rate and ties
//   at 8K, loses at 4K: SOBEL5_U8_NP=2 selects it.
//   W: warps per CTA.  2 for 24-96 M output pixels (8K: 42.7 us vs 44.8 at
//   W = 4, 43.7 at W = 1), 4 elsewhere (4K 13.6 vs 14.3, 16K 153.3 vs
//   154.8 us); SOBEL5_U8_WARPS forces 1 / 2 / 4.
//   band: 24 rows from 96 M output pixels (16K: 153.3 vs 156.1 us at 16),
//   else 16, halved while the grid would fill less than ~0.9 of one wave of
//   resident CTAs (1080p: 4 rows, 5.2 us vs 12.3 at 16; 4K: 16 rows, 13.6
//   vs 14.2 at 8).
U8Plan u8_fast_plan(int out_w, int out_h, int frames) {
    U8Plan pl;
    pl.np = env_or("SOBEL5_U8_NP", 4) == 2 ? 2 : 4;
    const int64_t px = int64_t{out_w} * out_h * frames;
    const int forced_w = env_or("SOBEL5_U8_WARPS", 0);
    pl.warps = forced_w == 1 || forced_w == 2 || forced_w == 4
                   ? forced_w
                   : (px >= (int64_t{24} << 20) && px < (int64_t{96} << 20) ? 2 : 4);
    pl.cta_cols = 32 * pl.warps * 2 * pl.np;
    const int forced = env_or("SOBEL5_BAND", 0);
    if (forced > 0) {
        pl.band = std::min(forced, kU8MaxBand);
        return pl;
    }
    const int64_t cols = (out_w + pl.cta_cols - 1) / pl.cta_cols;
    const int64_t per_sm = (pl.np == 4 ? 16 : 24) / pl.warps;  // resident CTAs per SM
    int band = env_or("SOBEL5_U8_BAND", px >= (int64_t{96} << 20) ? 24 : 16);
    while (band > 4 && cols * frames * ((out_h + band - 1) / band) * 10 < 148 * per_sm * 9) band /= 2;
    pl.band = band;
    return pl;
}

cudaError_t launch_u8_fast(const KernelParams& kp, int frames, const U8Plan& pl, cudaStream_t s) {
    return pl.np == 4 ? go_w<4>(kp, frames, pl.warps, s) : go_w<2>(kp, frames, pl.warps, s);
}

}  // namespace sobel5_b200
