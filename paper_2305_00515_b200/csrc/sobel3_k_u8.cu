// sobel3_k_u8.cu -- instantiations and launcher of the 3x3 u8-only
// clamp_abs kernel (sobel3_u8.cuh): plain images / batches and fused
// replicate padding (radius 1).
#include <algorithm>
#include <cstdint>
#include <cstdlib>

#include "sobel3_u8.cuh"
#include "sobel5_internal.h"

namespace sobel5_b200 {

namespace {
int env_or(const char* name, int dflt) {
    const char* v = std::getenv(name);
    return v && *v ? std::atoi(v) : dflt;
}

template <int W>
cudaError_t go(const KernelParams& kp, int frames, cudaStream_t s) {
    using G = U8Geom<4, W>;
    const dim3 grid(static_cast<unsigned>((kp.out_w + G::kCtaCols - 1) / G::kCtaCols),
                    static_cast<unsigned>((kp.out_h + kp.band - 1) / kp.band),
                    static_cast<unsigned>(frames));
    if (kp.pad) return launch_kp(sobel3_u8_kernel<4, true, W>, grid, G::kThreads, 0, s, kp);
    return launch_kp(sobel3_u8_kernel<4, false, W>, grid, G::kThreads, 0, s, kp);
}
}  // namespace

// Warps per CTA and output rows per CTA (profiles/r2/u3_sweep.txt): 2 warps
// for 24-96 M output pixels (8K 23.4 us vs 24.5 at 4 warps), 4 elsewhere
// (4K 7.8 vs 8.7, 16K 80.2 vs 83.0 us); 16-row bands halved until ~0.9 of a
// wave of resident CTAs is filled (4K: 8 rows, 1080p: 4 rows);
// SOBEL5_U8_WARPS / SOBEL5_BAND force them.
U8Plan u3_fast_plan(int out_w, int out_h, int frames) {
    U8Plan pl;
    pl.np = 4;
    const int64_t px = int64_t{out_w} * out_h * frames;
    const int forced_w = env_or("SOBEL5_U8_WARPS", 0);
    pl.warps = forced_w == 1 || forced_w == 2 || forced_w == 4
                   ? forced_w
                   : (px >= (int64_t{24} << 20) && px < (int64_t{96} << 20) ? 2 : 4);
    pl.cta_cols = 32 * pl.warps * 8;
    const int forced = env_or("SOBEL5_BAND", 0);
    if (forced > 0) {
        pl.band = std::min(forced, kU8MaxBand);
        return pl;
    }
    const int64_t cols = (out_w + pl.cta_cols - 1) / pl.cta_cols;
    const int64_t per_sm = 24 / pl.warps;
    int band = env_or("SOBEL5_U8_BAND", 16);
    while (band > 4 && cols * frames * ((out_h + band - 1) / band) * 10 < 148 * per_sm * 9) band /= 2;
    pl.band = band;
    return pl;
}

cudaError_t launch_u3_fast(const KernelParams& kp, int frames, const U8Plan& pl, cudaStream_t s) {
    switch (pl.warps) {
        case 1: return go<1>(kp, frames, s);
        case 2: return go<2>(kp, frames, s);
        default: return go<4>(kp, frames, s);
    }
}

}  // namespace sobel5_b200
