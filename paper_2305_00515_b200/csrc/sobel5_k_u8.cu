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
// pairs per lane: 4 (8 columns, 128 registers, 4 CTAs/SM) by default; 2
// (4 columns, 79 registers, 6 CTAs/SM) issues 18% more instructions at a
// higher issue rate and ties at 8K (44.7 vs 44.9 us), loses at 4K (14.6 vs
// 13.8 us): SOBEL5_U8_NP=2 selects it
int u8_np() { return env_or("SOBEL5_U8_NP", 4) == 2 ? 2 : 4; }

template <int NP>
cudaError_t go(const KernelParams& kp, int frames, cudaStream_t s) {
    const dim3 grid(static_cast<unsigned>((kp.out_w + U8Geom<NP>::kCtaCols - 1) / U8Geom<NP>::kCtaCols),
                    static_cast<unsigned>((kp.out_h + kp.band - 1) / kp.band),
                    static_cast<unsigned>(frames));
    if (kp.pad)
        return launch_kp(sobel5_u8_kernel<NP, true>, grid, kU8Threads, 0, s, kp);
    return launch_kp(sobel5_u8_kernel<NP, false>, grid, kU8Threads, 0, s, kp);
}
}  // namespace

int u8_fast_band(int out_w, int out_h, int frames) {
    const int forced = env_or("SOBEL5_BAND", 0);
    if (forced > 0) return std::min(forced, kU8MaxBand);
    // bands of 16 (20 input rows) unless that leaves fewer than ~6 CTAs per
    // SM (8K: 16 / 32 / 8 rows = 45.0 / 47.5 / 47.7 us; 1080p: 8 rows 5.3 us
    // vs 6.7 at 16; profiles/r2/u8_kernel.txt)
    const int cta_cols = u8_np() == 4 ? U8Geom<4>::kCtaCols : U8Geom<2>::kCtaCols;
    const int64_t cols = (out_w + cta_cols - 1) / cta_cols;
    int band = env_or("SOBEL5_U8_BAND", 16);
    while (band > 4 && cols * frames * ((out_h + band - 1) / band) < 148 * 6) band /= 2;
    return band;
}

int u8_fast_cta_cols() { return u8_np() == 4 ? U8Geom<4>::kCtaCols : U8Geom<2>::kCtaCols; }

cudaError_t launch_u8_fast(const KernelParams& kp, int frames, cudaStream_t s) {
    return u8_np() == 4 ? go<4>(kp, frames, s) : go<2>(kp, frames, s);
}

}  // namespace sobel5_b200
