// sobel3_u8.cuh -- the clamped uint8 edge map of the classic 3x3 operator
// alone: clamp_abs (image_io.hpp:235-240) of g = sqrt(gx^2 + gy^2) of
// run_stream_3x3 (pipeline.hpp:486-573; sobel3_2d, oracle.hpp:58-70), valid
// or replicate-padded (pad_replicate(img, 1), image_io.hpp:279-291).
//
// The issue-bound 3x3 contract on the skeleton of the 5x5 u8 kernel
// (sobel5_u8.cuh): band rows by TMA into shared memory, NP packed pixel
// pairs (c, c+2) per lane with the window E_k = byte k | byte k+2 << 16,
// W-warp CTAs.  Per pair and input row: F = p2 - p0 and H = p0 + 2 p1 + p2
// (3 ops); per output row gx = F0 + 2 F1 + F2 and gy = H2 - H0 from a
// 3-slot ring (3 ops); the biases that make a packed register two floats
// are folded into those ops (F carries 0x2000 per half, so gx carries
// 0x8000; gy gets 0x8000 in its subtraction).  S = gx^2 + gy^2 <= 2 * 1020^2
// is exact in float; then the clamp at 65280, MUFU.SQRT and the magic round
// of sobel5_u8.cuh (u8_round_sqrt2, checked for every S on the device).
#pragma once

#include <cstdint>

#include "sobel5_u8.cuh"

namespace sobel5_b200 {

template <int NP, int W>
struct U3Bounds {  // resident CTAs per SM the register budget is set for
    static constexpr int kMinBlocks = 24 / W;
};

// Per pair of one input row: F (biased 0x2000 per half) and H.
template <int NP, bool PAD>
__device__ __forceinline__ void u3_row(const uint8_t* srow, int x0, int width, uint32_t (&F)[NP],
                                       uint32_t (&H)[NP]) {
    constexpr int NW = NP / 2 + 1;
    uint32_t w[NW];
    u8_window<NP, PAD, 1>(srow, x0, width, w);
    // E_k = byte k | byte k+2 << 16, k = 0 .. 2NP - 1 (pair c uses E_c..E_c+2)
    uint32_t e[2 * NP + 2];
#pragma unroll
    for (int k = 0; k < NW; ++k) {
        e[4 * k] = __byte_perm(w[k], 0u, 0x4240);
        e[4 * k + 1] = __byte_perm(w[k], 0u, 0x4341);
        if (k + 1 < NW) {
            const uint32_t m = __byte_perm(w[k], w[k + 1], 0x5432);  // bytes 4k+2 .. 4k+5
            e[4 * k + 2] = __byte_perm(m, 0u, 0x4240);
            e[4 * k + 3] = __byte_perm(m, 0u, 0x4341);
        }
    }
#pragma unroll
    for (int q = 0; q < NP; ++q) {
        const int c = q < 2 ? q : q + 2;
        const uint32_t p0 = e[c], p1 = e[c + 1], p2 = e[c + 2];
        F[q] = p2 - p0 + 0x20002000u;  // f = (-1, 0, 1), biased (pipeline.hpp:500-504)
        H[q] = p0 + p2 + 2u * p1;      // h = (1, 2, 1) (:505-509)
    }
}

// Input row r >= 2 in ring slot S (static): output row r - 2 as 2NP u8 pixels.
template <int S, int NP>
__device__ __forceinline__ void u3_step(const uint32_t (&f)[NP], const uint32_t (&h)[NP],
                                        uint32_t (&F)[3][NP], uint32_t (&H)[3][NP],
                                        uint32_t (&u)[2 * NP]) {
    constexpr int s0 = (S + 1) % 3, s1 = (S + 2) % 3;  // rows r - 2, r - 1
#pragma unroll
    for (int j = 0; j < NP; ++j) {
        F[S][j] = f[j];
        H[S][j] = h[j];
        // gx = F(v-1) + 2 F(v) + F(v+1), gy = H(v+1) - H(v-1) (:536-537)
        const uint32_t gx = F[s0][j] + F[S][j] + 2u * F[s1][j];        // bias 0x8000 per half
        const uint32_t gy = H[S][j] - H[s0][j] + 0x80008000u;          // bias 0x8000 per half
        const float2 fx = u8_pair_float<0x8000u>(gx);
        const float2 fy = u8_pair_float<0x8000u>(gy);
        const float2 sq = __ffma2_rn(fy, fy, __fmul2_rn(fx, fx));  // exact: < 2^22
        const int c = j < 2 ? j : j + 2;
        u8_round_sqrt2(sq, u[c], u[c + 2]);
    }
}

template <int NP, bool PAD, int W>
__device__ __forceinline__ void u3_band_compute(const KernelParams& p, const uint8_t* s_band,
                                                uint64_t* s_bar, int tx, int oy0, int frame,
                                                int n_out) {
    using T = U8Band<NP, PAD, W, 1>;
    constexpr int kLaneCols = U8Geom<NP, W>::kLaneCols;
    const int n_in = n_out + 2;
    const int x0 = tx * U8Geom<NP, W>::kCtaCols + threadIdx.x * kLaneCols;
    if ((x0 & ~(kLaneCols * 32 - 1)) >= p.out_w) return;  // whole warp right of the image
    const bool full = x0 + kLaneCols <= p.out_w;
    const uint8_t* srow = s_band + T::kLead + threadIdx.x * kLaneCols;
    uint8_t* out = p.u8 + static_cast<int64_t>(frame) * p.out_frame_stride +
                   static_cast<int64_t>(oy0) * p.pitch + x0;

    uint32_t F[3][NP], H[3][NP];
    mbar_wait(&s_bar[0], 0);  // rows 0..2
    u3_row<NP, PAD>(srow, x0, p.width, F[0], H[0]);
    u3_row<NP, PAD>(srow + T::kRowBytes, x0, p.width, F[1], H[1]);
    // rows 2..n_in-1, each closing output row r - 2; slot of row r = r mod 3
    for (int base = 2; base < n_in; base += 3) {
#pragma unroll
        for (int k = 0; k < 3; ++k) {
            const int r = base + k;
            if (r >= n_in) break;
            if (r == 3) mbar_wait(&s_bar[1], 0);
            uint32_t f[NP], h[NP];
            u3_row<NP, PAD>(srow + r * T::kRowBytes, x0, p.width, f, h);
            uint32_t u[2 * NP];
            switch (k) {
                case 0: u3_step<2>(f, h, F, H, u); break;
                case 1: u3_step<0>(f, h, F, H, u); break;
                default: u3_step<1>(f, h, F, H, u); break;
            }
            u8_store<NP>(out, u, full, x0, p.out_w);
            out += p.pitch;
        }
    }
}

// grid = (column tiles of W * 32 * 2NP, bands, frames).
template <int NP, bool PAD, int W>
__global__ void __launch_bounds__(U8Geom<NP, W>::kThreads, U3Bounds<NP, W>::kMinBlocks)
    sobel3_u8_kernel(const __grid_constant__ KernelParams p) {
    pdl_enter();
    __shared__ __align__(128) uint8_t s_band[U8Band<NP, PAD, W, 1>::kBytes];
    __shared__ __align__(8) uint64_t s_bar[2];
    const int oy0 = blockIdx.y * p.band;
    const int n_out = min(p.band, p.out_h - oy0);
    u8_band_issue<NP, PAD, W, 1>(p, s_band, s_bar, n_out + 2);
    u3_band_compute<NP, PAD, W>(p, s_band, s_bar, blockIdx.x, oy0, blockIdx.z, n_out);
}

}  // namespace sobel5_b200
