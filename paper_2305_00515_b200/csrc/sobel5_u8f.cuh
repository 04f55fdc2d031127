// sobel5_u8f.cuh -- the clamped uint8 edge map alone (clamp_abs of the
// magnitude, image_io.hpp:235-240, of run_stream's four gradients,
// pipeline.hpp:304-414), default taps, with the arithmetic in packed FP32.
//
// Same contract, band staging and operator transformation as the packed-
// integer kernel (sobel5_u8.cuh); what changes is where the numbers become
// floats.  The integer kernel packs two pixels per 32-bit register (IADD3 /
// IMAD on 16-bit halves, 3-input adds for free) and converts gx, gy, N and Q
// to floats at the end: 4 conversions of 3 instructions per pixel pair and
// row.  Here the window bytes become floats once (one PRMT each into the
// mantissa of 2^23, one FADD2 per two), and the horizontal and vertical
// passes run on float2 (FADD2 / FFMA2: the same rate as the packed integer
// ops, every value an exact integer below 2^24).  The pair layout is split so
// that no converted byte has to be copied: lane pairs share 16 columns, lane
// 2m + h owns columns 16m + 4h + {0..3} and 16m + 4h + {8..11}; its pair c
// holds pixels (c, c + 8), whose 5-tap windows are the float2 E_k = (byte k,
// byte k + 8) of its 16-byte window, k = c .. c + 4 -- each byte converted
// exactly once.  Ring state doubles (two registers per pair), so the kernel
// runs at 8 warps per SM.
#pragma once

#include <cstdint>

#include "sobel5_u8.cuh"

namespace sobel5_b200 {

__device__ __forceinline__ float2 f2add(float2 a, float2 b) { return __fadd2_rn(a, b); }
__device__ __forceinline__ float2 f2sub(float2 a, float2 b) {
    return __ffma2_rn(b, make_float2(-1.0f, -1.0f), a);
}
__device__ __forceinline__ float2 f2fma(float2 a, float k, float2 c) {
    return __ffma2_rn(a, make_float2(k, k), c);
}

#ifndef SOBEL5_U8F_WARPS_PER_SM
#define SOBEL5_U8F_WARPS_PER_SM 8
#endif

// Per-pair horizontal results of one input row (float2 = pixels c, c + 8).
struct U8fRow {
    float2 F, D, H, K0, K1;
};

// The lane's 16 window bytes of one row (shared memory) as 4 words: columns
// base - 2*PAD .. base + 15 - 2*PAD.
template <bool PAD>
__device__ __forceinline__ void u8f_window(const uint8_t* srow, int base, int width,
                                           uint32_t (&w)[4]) {
    const uint32_t* s = reinterpret_cast<const uint32_t*>(srow);
    if constexpr (!PAD) {
#pragma unroll
        for (int k = 0; k < 4; ++k) w[k] = s[k];
    } else {
        uint32_t r[5];  // words at base - 4 .. base + 15
#pragma unroll
        for (int k = 0; k < 5; ++k) r[k] = s[k - 1];
        if (base == 0) r[0] = __byte_perm(r[1], 0u, 0x0000);  // left of column 0
#pragma unroll
        for (int k = 0; k < 4; ++k) w[k] = __byte_perm(r[k], r[k + 1], 0x5432);
        const int nv = width - (base - 2);  // window bytes inside the image
        if (nv < 16) u8_fix_right<4>(w, nv);
    }
}

template <bool PAD>
__device__ __forceinline__ void u8f_row(const uint8_t* srow, int base, int width, U8fRow (&o)[4]) {
    uint32_t w[4];
    u8f_window<PAD>(srow, base, width, w);
    // E_k = (byte k, byte k + 8) - 2^23 as exact floats, k = 0..7
    float2 e[8];
#pragma unroll
    for (int k = 0; k < 8; ++k) {
        const uint32_t sel = 0x7440u | static_cast<uint32_t>(k & 3);
        const float lo = __uint_as_float(__byte_perm(w[k >> 2], 0x4B000000u, sel));
        const float hi = __uint_as_float(__byte_perm(w[(k >> 2) + 2], 0x4B000000u, sel));
        e[k] = f2add(make_float2(lo, hi), make_float2(-8388608.0f, -8388608.0f));
    }
#pragma unroll
    for (int c = 0; c < 4; ++c) {
        const float2 p0 = e[c], p1 = e[c + 1], p2 = e[c + 2], p3 = e[c + 3], p4 = e[c + 4];
        const float2 d = f2sub(p3, p1);  // row_diff (pipeline.hpp:124-127)
        const float2 s04 = f2add(p0, p4), s13 = f2add(p1, p3);
        o[c].D = d;
        o[c].F = f2fma(d, 2.0f, f2sub(p4, p0));           // f = (-1,-2,0,2,1)
        o[c].H = f2fma(p2, 6.0f, f2fma(s13, 4.0f, s04));  // h = (1,4,6,4,1)
        o[c].K0 = f2fma(f2add(s04, s13), 3.0f, p2);        // -k0/2 = (3,3,1,3,3)
        o[c].K1 = f2fma(p2, 8.0f, f2fma(s13, 6.0f, s04));  // -k1/2 = (1,6,8,6,1)
    }
}

// Rows 0..3 of a band: fill the ring, open Q.
template <int S>
__device__ __forceinline__ void u8f_prime(const U8fRow (&h)[4], float2 (&F)[5][4],
                                          float2 (&D)[5][4], float2 (&H)[5][4],
                                          float2 (&aq)[5][4]) {
#pragma unroll
    for (int j = 0; j < 4; ++j) {
        F[S][j] = h[j].F;
        D[S][j] = h[j].D;
        H[S][j] = h[j].H;
        if (S >= 1) aq[(S + 4) % 5][j] = f2add(aq[(S + 4) % 5][j], h[j].K1);
        if (S >= 3) aq[(S + 2) % 5][j] = f2sub(aq[(S + 2) % 5][j], h[j].K1);
        aq[S][j] = h[j].K0;
    }
}

// One input row i >= 4 (ring slot S = i mod 5, static): the Q accumulators
// and output row i - 4 as 8 u8 pixels (lo[c] = column c, hi[c] = column
// c + 8, byte 0).  Same algebra as u8_step (sobel5_u8.cuh), no biases.
template <int S>
__device__ __forceinline__ void u8f_step(const U8fRow (&h)[4], float2 (&F)[5][4],
                                         float2 (&D)[5][4], float2 (&H)[5][4],
                                         float2 (&aq)[5][4], uint32_t (&lo)[4],
                                         uint32_t (&hi)[4]) {
    constexpr int s = S, s0 = (S + 1) % 5, s1 = (S + 2) % 5, s2 = (S + 3) % 5, s3 = (S + 4) % 5;
#pragma unroll
    for (int j = 0; j < 4; ++j) {
        F[s][j] = h[j].F;
        D[s][j] = h[j].D;
        H[s][j] = h[j].H;
        // Q(v) = K0'(v) + K1'(v+1) - K1'(v+3) - K0'(v+4) (Eq. 14/15)
        const float2 q = f2sub(aq[s0][j], h[j].K0);
        aq[s3][j] = f2add(aq[s3][j], h[j].K1);
        aq[s1][j] = f2sub(aq[s1][j], h[j].K1);
        aq[s][j] = h[j].K0;
        const float2 t = f2add(F[s0][j], F[s][j]), w = f2add(F[s1][j], F[s3][j]);
        const float2 gx = f2fma(F[s2][j], 6.0f, f2fma(w, 4.0f, t));
        const float2 n = f2fma(D[s2][j], 6.0f,
                               f2fma(f2add(D[s0][j], D[s][j]), -5.0f,
                                     f2fma(f2add(t, w), 3.0f, F[s2][j])));
        const float2 gy = f2fma(f2sub(H[s3][j], H[s1][j]), 2.0f, f2sub(H[s][j], H[s0][j]));
        // S = gx^2 + gy^2 + 2 (N^2 + Q^2) (see u8_step: exact while <= 65280)
        const float2 a = __ffma2_rn(gy, gy, __fmul2_rn(gx, gx));
        const float2 b = __ffma2_rn(q, q, __fmul2_rn(n, n));
        u8_round_sqrt2(f2fma(b, 2.0f, a), lo[j], hi[j]);
    }
}

// Bytes 0 of four words -> one word.
__device__ __forceinline__ uint32_t u8f_pack(const uint32_t (&u)[4]) {
    return __byte_perm(__byte_perm(u[0], u[1], 0x0040), __byte_perm(u[2], u[3], 0x0040), 0x5410);
}

// Rows of one band; FULL: all 12 of the lane's columns are inside the image
// (the per-byte guarded stores of the right edge are their own copy of the
// loop, so the common loop carries no per-row branch).
template <bool PAD, int W, bool FULL>
__device__ __forceinline__ void u8f_band_rows(const KernelParams& p, const uint8_t* srow,
                                              uint64_t* s_bar, int base, uint8_t* out, int n_out) {
    using T = U8Band<4, PAD, W>;
    const int n_in = n_out + 4;
    float2 F[5][4], D[5][4], H[5][4], aq[5][4];
    mbar_wait(&s_bar[0], 0);
    {
        U8fRow h[4];
        u8f_row<PAD>(srow, base, p.width, h);
        u8f_prime<0>(h, F, D, H, aq);
        u8f_row<PAD>(srow + T::kRowBytes, base, p.width, h);
        u8f_prime<1>(h, F, D, H, aq);
        u8f_row<PAD>(srow + 2 * T::kRowBytes, base, p.width, h);
        u8f_prime<2>(h, F, D, H, aq);
        u8f_row<PAD>(srow + 3 * T::kRowBytes, base, p.width, h);
        u8f_prime<3>(h, F, D, H, aq);
    }
    for (int b = 4; b < n_in; b += 5) {
#pragma unroll
        for (int k = 0; k < 5; ++k) {
            const int r = b + k;
            if (r >= n_in) break;
            if (r == 5) mbar_wait(&s_bar[1], 0);
            U8fRow h[4];
            u8f_row<PAD>(srow + r * T::kRowBytes, base, p.width, h);
            uint32_t lo[4], hi[4];
            switch (k) {
                case 0: u8f_step<4>(h, F, D, H, aq, lo, hi); break;
                case 1: u8f_step<0>(h, F, D, H, aq, lo, hi); break;
                case 2: u8f_step<1>(h, F, D, H, aq, lo, hi); break;
                case 3: u8f_step<2>(h, F, D, H, aq, lo, hi); break;
                default: u8f_step<3>(h, F, D, H, aq, lo, hi); break;
            }
            if constexpr (FULL) {
                asm volatile("st.global.cs.u32 [%0], %1;" ::"l"(out), "r"(u8f_pack(lo)) : "memory");
                asm volatile("st.global.cs.u32 [%0], %1;" ::"l"(out + 8), "r"(u8f_pack(hi))
                             : "memory");
            } else {
#pragma unroll
                for (int c = 0; c < 4; ++c) {
                    if (base + c < p.out_w) out[c] = static_cast<uint8_t>(lo[c] & 0xffu);
                    if (base + 8 + c < p.out_w) out[8 + c] = static_cast<uint8_t>(hi[c] & 0xffu);
                }
            }
            out += p.pitch;
        }
    }
}

template <bool PAD, int W>
__device__ __forceinline__ void u8f_band_compute(const KernelParams& p, const uint8_t* s_band,
                                                 uint64_t* s_bar, int tx, int oy0, int frame,
                                                 int n_out) {
    const int lane = threadIdx.x;
    const int cta_x0 = tx * U8Geom<4, W>::kCtaCols;
    const int base = cta_x0 + (lane >> 1) * 16 + (lane & 1) * 4;
    if ((base & ~255) >= p.out_w) return;  // whole warp (256 columns) right of the image
    const uint8_t* srow = s_band + U8Band<4, PAD, W>::kLead + (base - cta_x0);
    uint8_t* out = p.u8 + static_cast<int64_t>(frame) * p.out_frame_stride +
                   static_cast<int64_t>(oy0) * p.pitch + base;
    if (base + 12 <= p.out_w)
        u8f_band_rows<PAD, W, true>(p, srow, s_bar, base, out, n_out);
    else
        u8f_band_rows<PAD, W, false>(p, srow, s_bar, base, out, n_out);
}

// grid = (column tiles of W * 256, bands, frames): the geometry of
// sobel5_u8_kernel<4, PAD, W> (8 columns per lane).
template <bool PAD, int W>
__global__ void __launch_bounds__(32 * W, SOBEL5_U8F_WARPS_PER_SM / W)
    sobel5_u8f_kernel(const __grid_constant__ KernelParams p) {
    pdl_enter();
    __shared__ __align__(128) uint8_t s_band[U8Band<4, PAD, W>::kBytes];
    __shared__ __align__(8) uint64_t s_bar[2];
    const int oy0 = blockIdx.y * p.band;
    const int n_out = min(p.band, p.out_h - oy0);
    u8_band_issue<4, PAD, W>(p, s_band, s_bar, n_out + 4);
    u8f_band_compute<PAD, W>(p, s_band, s_bar, blockIdx.x, oy0, blockIdx.z, n_out);
}

}  // namespace sobel5_b200
