// sobel5_k_dense.cu -- ABLATION ONLY (SOBEL5_DENSE=1, default taps, plain
// images, the StreamResult planes or the u8 map alone): the four
// directional responses as four
// dense 5x5 correlations with the materialized kernels (filter_algebra.hpp
// materialize, the oracle's conv2d_valid order, oracle.hpp:19-33), i.e. the
// packed kernel WITHOUT the paper's operator transformation (Eq. 10-21).
// Same geometry, column sharing, prefetch ring, two-pixels-per-register
// packing and epilogue as sobel5_packed.cuh, so the timing difference is the
// transformation alone (profiles/r1/ablation.txt).
#include "sobel5_internal.h"
#include "sobel5_packed.cuh"

namespace sobel5_b200 {

namespace {

// materialize((1, 2, 6, 4), X / Y / D / DT), correlation weights K[i][j]
// applied as out(y, x) = sum K[i][j] * img(y + i, x + j)
__device__ constexpr int32_t kDense[4][5][5] = {
    {{-1, -2, 0, 2, 1}, {-4, -8, 0, 8, 4}, {-6, -12, 0, 12, 6}, {-4, -8, 0, 8, 4}, {-1, -2, 0, 2, 1}},
    {{-1, -4, -6, -4, -1}, {-2, -8, -12, -8, -2}, {0, 0, 0, 0, 0}, {2, 8, 12, 8, 2}, {1, 4, 6, 4, 1}},
    {{-6, -4, -1, -2, 0}, {-4, -12, -8, 0, 2}, {-1, -8, 0, 8, 1}, {-2, 0, 8, 12, 4}, {0, 2, 1, 4, 6}},
    {{0, -2, -1, -4, -6}, {2, 0, -8, -12, -4}, {1, 8, 0, -8, -1}, {4, 12, 8, 0, -2}, {6, 4, 1, 2, 0}},
};

template <bool U8>  // U8: the clamp_abs map alone, with the packed kernel's FP32 epilogue
__global__ void __launch_bounds__(kCtaThreads, kMinCtasPerSm)
    sobel5_dense_kernel(const __grid_constant__ KernelParams p) {
    const int lane = threadIdx.x & 31;
    const int warp = threadIdx.x >> 5;
    const int warp_x0 = (blockIdx.x * kCtaWarps + warp) * kWarpCols;
    const int x0 = warp_x0 + lane * 4;
    if (warp_x0 >= p.out_w) return;
    const int oy0 = blockIdx.y * p.band;
    const int n_out = min(p.band, p.out_h - oy0);
    const int n_in = n_out + 4;
    const bool load_a = x0 < p.width;
    const bool load_b = lane == 31 && x0 + 4 < p.width;
    const bool full = x0 + 3 < p.out_w;
    const PadEdge pe{0, 0, 0, 0u};
    const uint8_t* plain = p.mid + static_cast<int64_t>(oy0) * p.in_pitch + x0;
    auto load_row = [&](uint32_t& a, uint32_t& b) {
        a = load_a ? ld_row_word(plain) : 0u;
        b = load_b ? ld_row_word(plain + 4) : 0u;
        plain += p.in_pitch;
    };
    int64_t out_off = static_cast<int64_t>(oy0) * p.pitch + x0;

    uint32_t qa[5], qb[5], er[5][6];
    uint32_t cur_a = 0u, cur_b = 0u;
#pragma unroll
    for (int k = 0; k < 5; ++k) {
        if (k < n_in) load_row(qa[k], qb[k]);
        else qa[k] = qb[k] = 0u;
    }
    row_window<false>(qa[0], qb[0], lane, x0, p.width, pe, cur_a, cur_b);

    for (int base = 0; base < n_in; base += 5) {
#pragma unroll
        for (int s = 0; s < 5; ++s) {
            const int r = base + s;
            if (r >= n_in) break;
            const uint32_t wa = cur_a, wb = cur_b;
            if (r + 5 < n_in) load_row(qa[s], qb[s]);
            row_window<false>(qa[(s + 1) % 5], qb[(s + 1) % 5], lane, x0, p.width, pe, cur_a, cur_b);
            const uint32_t mid = __byte_perm(wa, wb, 0x5432);
            er[s][0] = __byte_perm(wa, 0u, 0x4240);
            er[s][1] = __byte_perm(wa, 0u, 0x4341);
            er[s][2] = __byte_perm(mid, 0u, 0x4240);
            er[s][3] = __byte_perm(mid, 0u, 0x4341);
            er[s][4] = __byte_perm(wb, 0u, 0x4240);
            er[s][5] = __byte_perm(wb, 0u, 0x4341);
            if (r < 4) continue;
            // output row r - 4 from input rows r-4 .. r (slots s+1 .. s)
            uint32_t acc[4][2];
#pragma unroll
            for (int d = 0; d < 4; ++d)
#pragma unroll
                for (int q = 0; q < 2; ++q) {
                    uint32_t a = 0u;
#pragma unroll
                    for (int i = 0; i < 5; ++i)
#pragma unroll
                        for (int j = 0; j < 5; ++j)
                            if (kDense[d][i][j] != 0)
                                a += static_cast<uint32_t>(kDense[d][i][j]) * er[(s + 1 + i) % 5][q + j];
                    acc[d][q] = a;
                }
            if constexpr (U8) {
                const int64_t row_off = out_off;
                out_off += p.pitch;
                uint32_t u[4];
#pragma unroll
                for (int q = 0; q < 2; ++q)
                    u8_from_sf2(sumsq4(pair_to_float2(acc[0][q] + kPairBias), pair_to_float2(acc[1][q] + kPairBias),
                                       pair_to_float2(acc[2][q] + kPairBias), pair_to_float2(acc[3][q] + kPairBias)),
                                u[q], u[q + 2]);
                if (full) {
                    st_cs_u32(p.u8 + row_off, pack_u8x4(u[0], u[1], u[2], u[3]));
                } else {
#pragma unroll
                    for (int j = 0; j < 4; ++j)
                        if (x0 + j < p.out_w) p.u8[row_off + j] = static_cast<uint8_t>(u[j]);
                }
                continue;
            }
            int32_t g4[4][4];  // [dir][pixel]
#pragma unroll
            for (int d = 0; d < 4; ++d)
#pragma unroll
                for (int q = 0; q < 2; ++q) {
                    g4[d][q] = lane_lo(acc[d][q]);
                    g4[d][q + 2] = lane_hi(acc[d][q]);
                }
            double g[4];
#pragma unroll
            for (int j = 0; j < 4; ++j)
                g[j] = sqrt_u30(static_cast<uint32_t>(g4[0][j] * g4[0][j]) +
                                static_cast<uint32_t>(g4[1][j] * g4[1][j]) +
                                static_cast<uint32_t>(g4[2][j] * g4[2][j]) +
                                static_cast<uint32_t>(g4[3][j] * g4[3][j]));
            const int64_t row_off = out_off;
            out_off += p.pitch;
            if (full) {
                st_cs_v4(p.gx + row_off, g4[0][0], g4[0][1], g4[0][2], g4[0][3]);
                st_cs_v4(p.gy + row_off, g4[1][0], g4[1][1], g4[1][2], g4[1][3]);
                st_cs_v4(p.gd + row_off, g4[2][0], g4[2][1], g4[2][2], g4[2][3]);
                st_cs_v4(p.gdt + row_off, g4[3][0], g4[3][1], g4[3][2], g4[3][3]);
                st_cs_v4d(p.g + row_off, g[0], g[1], g[2], g[3]);
            } else {
#pragma unroll
                for (int j = 0; j < 4; ++j)
                    if (x0 + j < p.out_w) {
                        p.gx[row_off + j] = g4[0][j];
                        p.gy[row_off + j] = g4[1][j];
                        p.gd[row_off + j] = g4[2][j];
                        p.gdt[row_off + j] = g4[3][j];
                        p.g[row_off + j] = g[j];
                    }
            }
        }
    }
}

}  // namespace

cudaError_t launch_dense_ablation(const KernelParams& kp, dim3 grid, cudaStream_t s) {
    if (kp.u8 && !kp.gx)
        sobel5_dense_kernel<true><<<grid, kCtaThreads, 0, s>>>(kp);
    else
        sobel5_dense_kernel<false><<<grid, kCtaThreads, 0, s>>>(kp);
    return cudaGetLastError();
}

}  // namespace sobel5_b200
