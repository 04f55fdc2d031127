// sobel3_packed.cuh -- the classic 3x3 two-direction operator
// (run_stream_3x3, reference pipeline.hpp:486-573; sobel3_2d, oracle.hpp:58-70)
// on the same B200 skeleton as the 5x5 kernel.
//
// Reference per strip and row (run_strip_3x3, pipeline.hpp:488-547):
//   F = row_conv3(-1, 0, 1),  H = row_conv3(1, 2, 1)      (:500-509)
//   gx = F(v-1) + 2 F(v) + F(v+1),  gy = H(v+1) - H(v-1)  (:536-537)
//   g  = sqrt(gx*gx + gy*gy)                              (:538-540)
// Here: one warp owns 128 output columns (4 per lane, one 32-bit load per
// row, right neighbour word by __shfl_down_sync), a CTA 512 columns and a
// band of rows; two pixels per 32-bit register (pairs (j, j+2), exact since
// |gx|, |gy| <= 1020); vertical sums as running accumulators over a 3-row
// window instead of the reference's F/H row rings (depth 3/4, :496-497).
// g is exact: gx^2 + gy^2 < 2^21, so sqrt of the integer sum is the
// reference's double.
#pragma once

#include <cstdint>

#include "sobel5_packed.cuh"

namespace sobel5_b200 {

// PF: 0 = load each row when consumed (Prefetch::off), 1 = 6-row register
// prefetch ring (Prefetch::on).  PAD: pad_replicate(img, 1) fused.
// TMAL: the CTA's band rows bulk-copied into shared memory at the start (as
// kGeomPlainTma of the 5x5 kernel; valid mode, prefetch on, band <= 32).
template <int PF, bool PAD, int OUTS, bool TMAL = false>
__global__ void __launch_bounds__(kCtaThreads, OUTS == kOutU8 ? SOBEL5_U8_MIN_CTAS : kMinCtasPerSm)
    sobel3_packed_kernel(const __grid_constant__ KernelParams p) {
    pdl_enter();
    constexpr int kTmaLead = PAD ? 16 : 0;  // PAD: lane 0's left word precedes the CTA's columns
    constexpr int kTmaRowBytes = kCtaCols + 16 + kTmaLead, kTmaRows = 34;
    __shared__ __align__(128) uint8_t s_band[TMAL ? kTmaRows * kTmaRowBytes : 16];
    __shared__ __align__(8) uint64_t s_bar[2];
    if constexpr (TMAL) {
        if (threadIdx.x == 0) {
            mbar_init(&s_bar[0], 1);
            mbar_init(&s_bar[1], 1);
            asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
        }
        __syncthreads();
        if (threadIdx.x < 32) {  // warp 0: one lane per row issues its bulk copy
            const int b_oy0 = blockIdx.y * p.band;
            const int b_in = min(p.band, p.out_h - b_oy0) + 2;
            const int n0 = min(6, b_in);
            const int cta_x0 = blockIdx.x * kCtaCols;
            const int src_x = max(cta_x0 - kTmaLead, 0);
            const int dst_off = src_x - (cta_x0 - kTmaLead);
            const uint32_t rb = static_cast<uint32_t>(
                min(kTmaRowBytes - dst_off, ((p.width + 15) & ~15) - src_x));
            if (threadIdx.x == 0) {
                mbar_expect_tx(&s_bar[0], rb * n0);
                mbar_expect_tx(&s_bar[1], rb * (b_in - n0));
            }
            __syncwarp();
            for (int r = threadIdx.x; r < b_in; r += 32) {  // bands up to kTmaRows - 2
                // PAD: padded row b_oy0 + r is image row clamp(b_oy0 + r - 1)
                const int y = PAD ? min(max(b_oy0 + r - 1, 0), p.mid_rows - 1) : b_oy0 + r;
                bulk_load(s_band + r * kTmaRowBytes + dst_off,
                          p.mid + static_cast<int64_t>(blockIdx.z) * p.in_frame_stride +
                              static_cast<int64_t>(y) * p.in_pitch + src_x,
                          rb, &s_bar[r < n0 ? 0 : 1]);
            }
        }
    }
    constexpr bool RT = OUTS == kOutRuntime;
    const bool w_gx = RT ? p.gx != nullptr : (OUTS & kOutGx) != 0;
    const bool w_gy = RT ? p.gy != nullptr : (OUTS & kOutGy) != 0;
    // gx, gy as int16 at the int32 pointers (the host path's narrow D2H
    // wire, |gx|, |gy| <= 1020)
    constexpr bool N16 = !RT && (OUTS & kOutN16) != 0;
    const bool w_g = RT ? p.g != nullptr : (OUTS & kOutG) != 0;
    const bool w_g32 = RT ? p.g32 != nullptr : (OUTS & kOutG32) != 0;
    const bool w_u8 = RT ? p.u8 != nullptr : (OUTS & kOutU8) != 0;
    const bool w_mm = RT ? p.minmax != nullptr : (OUTS & kOutMinMax) != 0;
    const bool u8_norm = RT ? p.u8_norm != 0 : (OUTS & kOutNorm) != 0;
    const bool w_s = RT ? p.s32 != nullptr : (OUTS & kOutS32) != 0;
    const bool need_g = w_g || w_g32;
    constexpr bool FU8 = OUTS == kOutU8;  // clamp_abs edge map alone
    const int lane = threadIdx.x & 31;
    const int warp = threadIdx.x >> 5;
    const int warp_x0 = (blockIdx.x * kCtaWarps + warp) * kWarpCols;
    const int x0 = warp_x0 + lane * 4;

    __shared__ uint32_t s_thr[257];
    float n_lo = 0.f, n_scale = 0.f;
    if (RT || (OUTS & kOutNorm)) {
        if (u8_norm) {
            const sobel5_norm_table* t = p.norm + blockIdx.z;
            for (int i = threadIdx.x; i < 257; i += kCtaThreads) s_thr[i] = t->thr[i];
            n_lo = t->lo_f;
            n_scale = t->scale_f;
            __syncthreads();
        }
    }
    if (warp_x0 >= p.out_w) return;
    const int oy0 = blockIdx.y * p.band;
    const int n_out = min(p.band, p.out_h - oy0);
    const int n_in = n_out + 2;
    const int64_t in_frame = static_cast<int64_t>(blockIdx.z) * p.in_frame_stride;
    const int64_t out_frame = static_cast<int64_t>(blockIdx.z) * p.out_frame_stride;
    const bool load_a = x0 < p.width;
    const int xoff = (PAD && lane == 0) ? -4 : 4;
    const bool load_b = (lane == 31 && x0 + 4 < p.width) || (PAD && lane == 0 && x0 > 0);
    const bool full = x0 + 3 < p.out_w;
    const PadEdge pe = PAD ? pad_edge_setup(p.width, warp_x0) : PadEdge{0, 0, 0, 0u};

    // rows load in order: a running pointer (valid mode) or the clamped row
    // of pad_replicate(img, 1) (image_io.hpp:285)
    const uint8_t* plain = p.mid + in_frame + static_cast<int64_t>(oy0) * p.in_pitch + x0;
    auto load_row = [&](int r, uint32_t& a, uint32_t& b) {
        if constexpr (TMAL) {
            if (r == 0) mbar_wait(&s_bar[0], 0);
            if (r == 6) mbar_wait(&s_bar[1], 0);
            const uint8_t* sr =
                s_band + r * kTmaRowBytes + kTmaLead + (x0 - static_cast<int>(blockIdx.x) * kCtaCols);
            a = load_a ? *reinterpret_cast<const uint32_t*>(sr) : 0u;
            b = load_b ? *reinterpret_cast<const uint32_t*>(sr + xoff) : 0u;
            return;
        }
        const uint8_t* rp;
        if (PAD) {
            const int y = min(max(oy0 + r - 1, 0), p.mid_rows - 1);
            rp = p.mid + in_frame + static_cast<int64_t>(y) * p.in_pitch + x0;
        } else {
            rp = plain;
            plain += p.in_pitch;
        }
        a = load_a ? ld_row_word(rp) : 0u;
        b = load_b ? ld_row_word(rp + xoff) : 0u;
    };

    int64_t out_off = out_frame + static_cast<int64_t>(oy0) * p.pitch + x0;
    constexpr int kRing = 6;  // multiple of the 3-row accumulator window
    uint32_t ax[3][2], ay[3][2];
    uint32_t qa[kRing], qb[kRing];
    uint32_t cur_a = 0u, cur_b = 0u;
    uint32_t s_min = 0xffffffffu, s_max = 0u;
    if (PF > 0) {
#pragma unroll
        for (int k = 0; k < kRing; ++k) {
            if (k < n_in) load_row(k, qa[k], qb[k]);
            else qa[k] = qb[k] = 0u;
        }
        row_window<PAD, 1>(qa[0], qb[0], lane, x0, p.width, pe, cur_a, cur_b);
    }

    for (int base = 0; base < n_in; base += kRing) {
#pragma unroll
        for (int s = 0; s < kRing; ++s) {
            const int r = base + s;
            if (r >= n_in) break;
            uint32_t wa, wb;
            if (PF > 0) {
                wa = cur_a;
                wb = cur_b;
                if (r + kRing < n_in) load_row(r + kRing, qa[s], qb[s]);
                const int sn = (s + 1) % kRing;
                row_window<PAD, 1>(qa[sn], qb[sn], lane, x0, p.width, pe, cur_a, cur_b);
            } else {
                uint32_t o, x;
                load_row(r, o, x);
                row_window<PAD, 1>(o, x, lane, x0, p.width, pe, wa, wb);
            }
            // E_k = byte k | byte k+2 << 16 (k = 0..3)
            const uint32_t mid = __byte_perm(wa, wb, 0x5432);
            const uint32_t e0 = __byte_perm(wa, 0u, 0x4240);
            const uint32_t e1 = __byte_perm(wa, 0u, 0x4341);
            const uint32_t e2 = __byte_perm(mid, 0u, 0x4240);
            const uint32_t e3 = __byte_perm(mid, 0u, 0x4341);
            const uint32_t e[4] = {e0, e1, e2, e3};
            const int s0 = s % 3, s1 = (s + 2) % 3, s2 = (s + 1) % 3;
#pragma unroll
            for (int q = 0; q < 2; ++q) {
                const uint32_t f = e[q + 2] - e[q];                  // (-1, 0, 1)
                const uint32_t hh = e[q] + 2u * e[q + 1] + e[q + 2];  // (1, 2, 1)
                ax[s0][q] = f;  // i = 0 opens output row r
                ay[s0][q] = 0u - hh;
                ax[s1][q] += 2u * f;  // i = 1
                ax[s2][q] += f;       // i = 2 closes output row r - 2
                ay[s2][q] += hh;
            }
            if (FU8 && r >= 2) {
                // u8 clamp_abs only: packed-float epilogue (sobel5_packed.cuh);
                // S = gx^2 + gy^2 < 2^21 is exact in FP32
                const int64_t row_off = out_off;
                out_off += p.pitch;
                uint32_t u[4];
#pragma unroll
                for (int q = 0; q < 2; ++q) {  // pair q holds pixels (q, q + 2)
                    const float2 fx = pair_to_float2(ax[s2][q] + kPairBias);
                    const float2 fy = pair_to_float2(ay[s2][q] + kPairBias);
                    u8_from_sf2(__ffma2_rn(fy, fy, __fmul2_rn(fx, fx)), u[q], u[q + 2]);
                }
                if (full) {
                    st_cs_u32(p.u8 + row_off, pack_u8x4(u[0], u[1], u[2], u[3]));
                } else {
#pragma unroll
                    for (int j = 0; j < 4; ++j)
                        if (x0 + j < p.out_w) p.u8[row_off + j] = static_cast<uint8_t>(u[j]);
                }
            } else if (r >= 2) {
                int32_t gx[4], gy[4];
#pragma unroll
                for (int q = 0; q < 2; ++q) {
                    gx[q] = lane_lo(ax[s2][q]);
                    gx[q + 2] = lane_hi(ax[s2][q]);
                    gy[q] = lane_lo(ay[s2][q]);
                    gy[q + 2] = lane_hi(ay[s2][q]);
                }
                const int64_t row_off = out_off;
                out_off += p.pitch;
                uint32_t S[4];
#pragma unroll
                for (int j = 0; j < 4; ++j)
                    S[j] = static_cast<uint32_t>(gx[j] * gx[j]) + static_cast<uint32_t>(gy[j] * gy[j]);
                if (w_mm) {
#pragma unroll
                    for (int j = 0; j < 4; ++j)
                        if (full || x0 + j < p.out_w) {
                            s_min = min(s_min, S[j]);
                            s_max = max(s_max, S[j]);
                        }
                }
                if (w_s) {
                    if (full) {
                        *reinterpret_cast<uint4*>(p.s32 + row_off) = make_uint4(S[0], S[1], S[2], S[3]);
                    } else {
#pragma unroll
                        for (int j = 0; j < 4; ++j)
                            if (x0 + j < p.out_w) p.s32[row_off + j] = S[j];
                    }
                }
                double g[4] = {0.0, 0.0, 0.0, 0.0};
                if (need_g) {
#pragma unroll
                    for (int j = 0; j < 4; ++j) g[j] = sqrt_u30(S[j]);
                }
                uint32_t u[4] = {0u, 0u, 0u, 0u};
                if (w_u8) {
#pragma unroll
                    for (int j = 0; j < 4; ++j)
                        u[j] = u8_norm ? u8_normalize_s(S[j], s_thr, n_lo, n_scale) : u8_from_s(S[j]);
                }
                if constexpr (N16) {
                    auto st16 = [&](int32_t* plane, const int32_t (&v)[4]) {
                        int16_t* q = reinterpret_cast<int16_t*>(plane) + row_off;
                        if (full) {
                            st_wb_v2u(q, __byte_perm(v[0], v[1], 0x5410), __byte_perm(v[2], v[3], 0x5410));
                        } else {
#pragma unroll
                            for (int j = 0; j < 4; ++j)
                                if (x0 + j < p.out_w) q[j] = static_cast<int16_t>(v[j]);
                        }
                    };
                    st16(p.gx, gx);
                    st16(p.gy, gy);
                    if (w_g) {  // (without g: the host rebuilds it from the wire)
                        if (full) {
                            st_cs_v4d(p.g + row_off, g[0], g[1], g[2], g[3]);
                        } else {
#pragma unroll
                            for (int j = 0; j < 4; ++j)
                                if (x0 + j < p.out_w) p.g[row_off + j] = g[j];
                        }
                    }
                } else if (full) {
                    if (w_gx) st_cs_v4(p.gx + row_off, gx[0], gx[1], gx[2], gx[3]);
                    if (w_gy) st_cs_v4(p.gy + row_off, gy[0], gy[1], gy[2], gy[3]);
                    if (w_g) st_cs_v4d(p.g + row_off, g[0], g[1], g[2], g[3]);
                    if (w_g32)
                        st_cs_v4f(p.g32 + row_off, __double2float_rn(g[0]), __double2float_rn(g[1]),
                                  __double2float_rn(g[2]), __double2float_rn(g[3]));
                    if (w_u8)
                        st_cs_u32(p.u8 + row_off, pack_u8x4(u[0], u[1], u[2], u[3]));
                } else {
#pragma unroll
                    for (int j = 0; j < 4; ++j) {
                        if (x0 + j < p.out_w) {
                            if (w_gx) p.gx[row_off + j] = gx[j];
                            if (w_gy) p.gy[row_off + j] = gy[j];
                            if (w_g) p.g[row_off + j] = g[j];
                            if (w_g32) p.g32[row_off + j] = __double2float_rn(g[j]);
                            if (w_u8) p.u8[row_off + j] = static_cast<uint8_t>(u[j]);
                        }
                    }
                }
            }
        }
    }
    if (w_mm) {
        s_min = __reduce_min_sync(0xffffffffu, s_min);
        s_max = __reduce_max_sync(0xffffffffu, s_max);
        if (lane == 0 && s_min <= s_max) {
            sobel5_minmax* mm = p.minmax + blockIdx.z;
            atomicMin(reinterpret_cast<unsigned long long*>(&mm->lo_key), dkey(sqrt_u30(s_min)));
            atomicMax(reinterpret_cast<unsigned long long*>(&mm->hi_key), dkey(sqrt_u30(s_max)));
        }
    }
}

}  // namespace sobel5_b200
