// sobel5_f32x2.cuh -- the streaming kernel for ANY taps whose responses stay
// below 2^22 (e.g. FilterParams (2, 3, 5, 7), whose responses overflow the
// int16 lanes of sobel5_packed.cuh), in packed FP32: two pixels per FFMA2.
//
// Integers below 2^24 are exact in FP32 and an FMA rounds once, so every
// product-accumulate of integer taps and integer pixel values is exact as
// long as each partial sum stays below 2^24 -- the host proves that bound
// from the taps (taps_fit_f32 in sobel5_abi.cu) with the absolute-sum argument
// (every partial sum of sum_i c_i x_i is at most 255 * sum_i |c_i|), and
// asks for 2^22 so the final values also convert to int32 by one FADD2 with
// 1.5 * 2^23 (the integer lands in the low mantissa bits).  The taps are
// runtime values (uniform-register operands of FFMA2), the arithmetic is the
// reference's schedule (pipeline.hpp:117-189): row_conv5 F, H, K0, K1 and
// row_diff D per input row, then vagg5 / vagg_gd_minus / vagg_gd_plus as
// running sums, recover_diag with its parity check (:268-282), and the
// magnitude either from the exact integer sum of squares (MagMode kMagU32)
// or in the reference's double order (kMagF64).
//
// Geometry, prefetch ring and column sharing are those of the packed kernel:
// a lane owns 4 output columns x0..x0+3 as pixel pairs (x0+q, x0+q+2), q =
// 0, 1, with window values E_k = {p_k, p_{k+2}}.
#pragma once

#include <cstdint>

#include "sobel5_packed.cuh"

namespace sobel5_b200 {

// float2 {p_j, p_{j+2}} of window bytes j, j+2 (wa = bytes 0..3, wb = 4..7),
// exact: the byte is spliced under the exponent of 2^23 and 2^23 removed.
__device__ __forceinline__ float2 window_pair(uint32_t lo_word, uint32_t hi_word, uint32_t sel_lo,
                                              uint32_t sel_hi) {
    const float a = __uint_as_float(__byte_perm(lo_word, 0x4B000000u, sel_lo));
    const float b = __uint_as_float(__byte_perm(hi_word, 0x4B000000u, sel_hi));
    return __fadd2_rn(make_float2(a, b), make_float2(-8388608.0f, -8388608.0f));
}

// Exact int32 of an integer-valued float with |v| < 2^22: adding 1.5 * 2^23
// puts v in the low mantissa bits (round-to-nearest is exact here).
__device__ __forceinline__ void f2_to_int(float2 v, int32_t& a, int32_t& b) {
    const float2 m = __fadd2_rn(v, make_float2(12582912.0f, 12582912.0f));
    a = static_cast<int32_t>(__float_as_uint(m.x) - 0x4B400000u);
    b = static_cast<int32_t>(__float_as_uint(m.y) - 0x4B400000u);
}

__device__ __forceinline__ float2 f2(float t) { return make_float2(t, t); }

#ifndef SOBEL5_F32_MIN_CTAS
#define SOBEL5_F32_MIN_CTAS 3  // 12 warps/SM: the float2 accumulators need ~160 registers
#endif
// OUTS: kOutSR (the drop-in StreamResult, compile-time) or kOutRuntime (any
// plane set from the pointers, detect-path flags).  MAG: kMagU32 when the
// exact integer sum of squares fits 32 bits, else kMagU64 -- with every
// value below 2^22, S < 2^46 is exact in uint64 and in double, so
// sqrt((double)S) equals the reference's double ((x*x + y*y) + d*d) + t*t.
template <int PF, int GEOM, int MAG, int OUTS>
__global__ void __launch_bounds__(kCtaThreads, SOBEL5_F32_MIN_CTAS)
    sobel5_f32x2_kernel(const __grid_constant__ KernelParams p) {
    pdl_enter();
    __shared__ OddSlot s_odd[kCtaThreads];  // ParityViolation
    if (p.diag) odd_init(s_odd);
    constexpr bool SEG = GEOM == kGeomSeg;
    constexpr bool PAD = GEOM == kGeomPad;
    // TMAL: the CTA's band rows bulk-copied into shared memory at CTA start
    // (tma_band_issue, as kernel A's kGeomPlainTma), read when consumed
    // (instantiated with PF = 0): no global-load latency in the row loop
    constexpr bool TMAL = GEOM == kGeomPlainTma;
    __shared__ __align__(128) uint8_t s_band[TMAL ? TmaBand<false>::kBytes : 16];
    __shared__ __align__(8) uint64_t s_bar[2];
    if constexpr (TMAL) tma_band_issue<false>(p, s_band, s_bar);
    constexpr bool RT = OUTS == kOutRuntime;
    const bool w_gx = RT ? p.gx != nullptr : (OUTS & kOutGx) != 0;
    const bool w_gy = RT ? p.gy != nullptr : (OUTS & kOutGy) != 0;
    const bool w_gd = RT ? p.gd != nullptr : (OUTS & kOutGd) != 0;
    const bool w_gdt = RT ? p.gdt != nullptr : (OUTS & kOutGdt) != 0;
    const bool w_g = RT ? p.g != nullptr : (OUTS & kOutG) != 0;
    const bool w_g32 = RT && p.g32 != nullptr;
    const bool w_u8 = RT && p.u8 != nullptr;
    const bool w_mm = RT && p.minmax != nullptr;
    const bool need_mag = RT ? p.need_mag != 0 : (OUTS & kOutG) != 0;
    const int lane = threadIdx.x & 31;
    const int warp = threadIdx.x >> 5;
    const int warp_x0 = (blockIdx.x * kCtaWarps + warp) * kWarpCols;
    const int x0 = warp_x0 + lane * 4;
    double n_lo = 0.0, n_span = 0.0;
    if (RT && p.u8_norm) {
        n_lo = p.norm[blockIdx.z].lo;
        n_span = p.norm[blockIdx.z].span;
    }
    if (warp_x0 >= p.out_w) return;
    const int oy0 = blockIdx.y * p.band;
    const int n_out = min(p.band, p.out_h - oy0);
    const int n_in = n_out + 4;
    const int64_t in_frame = static_cast<int64_t>(blockIdx.z) * p.in_frame_stride;
    const int64_t out_frame = static_cast<int64_t>(blockIdx.z) * p.out_frame_stride;
    const bool load_a = x0 < p.width;
    const int xoff = (PAD && lane == 0) ? -4 : 4;
    const bool load_b = (lane == 31 && x0 + 4 < p.width) || (PAD && lane == 0 && x0 > 0);
    const bool full = x0 + 3 < p.out_w;
    const PadEdge pe = PAD ? pad_edge_setup(p.width, warp_x0) : PadEdge{0, 0, 0, 0u};
    unsigned long long g_min = ~0ull, g_max = 0ull;  // order keys of g (normalize pass 1)

    const uint8_t* plain = p.mid + in_frame + static_cast<int64_t>(oy0) * p.in_pitch + x0;
    auto load_row = [&](int r, uint32_t& a, uint32_t& b) {
        if constexpr (TMAL) {
            const uint8_t* sr = tma_band_row<false>(s_band, s_bar, r, x0);
            a = load_a ? *reinterpret_cast<const uint32_t*>(sr) : 0u;
            b = load_b ? *reinterpret_cast<const uint32_t*>(sr + xoff) : 0u;
            return;
        }
        const uint8_t* rp;
        if (SEG) {
            rp = stacked_row(p, in_frame, oy0 + r) + x0;
        } else if (PAD) {
            const int y = min(max(oy0 + r - 2, 0), p.mid_rows - 1);
            rp = p.mid + in_frame + static_cast<int64_t>(y) * p.in_pitch + x0;
        } else {
            rp = plain;
            plain += p.in_pitch;
        }
        a = load_a ? ld_row_word(rp) : 0u;
        b = load_b ? ld_row_word(rp + xoff) : 0u;
    };
    int64_t out_off = out_frame + static_cast<int64_t>(oy0) * p.pitch + x0;

    // pending accumulators [slot = output row mod 5][pair]: gx, gy, M, P.
    // Each row first closes slot (s+1) mod 5 (coefficient i = 4) and runs
    // its epilogue, then adds i = 3..1 and opens slot s (i = 0), so only four
    // slots are ever live.
    float2 ax[5][2], ay[5][2], am[5][2], ap[5][2];
    uint32_t qa[5], qb[5];
    uint32_t cur_a = 0u, cur_b = 0u;
    if (PF > 0) {
#pragma unroll
        for (int k = 0; k < 5; ++k) {
            if (k < n_in) load_row(k, qa[k], qb[k]);
            else qa[k] = qb[k] = 0u;
        }
        row_window<PAD>(qa[0], qb[0], lane, x0, p.width, pe, cur_a, cur_b);
    }

    for (int base = 0; base < n_in; base += 5) {
#pragma unroll
        for (int s = 0; s < 5; ++s) {
            const int r = base + s;
            if (r >= n_in) break;
            uint32_t wa, wb;
            if (PF > 0) {
                wa = cur_a;
                wb = cur_b;
                if (r + 5 < n_in) load_row(r + 5, qa[s], qb[s]);
                const int sn = (s + 1) % 5;
                row_window<PAD>(qa[sn], qb[sn], lane, x0, p.width, pe, cur_a, cur_b);
            } else {
                uint32_t o, x;
                load_row(r, o, x);
                row_window<PAD>(o, x, lane, x0, p.width, pe, wa, wb);
            }
            // E_k = {p_k, p_{k+2}}, k = 0..5 (selector: byte, 0x00, 0x00, 0x4B)
            float2 e[6];
            e[0] = window_pair(wa, wa, 0x7540u, 0x7542u);
            e[1] = window_pair(wa, wa, 0x7541u, 0x7543u);
            e[2] = window_pair(wa, wb, 0x7542u, 0x7540u);
            e[3] = window_pair(wa, wb, 0x7543u, 0x7541u);
            e[4] = window_pair(wb, wb, 0x7540u, 0x7542u);
            e[5] = window_pair(wb, wb, 0x7541u, 0x7543u);

            // row_conv5 / row_diff (pipeline.hpp:117-127) for both pairs
            float2 F[2], H[2], D[2], K0[2], K1[2];
#pragma unroll
            for (int q = 0; q < 2; ++q) {
                float2 f = __fmul2_rn(f2(p.tf[0][0]), e[q]);
                float2 hh = __fmul2_rn(f2(p.tf[1][0]), e[q]);
                float2 k0 = __fmul2_rn(f2(p.tf[2][0]), e[q]);
                float2 k1 = __fmul2_rn(f2(p.tf[3][0]), e[q]);
#pragma unroll
                for (int t = 1; t < 5; ++t) {
                    f = __ffma2_rn(f2(p.tf[0][t]), e[q + t], f);
                    hh = __ffma2_rn(f2(p.tf[1][t]), e[q + t], hh);
                    k0 = __ffma2_rn(f2(p.tf[2][t]), e[q + t], k0);
                    k1 = __ffma2_rn(f2(p.tf[3][t]), e[q + t], k1);
                }
                F[q] = f;
                H[q] = hh;
                K0[q] = k0;
                K1[q] = k1;
                D[q] = __ffma2_rn(f2(-1.0f), e[q + 1], e[q + 3]);  // p3 - p1
            }

            // i = 4 closes output row r - 4 (vagg5 / vagg_gd_minus /
            // vagg_gd_plus, pipeline.hpp:136-189, as running sums)
            if (r >= 4) {
                const int sl = (s + 1) % 5;
                int32_t gx[4], gy[4], gd[4], gdt[4];
                bool odd_any = false;
                int32_t odd_p = 0, odd_m = 0, odd_x = 0;
#pragma unroll
                for (int q = 0; q < 2; ++q) {  // pair q holds pixels (q, q + 2)
                    const float2 vx = __ffma2_rn(f2(p.tf[4][4]), F[q], ax[sl][q]);
                    const float2 vy = __ffma2_rn(f2(p.tf[5][4]), H[q], ay[sl][q]);
                    const float2 vm = __ffma2_rn(f2(p.tf[6][4]), F[q],
                                                 __ffma2_rn(f2(p.tf[7][4]), D[q], am[sl][q]));
                    const float2 vp = __ffma2_rn(f2(-1.0f), K0[q], ap[sl][q]);
                    f2_to_int(vx, gx[q], gx[q + 2]);
                    f2_to_int(vy, gy[q], gy[q + 2]);
                    // recover_diag (pipeline.hpp:268-282): gd = (P+M)/2,
                    // gdt = (P-M)/2, ParityViolation when P+M is odd; P +- M
                    // are exact in FP32 (host bound: |P| + |M| < 2^22).
                    // (Extracting P and M as ints first and subtracting
                    // there gave unshifted gdt on the low lanes with nvcc
                    // 12.9 -O3; root cause not isolated.)
                    int32_t s0, s1, d0, d1;
                    f2_to_int(__fadd2_rn(vp, vm), s0, s1);
                    f2_to_int(__ffma2_rn(f2(-1.0f), vm, vp), d0, d1);
                    gd[q] = s0 >> 1;
                    gd[q + 2] = s1 >> 1;
                    gdt[q] = d0 >> 1;
                    gdt[q + 2] = d1 >> 1;
                    const bool odd0 = (s0 & 1) != 0 && x0 + q < p.out_w;
                    const bool odd1 = (s1 & 1) != 0 && x0 + q + 2 < p.out_w;
                    // report (P, M) = ((s+d)/2, (s-d)/2) of the leftmost odd
                    // pixel of the lane (pair q holds columns q and q + 2)
                    if (odd0 || odd1) {
                        const int xq = x0 + q + (odd0 ? 0 : 2);
                        if (!odd_any || xq < odd_x) {
                            const int32_t ss = odd0 ? s0 : s1, dd = odd0 ? d0 : d1;
                            odd_p = (ss + dd) / 2;
                            odd_m = (ss - dd) / 2;
                            odd_x = xq;
                        }
                    }
                    odd_any |= odd0 || odd1;
                }
                const unsigned odd_mask = __ballot_sync(0xffffffffu, odd_any);
                if (odd_mask && p.diag) {
                    if (lane == __ffs(odd_mask) - 1) atomicAdd(&p.diag->violations, 1);
                    if (odd_any)
                        odd_note(s_odd, p.diag, blockIdx.z + p.diag_frame0, p.diag_row0 + oy0 + r - 4,
                                 odd_x, odd_p, odd_m);
                }
                const int64_t row_off = out_off;
                out_off += p.pitch;
                if (full) {
                    if (w_gx) st_cs_v4(p.gx + row_off, gx[0], gx[1], gx[2], gx[3]);
                    if (w_gy) st_cs_v4(p.gy + row_off, gy[0], gy[1], gy[2], gy[3]);
                    if (w_gd) st_cs_v4(p.gd + row_off, gd[0], gd[1], gd[2], gd[3]);
                    if (w_gdt) st_cs_v4(p.gdt + row_off, gdt[0], gdt[1], gdt[2], gdt[3]);
                } else {
#pragma unroll
                    for (int j = 0; j < 4; ++j) {
                        if (x0 + j < p.out_w) {
                            if (w_gx) p.gx[row_off + j] = gx[j];
                            if (w_gy) p.gy[row_off + j] = gy[j];
                            if (w_gd) p.gd[row_off + j] = gd[j];
                            if (w_gdt) p.gdt[row_off + j] = gdt[j];
                        }
                    }
                }
                if (need_mag) {
                    double g[4];
#pragma unroll
                    for (int j = 0; j < 4; ++j) {
                        if (MAG == kMagU32) {  // exact integer S (host-proven < 2^32)
                            const uint32_t ux = static_cast<uint32_t>(gx[j]);
                            const uint32_t uy = static_cast<uint32_t>(gy[j]);
                            const uint32_t ud = static_cast<uint32_t>(gd[j]);
                            const uint32_t ut = static_cast<uint32_t>(gdt[j]);
                            g[j] = __dsqrt_rn(__uint2double_rn(ux * ux + uy * uy + ud * ud + ut * ut));
                        } else {  // exact integer S < 2^46
                            const int64_t S = static_cast<int64_t>(gx[j]) * gx[j] +
                                              static_cast<int64_t>(gy[j]) * gy[j] +
                                              static_cast<int64_t>(gd[j]) * gd[j] +
                                              static_cast<int64_t>(gdt[j]) * gdt[j];
                            g[j] = __dsqrt_rn(__ll2double_rn(S));
                        }
                        if (w_mm && x0 + j < p.out_w) {
                            const unsigned long long b = dkey(g[j]);
                            g_min = min(g_min, b);
                            g_max = max(g_max, b);
                        }
                    }
                    uint32_t u[4] = {0u, 0u, 0u, 0u};
                    if (w_u8) {
#pragma unroll
                        for (int j = 0; j < 4; ++j)
                            u[j] = p.u8_norm ? normalize_u8(g[j], n_lo, n_span) : clamp_abs_u8(g[j]);
                    }
                    if (full) {
                        if (w_g) st_cs_v4d(p.g + row_off, g[0], g[1], g[2], g[3]);
                        if (w_g32)
                            st_cs_v4f(p.g32 + row_off, __double2float_rn(g[0]),
                                      __double2float_rn(g[1]), __double2float_rn(g[2]),
                                      __double2float_rn(g[3]));
                        if (w_u8) st_cs_u32(p.u8 + row_off, pack_u8x4(u[0], u[1], u[2], u[3]));
                    } else {
#pragma unroll
                        for (int j = 0; j < 4; ++j) {
                            if (x0 + j < p.out_w) {
                                if (w_g) p.g[row_off + j] = g[j];
                                if (w_g32) p.g32[row_off + j] = __double2float_rn(g[j]);
                                if (w_u8) p.u8[row_off + j] = static_cast<uint8_t>(u[j]);
                            }
                        }
                    }
                }
            }

            // i = 3..1, then i = 0 opens output row r
#pragma unroll
            for (int q = 0; q < 2; ++q) {
#pragma unroll
                for (int i = 3; i >= 0; --i) {
                    const int sl = (s - i + 5) % 5;
                    if (i == 0) {
                        ax[sl][q] = __fmul2_rn(f2(p.tf[4][0]), F[q]);
                        ay[sl][q] = __fmul2_rn(f2(p.tf[5][0]), H[q]);
                        am[sl][q] = __ffma2_rn(f2(p.tf[6][0]), F[q], __fmul2_rn(f2(p.tf[7][0]), D[q]));
                        ap[sl][q] = K0[q];
                    } else {
                        ax[sl][q] = __ffma2_rn(f2(p.tf[4][i]), F[q], ax[sl][q]);
                        ay[sl][q] = __ffma2_rn(f2(p.tf[5][i]), H[q], ay[sl][q]);
                        am[sl][q] = __ffma2_rn(f2(p.tf[6][i]), F[q],
                                               __ffma2_rn(f2(p.tf[7][i]), D[q], am[sl][q]));
                        if (i == 1) ap[sl][q] = __fadd2_rn(ap[sl][q], K1[q]);
                        if (i == 3) ap[sl][q] = __ffma2_rn(f2(-1.0f), K1[q], ap[sl][q]);
                    }
                }
            }
        }
    }
    if (w_mm) {  // normalize pass 1: frame min / max of g
        for (int o = 16; o > 0; o >>= 1) {
            g_min = min(g_min, __shfl_xor_sync(0xffffffffu, g_min, o));
            g_max = max(g_max, __shfl_xor_sync(0xffffffffu, g_max, o));
        }
        if (lane == 0 && g_min <= g_max) {
            sobel5_minmax* mm = p.minmax + blockIdx.z;
            atomicMin(reinterpret_cast<unsigned long long*>(&mm->lo_key), g_min);
            atomicMax(reinterpret_cast<unsigned long long*>(&mm->hi_key), g_max);
        }
    }
    if (p.diag) odd_flush(s_odd, p.diag);
}

}  // namespace sobel5_b200
