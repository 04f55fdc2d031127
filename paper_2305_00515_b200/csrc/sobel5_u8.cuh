// sobel5_u8.cuh -- the clamped uint8 edge map alone (clamp_abs of the
// magnitude, image_io.hpp:235-240, of run_stream's four gradients,
// pipeline.hpp:304-414), default taps: the issue-bound contract.
//
// The StreamResult kernel (sobel5_packed.cuh) writes 24 B/px and is bound by
// HBM; this one moves 2 B/px, so its time is instruction issue.  It is laid
// out for that:
//   * NP packed pixel pairs per lane (NP = 2: 4 columns, NP = 4: 8 columns);
//     pair q holds pixels (x0 + c_q, x0 + c_q + 2), c = 0, 1 (, 4, 5), and
//     its 5-tap window is E_c..E_c+4 with E_k = byte k | byte k+2 << 16 of
//     the lane's window (one byte permute per E_k).
//   * the CTA's band rows arrive by TMA bulk copies (one per row, issued at
//     CTA start, two mbarrier stages) and each lane reads its window words of
//     a row from shared memory -- no shuffle, no lane-31 special case, no
//     register prefetch ring.
//   * horizontal pass per pair and input row (the operator transformation,
//     Eq. 10-21): D = p3-p1, s04, s13, then F, H, K0', K1' -- 11 packed
//     integer ops for two pixels.
//   * vertical pass as a RING of the last five rows' F, D and H (static slots,
//     the 5-row unroll): with T = F0+F4, U = F1+F3 the symmetric taps share
//     work, gx = T + 4U + 6F2 and N = 3(T+U) + F2 - 5(D0+D4) + 6D2 cost 9 ops
//     together, gy = (H4-H0) + 2(H3-H1) 3 ops; the Kd+ response Q keeps
//     running accumulators (3 ops per row, 4 registers instead of 8).
//   * the half-word bias that lets a packed register become two floats is
//     folded into ops that exist anyway (F carries 2^27+2^11 per pixel pair,
//     so gx carries 0x80008000 and N 0x68006800; gy and Q get it in their
//     last three-input add) -- no bias instructions.
//   * magnitude: S = gx^2 + gy^2 + 2(N^2 + Q^2) (gd^2 + gdt^2 = 2N^2 + 2Q^2
//     since gd = N-Q, gdt = -N-Q), packed FP32, then a clamp, MUFU.SQRT and a
//     magic-number round (no F2I).
#pragma once

#include <cstdint>

#include "sobel5_packed.cuh"

namespace sobel5_b200 {

constexpr int kU8MaxBand = 32;  // output rows per CTA (<=)

// W warps per CTA side by side (W = 1, 2, 4: the launcher picks by size).
template <int NP, int W>
struct U8Geom {
    static constexpr int kThreads = 32 * W;
    static constexpr int kLaneCols = 2 * NP;
    static constexpr int kCtaCols = kThreads * kLaneCols;
};

// Shared-memory band: rows of the CTA's columns [x0c - lead, x0c + cols + 16)
// (R = operator radius: 2 for the 5x5 operator, 1 for the 3x3 one).
template <int NP, bool PAD, int W, int R = 2>
struct U8Band {
    static constexpr int kLead = PAD ? 16 : 0;
    static constexpr int kRowBytes = U8Geom<NP, W>::kCtaCols + 16 + kLead;
    static constexpr int kRows = kU8MaxBand + 2 * R;
    static constexpr int kBytes = kRows * kRowBytes;
};

// A packed register holding (lo + B, hi + B) as unsigned halves -> the pair
// {lo, hi} as exact floats (splice under the exponent of 2^23, one FADD2).
template <uint32_t B>
__device__ __forceinline__ float2 u8_pair_float(uint32_t w) {
    const float lo = __uint_as_float(__byte_perm(w, 0x4B000000u, 0x7610));
    const float hi = __uint_as_float(__byte_perm(w, 0x4B000000u, 0x7632));
    constexpr float kOff = 8388608.0f + static_cast<float>(B);
    return __fadd2_rn(make_float2(lo, hi), make_float2(-kOff, -kOff));
}

// sqrt(S) rounded to nearest and saturated to 255 (clamp_abs), returned in
// the LOW BYTE of the result (the other bytes are 0x4B40_00): S is clamped to
// 65280 first (sqrt(65280) = 255.4995 rounds to 255, the saturation of every
// larger S), MUFU.SQRT, then one FADD of 1.5 * 2^23 rounds to the nearest
// integer, which lands in the low mantissa bits -- one XU instruction per
// pixel instead of MUFU + F2I.  S is exact whenever the true sum is <= 65280
// and >= 65281 otherwise (see u8_step); sqrt(S) for integer S is never within
// 4.9e-4 of k + 0.5, far above the approximation's error (checked for every
// S on the device: sobel5_selftest 4 / 5).
__device__ __forceinline__ uint32_t u8_round_sqrt(float S) {
    float y;
    asm("sqrt.approx.ftz.f32 %0, %1;" : "=f"(y) : "f"(fminf(S, 65280.0f)));
    return __float_as_uint(__fadd_rn(y, 12582912.0f));
}
__device__ __forceinline__ void u8_round_sqrt2(float2 S, uint32_t& a, uint32_t& b) {
    float ya, yb;
    asm("sqrt.approx.ftz.f32 %0, %1;" : "=f"(ya) : "f"(fminf(S.x, 65280.0f)));
    asm("sqrt.approx.ftz.f32 %0, %1;" : "=f"(yb) : "f"(fminf(S.y, 65280.0f)));
    const float2 r = __fadd2_rn(make_float2(ya, yb), make_float2(12582912.0f, 12582912.0f));
    a = __float_as_uint(r.x);
    b = __float_as_uint(r.y);
}

// One band's rows by TMA: rows 0..2R complete on bar[0], the rest on bar[1].
template <int NP, bool PAD, int W, int R = 2>
struct U8BandCopy {
    using T = U8Band<NP, PAD, W, R>;
    int src_x, dst_off, n0, b_in;
    uint32_t rb;
    __device__ __forceinline__ U8BandCopy(const KernelParams& p, int tx, int b_in_) {
        const int cta_x0 = tx * U8Geom<NP, W>::kCtaCols;
        src_x = max(cta_x0 - T::kLead, 0);
        dst_off = src_x - (cta_x0 - T::kLead);
        rb = static_cast<uint32_t>(min(T::kRowBytes - dst_off, ((p.width + 15) & ~15) - src_x));
        b_in = b_in_;
        n0 = min(2 * R + 1, b_in);
    }
    // one thread: arm both barriers with the bytes they will receive
    __device__ __forceinline__ void arm(uint64_t* bar) const {
        mbar_expect_tx(&bar[0], rb * n0);
        mbar_expect_tx(&bar[1], rb * (b_in - n0));
    }
    // thread t of nt issues rows t, t + nt, ... (after the barriers are armed)
    __device__ __forceinline__ void copy(const KernelParams& p, uint8_t* s_band, uint64_t* bar,
                                         int oy0, int frame, int t, int nt) const {
        for (int r = t; r < b_in; r += nt) {
            const int y = PAD ? min(max(oy0 + r - R, 0), p.mid_rows - 1) : oy0 + r;
            bulk_load(s_band + r * T::kRowBytes + dst_off,
                      p.mid + static_cast<int64_t>(frame) * p.in_frame_stride +
                          static_cast<int64_t>(y) * p.in_pitch + src_x,
                      rb, &bar[r < n0 ? 0 : 1]);
        }
    }
};

// Block-wide: barrier init, then warp 0 issues one bulk copy per band row.
// Every thread must call it (__syncthreads inside).
template <int NP, bool PAD, int W, int R = 2>
__device__ __forceinline__ void u8_band_issue(const KernelParams& p, uint8_t* s_band,
                                              uint64_t* s_bar, int b_in) {
    if (threadIdx.x == 0) {
        mbar_init(&s_bar[0], 1);
        mbar_init(&s_bar[1], 1);
        asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
    }
    __syncthreads();
    if (threadIdx.x < 32) {
        const U8BandCopy<NP, PAD, W, R> bc(p, blockIdx.x, b_in);
        if (threadIdx.x == 0) bc.arm(s_bar);
        __syncwarp();
        bc.copy(p, s_band, s_bar, blockIdx.y * p.band, blockIdx.z, threadIdx.x, 32);
    }
}

// Per-pair horizontal results of one input row.
struct U8Row {
    uint32_t F, D, H, K0, K1;
};

// Replicate column width-1 over the window bytes at or past index nv
// (pad_replicate, image_io.hpp:286); the window is NW words.
template <int NW>
__device__ __forceinline__ void u8_fix_right(uint32_t (&w)[NW], int nv) {
    const int e = nv - 1;  // window byte of column width-1
    uint32_t src = w[0];
#pragma unroll
    for (int k = 1; k < NW; ++k)
        if (e >= 4 * k) src = w[k];
    const uint32_t rep = __byte_perm(src, 0u, static_cast<uint32_t>(e & 3) * 0x1111u);
#pragma unroll
    for (int k = 0; k < NW; ++k) {
        const int keep = nv - 4 * k;  // bytes of this word still inside
        if (keep < 4) {
            const uint32_t m = keep <= 0 ? 0u : (0xffffffffu >> (8 * (4 - keep)));
            w[k] = (w[k] & m) | (rep & ~m);
        }
    }
}

// The lane's window of one row (shared memory) -> E_k, then the horizontal
// pass of its NP pairs.  Valid mode: window = columns x0 .. x0 + 2NP + 3.
// PAD: it starts 2 columns left of x0, built from the words left and right
// of the lane's own bytes; columns outside the image take the edge pixel.
// The lane's NW window words of one row: columns x0 - R*PAD ... (radius R).
template <int NP, bool PAD, int R = 2>
__device__ __forceinline__ void u8_window(const uint8_t* srow, int x0, int width,
                                          uint32_t (&w)[NP / 2 + 1]) {
    constexpr int NW = NP / 2 + 1;  // window words
    if constexpr (!PAD) {
        if constexpr (NP == 4) {
            const uint2 a = *reinterpret_cast<const uint2*>(srow);
            w[0] = a.x;
            w[1] = a.y;
        } else {
            w[0] = *reinterpret_cast<const uint32_t*>(srow);
        }
        w[NW - 1] = *reinterpret_cast<const uint32_t*>(srow + 4 * (NW - 1));
    } else {
        uint32_t r[NW + 1];  // words at x0 - 4 .. x0 + 4 * NW - 4
        r[0] = *reinterpret_cast<const uint32_t*>(srow - 4);
        if constexpr (NP == 4) {
            const uint2 a = *reinterpret_cast<const uint2*>(srow);
            r[1] = a.x;
            r[2] = a.y;
        } else {
            r[1] = *reinterpret_cast<const uint32_t*>(srow);
        }
        r[NW] = *reinterpret_cast<const uint32_t*>(srow + 4 * (NW - 1));
        if (x0 == 0) r[0] = __byte_perm(r[1], 0u, 0x0000);  // left of column 0
        // window starts R bytes left of x0: bytes 4-R .. 7-R of (r[k], r[k+1])
        constexpr uint32_t kSel = R == 2 ? 0x5432u : 0x6543u;
#pragma unroll
        for (int k = 0; k < NW; ++k) w[k] = __byte_perm(r[k], r[k + 1], kSel);
        const int nv = width - (x0 - R);  // window bytes inside the image
        if (nv < 4 * NW) u8_fix_right<NW>(w, nv);
    }
}

template <int NP, bool PAD>
__device__ __forceinline__ void u8_row(const uint8_t* srow, int x0, int width, U8Row (&o)[NP]) {
    constexpr int NW = NP / 2 + 1;  // window words
    uint32_t w[NW];
    u8_window<NP, PAD, 2>(srow, x0, width, w);
    // E_k = byte k | byte k+2 << 16, k = 0 .. 2NP + 1
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
        const uint32_t p0 = e[c], p1 = e[c + 1], p2 = e[c + 2], p3 = e[c + 3], p4 = e[c + 4];
        const uint32_t d = p3 - p1;                  // row_diff (pipeline.hpp:124-127)
        const uint32_t s04 = p0 + p4, s13 = p1 + p3;
        o[q].D = d;
        o[q].F = (p4 - p0 + 0x08000800u) + 2u * d;   // f = (-1,-2,0,2,1), biased
        o[q].H = s04 + 4u * s13 + 6u * p2;           // h = (1,4,6,4,1)
        o[q].K0 = 3u * (s04 + s13) + p2;             // -k0/2 = (3,3,1,3,3)
        o[q].K1 = s04 + 6u * s13 + 8u * p2;          // -k1/2 = (1,6,8,6,1)
    }
}

// Rows 0..3 of a band: fill the ring, open Q.
template <int S, int NP>
__device__ __forceinline__ void u8_prime(const U8Row (&h)[NP], uint32_t (&F)[5][NP],
                                         uint32_t (&D)[5][NP], uint32_t (&H)[5][NP],
                                         uint32_t (&aq)[5][NP]) {
#pragma unroll
    for (int j = 0; j < NP; ++j) {
        F[S][j] = h[j].F;
        D[S][j] = h[j].D;
        H[S][j] = h[j].H;
        if (S >= 1) aq[(S + 4) % 5][j] += h[j].K1;
        if (S >= 3) aq[(S + 2) % 5][j] -= h[j].K1;
        aq[S][j] = h[j].K0;
    }
}

// One input row i >= 4 (ring slot S = i mod 5, static): the Q accumulators
// and output row i - 4 as 2NP u8 pixels (byte 0 of each u[k]).
// Exact S of a packed pair whose halves carry the bias 0x8000: XOR turns the
// halves into two's complement, then sign extension / arithmetic shift.
__device__ __forceinline__ void pair_ints(uint32_t vb, int32_t& lo, int32_t& hi) {
    const uint32_t v = vb ^ 0x80008000u;
    lo = static_cast<int32_t>(static_cast<int16_t>(v & 0xffffu));
    hi = static_cast<int32_t>(v) >> 16;
}

// One input row i >= 4 (ring slot S = i mod 5, static): the Q accumulators
// and output row i - 4.  MODE 0: 2NP clamp_abs u8 pixels (byte 0 of each
// u[k]); MODE 1: the exact integer S = gx^2 + gy^2 + gd^2 + gdt^2 of each
// pixel in u[k] (normalize pass 1, image_io.hpp:242-255: the S plane and the
// frame's min / max).
template <int S, int NP, int MODE = 0>
__device__ __forceinline__ void u8_step(const U8Row (&h)[NP], uint32_t (&F)[5][NP],
                                        uint32_t (&D)[5][NP], uint32_t (&H)[5][NP],
                                        uint32_t (&aq)[5][NP], uint32_t (&u)[2 * NP]) {
    constexpr uint32_t kB = 0x80008000u;
    constexpr int s = S, s0 = (S + 1) % 5, s1 = (S + 2) % 5, s2 = (S + 3) % 5, s3 = (S + 4) % 5;
#pragma unroll
    for (int j = 0; j < NP; ++j) {
        F[s][j] = h[j].F;
        D[s][j] = h[j].D;
        H[s][j] = h[j].H;
        // Q(v) = K0'(v) + K1'(v+1) - K1'(v+3) - K0'(v+4) (Eq. 14/15): close
        // output row v = i - 4 (slot s0), bias folded in; open row i
        const uint32_t q = aq[s0][j] - h[j].K0 + kB;
        aq[s3][j] += h[j].K1;
        aq[s1][j] -= h[j].K1;
        aq[s][j] = h[j].K0;
        // output row v: input rows v..v+4 are slots s0, s1, s2, s3, s
        const uint32_t t = F[s0][j] + F[s][j], w = F[s1][j] + F[s3][j];
        const uint32_t gx = (t + 4u * w) + 6u * F[s2][j];  // bias 0x80008000
        const uint32_t n = 3u * (t + w) + F[s2][j] - 5u * (D[s0][j] + D[s][j]) +
                           6u * D[s2][j];                   // bias 0x68006800
        const uint32_t gy = (H[s][j] - H[s0][j] + kB) + 2u * (H[s3][j] - H[s1][j]);
        const int c = j < 2 ? j : j + 2;  // pair j = pixels (c, c + 2)
        if constexpr (MODE == 1) {
            // gd = N - Q and gdt = -N - Q with the bias 0x8000 per half:
            // n - q carries 0x6800 - 0x8000 per half, -n - q carries -0xE800
            const uint32_t gd = n - q + 0x98009800u, gdt = 0x68016800u - n - q;
            int32_t a0, a1, b0, b1, c0, c1, d0, d1;
            pair_ints(gx, a0, a1);
            pair_ints(gy, b0, b1);
            pair_ints(gd, c0, c1);
            pair_ints(gdt, d0, d1);
            u[c] = static_cast<uint32_t>(a0 * a0 + b0 * b0 + c0 * c0 + d0 * d0);
            u[c + 2] = static_cast<uint32_t>(a1 * a1 + b1 * b1 + c1 * c1 + d1 * d1);
        } else {
            const float2 fx = u8_pair_float<0x8000u>(gx);
            const float2 fy = u8_pair_float<0x8000u>(gy);
            const float2 fn = u8_pair_float<0x6800u>(n);
            const float2 fq = u8_pair_float<0x8000u>(q);
            // S = gx^2 + gy^2 + 2 (N^2 + Q^2): every partial sum is an exact
            // integer while the true sum is <= 65280; above it the rounded
            // partial sums are monotone, so the result is >= 65281 -- all
            // clamp_abs needs (saturation at 255)
            const float2 a = __ffma2_rn(fy, fy, __fmul2_rn(fx, fx));
            const float2 b = __ffma2_rn(fq, fq, __fmul2_rn(fn, fn));
            const float2 Sq = __ffma2_rn(b, make_float2(2.0f, 2.0f), a);
            u8_round_sqrt2(Sq, u[c], u[c + 2]);
        }
    }
}

// 2NP u8 pixels (byte 0 of each u[k]) to the output row.
template <int NP>
__device__ __forceinline__ void u8_store(uint8_t* out, const uint32_t (&u)[2 * NP], bool full,
                                         int x0, int out_w) {
    if (full) {
        const uint32_t lo = __byte_perm(__byte_perm(u[0], u[1], 0x0040),
                                        __byte_perm(u[2], u[3], 0x0040), 0x5410);
        if constexpr (NP == 4) {
            const uint32_t hi = __byte_perm(__byte_perm(u[4], u[5], 0x0040),
                                            __byte_perm(u[6], u[7], 0x0040), 0x5410);
            asm volatile("st.global.cs.v2.u32 [%0], {%1, %2};" ::"l"(out), "r"(lo), "r"(hi)
                         : "memory");
        } else {
            asm volatile("st.global.cs.u32 [%0], %1;" ::"l"(out), "r"(lo) : "memory");
        }
    } else {
#pragma unroll
        for (int i = 0; i < 2 * NP; ++i)
            if (x0 + i < out_w) out[i] = static_cast<uint8_t>(u[i] & 0xffu);
    }
}

#ifndef SOBEL5_U8_WARPS_PER_SM
#define SOBEL5_U8_WARPS_PER_SM 16  // NP = 4: 128 registers; 20 / 24 spill (88 / 152 B) and were slower
#endif
template <int NP, int W>
struct U8Bounds {  // resident CTAs per SM the register budget is set for
    static constexpr int kMinBlocks = (NP == 4 ? SOBEL5_U8_WARPS_PER_SM : 24) / W;
};

// 2NP exact S values (u[k] = pixel x0 + k) to the S plane row (MODE 1).
template <int NP>
__device__ __forceinline__ void s32_store(uint32_t* out, const uint32_t (&u)[2 * NP], bool full,
                                          int x0, int out_w) {
    if (full) {
#pragma unroll
        for (int i = 0; i < 2 * NP; i += 4)
            *reinterpret_cast<uint4*>(out + i) = make_uint4(u[i], u[i + 1], u[i + 2], u[i + 3]);
    } else {
#pragma unroll
        for (int i = 0; i < 2 * NP; ++i)
            if (x0 + i < out_w) out[i] = u[i];
    }
}

// One band of one lane from shared memory: rows 0..4 wait on bar[0], row 5
// on bar[1] (phase `par`), output rows oy0 .. oy0 + n_out - 1 at `o0`.
// MODE 0: the clamp_abs u8 plane; MODE 1: the exact S plane (p.s32) and the
// frame's min / max of g (p.minmax; normalize pass 1).  (Two copies of the
// loop, whole lanes and right-edge lanes, drop the per-row branch but ran
// 17-42% slower: profiles/r2/u8_split.txt.)
template <int NP, bool PAD, int W, int MODE>
__device__ __forceinline__ void u8_band_rows(const KernelParams& p, const uint8_t* srow,
                                             uint64_t* s_bar, uint32_t par, int x0, int64_t o0,
                                             int n_out, uint32_t& s_min, uint32_t& s_max) {
    using T = U8Band<NP, PAD, W>;
    const bool full = x0 + U8Geom<NP, W>::kLaneCols <= p.out_w;  // all 2NP columns inside
    const int n_in = n_out + 4;
    uint8_t* out = MODE == 0 ? p.u8 + o0 : nullptr;
    uint32_t* outs = MODE == 1 ? p.s32 + o0 : nullptr;

    // ring [slot = input row mod 5][pair]; Q accumulators [slot = output row mod 5]
    uint32_t F[5][NP], D[5][NP], H[5][NP], aq[5][NP];
    mbar_wait(&s_bar[0], par);
    {
        U8Row h[NP];
        u8_row<NP, PAD>(srow, x0, p.width, h);
        u8_prime<0>(h, F, D, H, aq);
        u8_row<NP, PAD>(srow + T::kRowBytes, x0, p.width, h);
        u8_prime<1>(h, F, D, H, aq);
        u8_row<NP, PAD>(srow + 2 * T::kRowBytes, x0, p.width, h);
        u8_prime<2>(h, F, D, H, aq);
        u8_row<NP, PAD>(srow + 3 * T::kRowBytes, x0, p.width, h);
        u8_prime<3>(h, F, D, H, aq);
    }
    // rows 4..n_in-1, each closing output row r - 4; slot of row r = r mod 5
    for (int base = 4; base < n_in; base += 5) {
#pragma unroll
        for (int k = 0; k < 5; ++k) {
            const int r = base + k;
            if (r >= n_in) break;
            if (r == 5) mbar_wait(&s_bar[1], par);
            U8Row h[NP];
            u8_row<NP, PAD>(srow + r * T::kRowBytes, x0, p.width, h);
            uint32_t u[2 * NP];
            switch (k) {
                case 0: u8_step<4, NP, MODE>(h, F, D, H, aq, u); break;
                case 1: u8_step<0, NP, MODE>(h, F, D, H, aq, u); break;
                case 2: u8_step<1, NP, MODE>(h, F, D, H, aq, u); break;
                case 3: u8_step<2, NP, MODE>(h, F, D, H, aq, u); break;
                default: u8_step<3, NP, MODE>(h, F, D, H, aq, u); break;
            }
            if constexpr (MODE == 1) {
                s32_store<NP>(outs, u, full, x0, p.out_w);
                outs += p.pitch;
#pragma unroll
                for (int i = 0; i < 2 * NP; ++i) {
                    if (full || x0 + i < p.out_w) {
                        s_min = min(s_min, u[i]);
                        s_max = max(s_max, u[i]);
                    }
                }
            } else {
                u8_store<NP>(out, u, full, x0, p.out_w);
                out += p.pitch;
            }
        }
    }
}

template <int NP, bool PAD, int W, int MODE = 0>
__device__ __forceinline__ void u8_band_compute(const KernelParams& p, const uint8_t* s_band,
                                                uint64_t* s_bar, uint32_t par, int tx, int oy0,
                                                int frame, int n_out) {
    constexpr int kLaneCols = U8Geom<NP, W>::kLaneCols;
    const int x0 = tx * U8Geom<NP, W>::kCtaCols + threadIdx.x * kLaneCols;
    if ((x0 & ~(kLaneCols * 32 - 1)) >= p.out_w) return;  // whole warp right of the image
    const uint8_t* srow = s_band + U8Band<NP, PAD, W>::kLead + threadIdx.x * kLaneCols;
    const int64_t o0 = static_cast<int64_t>(frame) * p.out_frame_stride +
                       static_cast<int64_t>(oy0) * p.pitch + x0;
    uint32_t s_min = 0xffffffffu, s_max = 0u;
    u8_band_rows<NP, PAD, W, MODE>(p, srow, s_bar, par, x0, o0, n_out, s_min, s_max);
    if constexpr (MODE == 1) {  // the frame's min / max of g = sqrt(S), monotone in S
        s_min = __reduce_min_sync(0xffffffffu, s_min);
        s_max = __reduce_max_sync(0xffffffffu, s_max);
        if ((threadIdx.x & 31) == 0 && s_min <= s_max) {
            sobel5_minmax* mm = p.minmax + frame;
            atomicMin(reinterpret_cast<unsigned long long*>(&mm->lo_key), dkey(sqrt_u30(s_min)));
            atomicMax(reinterpret_cast<unsigned long long*>(&mm->hi_key), dkey(sqrt_u30(s_max)));
        }
    }
}

// The kernel: grid = (column tiles of W * 32 * 2NP, bands, frames).
template <int NP, bool PAD, int W, int MODE = 0>
__global__ void __launch_bounds__(U8Geom<NP, W>::kThreads, U8Bounds<NP, W>::kMinBlocks)
    sobel5_u8_kernel(const __grid_constant__ KernelParams p) {
    pdl_enter();
    __shared__ __align__(128) uint8_t s_band[U8Band<NP, PAD, W>::kBytes];
    __shared__ __align__(8) uint64_t s_bar[2];
    const int oy0 = blockIdx.y * p.band;
    const int n_out = min(p.band, p.out_h - oy0);
    u8_band_issue<NP, PAD, W>(p, s_band, s_bar, n_out + 4);
    u8_band_compute<NP, PAD, W, MODE>(p, s_band, s_bar, 0u, blockIdx.x, oy0, blockIdx.z, n_out);
}

}  // namespace sobel5_b200
