// sobel5_packed.cuh -- two-pixels-per-register variant of the fused kernel.
//
// Every stage of the operator is linear with integer coefficients, so two
// pixels can share one 32-bit register as V = lo + hi * 2^16 (lo, hi signed):
// IADD / IMAD-by-constant / LEA on V act on both lanes at once, and 32-bit
// wrap-around is harmless because arithmetic mod 2^32 is a ring
// homomorphism.  The lanes are recovered exactly at the end,
//     lo = sext16(V),   hi = (V + 0x8000) >> 16 (arithmetic),
// provided every EXTRACTED quantity lies in [-2^15, 2^15).  The host proves
// that bound from the taps before selecting this kernel (taps_fit_packed in
// sobel5_abi.cu); for the default (1, 2, 6, 4) taps the extracted maxima are
// |gx|, |gy|, |gd|, |gdt| <= 12240 and |P|/2 <= 8925.
//
// Lane pairing: a lane owns output columns x0..x0+3 and packs pixel pairs
// (x0, x0+2) and (x0+1, x0+3); the 5-tap window of pair A is E0..E4 and of
// pair B E1..E5 with E_k = byte_k | byte_{k+2} << 16 of the 8-byte window.
//
// Default-taps algebra (make_stream_taps for (1,2,6,4), pipeline.hpp:82-92),
// with s04 = p0+p4, s13 = p1+p3, D = p3-p1 (row_diff), d04 = p4-p0:
//   F   = d04 + 2 D                      (Eq. 6, b = 2)
//   H   = s04 + 4 s13 + 6 p2             (h = 1,4,6,4,1)
//   K0  = -2 K0',  K0' = 3 (s04 + s13) + p2
//   K1  = -2 K1',  K1' = s04 + 6 s13 + 8 p2
//   gx  = F(v) + 4F(v+1) + 6F(v+2) + 4F(v+3) + F(v+4)          (Eq. 7)
//   gy  = -H(v) - 2H(v+1) + 2H(v+3) + H(v+4)
//   P   = -2 Q,  Q = K0'(v) + K1'(v+1) - K1'(v+3) - K0'(v+4)  (Eq. 14/15)
//   M   =  2 N,  N = 3F(v)+3F(v+1)+F(v+2)+3F(v+3)+3F(v+4)
//                    - 5D(v) + 6D(v+2) - 5D(v+4)              (Eq. 19/21)
//   gd  = (P+M)/2 = N - Q,   gdt = (P-M)/2 = -N - Q           (Eq. 11)
// P+M = 2(N-Q) is even by construction, so recover_diag's ParityViolation
// (pipeline.hpp:268-273) cannot fire and needs no per-pixel check.
#pragma once

#include <cstdint>

#include "sobel5_stream.cuh"

namespace sobel5_b200 {

// Output-set bits (template OUTS); kOutRuntime checks the plane pointers.
enum : int {
    kOutGx = 1, kOutGy = 2, kOutGd = 4, kOutGdt = 8, kOutG = 16, kOutG32 = 32, kOutU8 = 64,
    kOutMinMax = 128, kOutNorm = 256, kOutS32 = 512,
    // gx, gy, gd, gdt written as int16 (the host path's narrow D2H wire:
    // every packed-kernel gradient lies in [-2^15, 2^15), sobel5_ctx.cu
    // widens them into the caller's int32 planes)
    kOutN16 = 1024,
    kOutSR = 31, kOutRuntime = -1
};

// Output-set bits of a launch (selects the compile-time instantiation).
inline int packed_out_set(const KernelParams& kp) {
    return (kp.gx ? kOutGx : 0) | (kp.gy ? kOutGy : 0) | (kp.gd ? kOutGd : 0) |
           (kp.gdt ? kOutGdt : 0) | (kp.g ? kOutG : 0) | (kp.g32 ? kOutG32 : 0) |
           (kp.u8 ? kOutU8 : 0) | (kp.minmax ? kOutMinMax : 0) |
           (kp.u8 && kp.u8_norm ? kOutNorm : 0) | (kp.s32 ? kOutS32 : 0) | (kp.n16 ? kOutN16 : 0);
}

// Double magnitude of an exact integer sum of squares S < 2^32: IEEE sqrt
// (__dsqrt_rn), bit-identical to std::sqrt((double)S).  A float-seeded
// two-step Newton variant was measured 2% faster at 8K but is not correctly
// rounded for every S (it broke the 1920x1080 golden hash), so the IEEE
// routine stays.
__device__ __forceinline__ double sqrt_u30(uint32_t S) {
    return __dsqrt_rn(__uint2double_rn(S));
}

// clamp_abs(sqrt(S)) for an integer S, without the double: sqrt(S) is never
// within 4.9e-4 of k + 0.5 (the nearest case is S = 255*256), and the float
// estimate S * rsqrt(S) (MUFU.RSQ) is within 7e-5 of sqrt(S) below 65281
// (checked for every 32-bit S on the device by test_u8_from_s_exhaustive).
__device__ __forceinline__ float rsqrt_approx(float x) {
    float y;
    asm("rsqrt.approx.ftz.f32 %0, %1;" : "=f"(y) : "f"(x));
    return y;
}
// Branch-free: S is clamped to 65280 first (sqrt(65280) = 255.4995 -> 255),
// which is the saturation of clamp_abs for every larger S.
__device__ __forceinline__ uint32_t u8_from_s(uint32_t S) {
    const float f = __uint2float_rn(min(S, 65280u));
    const float y = f * rsqrt_approx(fmaxf(f, 1.0f));
    return static_cast<uint32_t>(__float2int_rn(y));
}

// ---- u8-only epilogue in packed FP32 (the issue-bound clamp_abs contract) --
//
// A packed register V = lo + hi * 2^16 (|lo|, |hi| < 2^15) biased by
// 0x80008000 holds lo + 2^15 and hi + 2^15 as its two unsigned halves (no
// carry crosses).  One byte permute per half splices a half under the
// exponent of 2^23 (0x4B00xxxx = 2^23 + half), so after one packed FADD2 the
// pair is {lo, hi} as exact floats: 1.5 instructions per value instead of the
// integer extraction's 1.5 plus 1 IMAD per square.
constexpr uint32_t kPairBias = 0x80008000u;
__device__ __forceinline__ float2 pair_to_float2(uint32_t w_biased) {
    const float lo = __uint_as_float(__byte_perm(w_biased, 0x4B000000u, 0x7610));
    const float hi = __uint_as_float(__byte_perm(w_biased, 0x4B000000u, 0x7632));
    return __fadd2_rn(make_float2(lo, hi), make_float2(-8421376.0f, -8421376.0f));  // 2^23 + 2^15
}
// Sum of four squares with packed FMAs.  Exact whenever the true sum is
// <= 65280 (every partial sum is then an integer below 2^24); when the true
// sum is >= 65281 the rounded partial sums are non-decreasing and the first
// one above 65280 rounds to >= 65281 (representable), so the result is
// >= 65281 -- exactly what clamp_abs needs (saturation at 255).
__device__ __forceinline__ float2 sumsq4(float2 a, float2 b, float2 c, float2 d) {
    return __ffma2_rn(d, d, __ffma2_rn(c, c, __ffma2_rn(b, b, __fmul2_rn(a, a))));
}
// clamp_abs of sqrt(S) for the float S above: S * rsqrt(S) (MUFU.RSQ) is
// within 7e-5 of sqrt(S), sqrt(S) is never within 4.9e-4 of k + 0.5 for
// integer S <= 65280, and cvt.rni.sat.u8 rounds and saturates in one
// instruction (S >= 65281 -> >= 255.5 -> 255).  S = 0 gives 0 * inf = NaN,
// which the conversion maps to 0.  Checked for every integer S <= 65280 and
// every float S >= 65281 by sobel5_selftest(2 / 3).
__device__ __forceinline__ uint32_t u8_from_sf(float y_times_rsqrt) {
    uint32_t r;
    asm("cvt.rni.sat.u8.f32 %0, %1;" : "=r"(r) : "f"(y_times_rsqrt));
    return r;
}
__device__ __forceinline__ void u8_from_sf2(float2 S, uint32_t& a, uint32_t& b) {
    float ra, rb;
    asm("rsqrt.approx.ftz.f32 %0, %1;" : "=f"(ra) : "f"(S.x));
    asm("rsqrt.approx.ftz.f32 %0, %1;" : "=f"(rb) : "f"(S.y));
    const float2 y = __fmul2_rn(S, make_float2(ra, rb));
    a = u8_from_sf(y.x);
    b = u8_from_sf(y.y);
}

// ---- TMA bulk loads (cp.async.bulk shared <- global, mbarrier completion) --
__device__ __forceinline__ uint32_t smem_addr(const void* p) {
    return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}
__device__ __forceinline__ void mbar_init(uint64_t* bar, uint32_t count) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_addr(bar)), "r"(count) : "memory");
}
__device__ __forceinline__ void mbar_expect_tx(uint64_t* bar, uint32_t bytes) {
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_addr(bar)),
                 "r"(bytes)
                 : "memory");
}
__device__ __forceinline__ void mbar_wait(uint64_t* bar, uint32_t parity) {
    asm volatile(
        "{\n .reg .pred p;\n"
        "W: mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n"
        " @!p bra W;\n}" ::"r"(smem_addr(bar)),
        "r"(parity)
        : "memory");
}
__device__ __forceinline__ void bulk_load(void* sdst, const void* gsrc, uint32_t bytes, uint64_t* bar) {
    asm volatile(
        "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
            smem_addr(sdst)),
        "l"(gsrc), "r"(bytes), "r"(smem_addr(bar))
        : "memory");
}

// ---- TMA band rows shared by the packed kernels ---------------------------
// The CTA's band (n_in rows x its 512 + 16 columns) is bulk-copied into
// shared memory at CTA start, rows 0..4 and 5..n_in-1 on two mbarriers; the
// kernels read each row from shared memory when it is consumed (band <= 32).
// Row layout: PAD keeps 16 bytes left of the CTA's first column (lane 0's
// left word) at offset 0, so a row holds columns [x0 - 16, x0 + 528).
template <bool PAD>
struct TmaBand {
    static constexpr int kLead = PAD ? 16 : 0;
    static constexpr int kRowBytes = kCtaCols + 16 + kLead;
    static constexpr int kRows = 36;
    static constexpr int kBytes = kRows * kRowBytes;
};

// Block-wide: initialise the two mbarriers, then warp 0 issues one bulk copy
// per band row (lanes stride over the rows).  Every thread of the CTA must
// call it (it contains a __syncthreads).  SEG (stacked [top; mid; bot]):
// only CTAs whose rows all lie in `mid` use TMA -- the halo rows (possibly a
// peer GPU's memory) are never bulk-copied; the return value says whether
// this CTA's band is in shared memory (block-uniform).
template <bool PAD, bool SEG = false>
__device__ __forceinline__ bool tma_band_issue(const KernelParams& p, uint8_t* s_band,
                                               uint64_t* s_bar) {
    using T = TmaBand<PAD>;
    const int b_oy0 = blockIdx.y * p.band;
    const int b_in = min(p.band, p.out_h - b_oy0) + 4;
    if (SEG && (b_oy0 < p.top_rows || b_oy0 + b_in > p.top_rows + p.mid_rows)) return false;
    if (threadIdx.x == 0) {
        mbar_init(&s_bar[0], 1);
        mbar_init(&s_bar[1], 1);
        asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
    }
    __syncthreads();  // barrier init visible before anyone waits
    if (threadIdx.x < 32) {
        const int n0 = min(5, b_in);
        const int cta_x0 = blockIdx.x * kCtaCols;
        // source columns [src_x, ...): 16-B aligned, inside the row (pitch is
        // a multiple of 16 >= width); PAD starts 16 columns early except at
        // the left image edge
        const int src_x = max(cta_x0 - T::kLead, 0);
        const int dst_off = src_x - (cta_x0 - T::kLead);
        const uint32_t rb = static_cast<uint32_t>(
            min(T::kRowBytes - dst_off, ((p.width + 15) & ~15) - src_x));
        if (threadIdx.x == 0) {
            mbar_expect_tx(&s_bar[0], rb * n0);
            mbar_expect_tx(&s_bar[1], rb * (b_in - n0));
        }
        __syncwarp();
        for (int r = threadIdx.x; r < b_in; r += 32) {
            // PAD: padded row b_oy0 + r is image row clamp(b_oy0 + r - 2);
            // SEG: stacked row b_oy0 + r is mid row b_oy0 + r - top_rows
            const int y = PAD   ? min(max(b_oy0 + r - 2, 0), p.mid_rows - 1)
                          : SEG ? b_oy0 + r - p.top_rows
                                : b_oy0 + r;
            bulk_load(s_band + r * T::kRowBytes + dst_off,
                      p.mid + static_cast<int64_t>(blockIdx.z) * p.in_frame_stride +
                          static_cast<int64_t>(y) * p.in_pitch + src_x,
                      rb, &s_bar[r < n0 ? 0 : 1]);
        }
    }
    return true;
}

// Row r of the band at the thread's column x0 (waits for its mbarrier when r
// is the first row of a stage).
template <bool PAD>
__device__ __forceinline__ const uint8_t* tma_band_row(uint8_t* s_band, uint64_t* s_bar, int r,
                                                       int x0) {
    if (r == 0) mbar_wait(&s_bar[0], 0);
    if (r == 5) mbar_wait(&s_bar[1], 0);
    return s_band + r * TmaBand<PAD>::kRowBytes + TmaBand<PAD>::kLead +
           (x0 - static_cast<int>(blockIdx.x) * kCtaCols);
}

// ---- TMA bulk stores (cp.async.bulk global <- shared, bulk-group completion)
__device__ __forceinline__ void bulk_store(void* gdst, const void* ssrc, uint32_t bytes) {
    asm volatile("cp.async.bulk.global.shared::cta.bulk_group [%0], [%1], %2;" ::"l"(gdst),
                 "r"(static_cast<uint32_t>(__cvta_generic_to_shared(ssrc))), "r"(bytes)
                 : "memory");
}
__device__ __forceinline__ void bulk_commit() {
    asm volatile("cp.async.bulk.commit_group;" ::: "memory");
}
template <int N>
__device__ __forceinline__ void bulk_wait_read() {  // <= N groups still reading smem
    asm volatile("cp.async.bulk.wait_group.read %0;" ::"n"(N) : "memory");
}
__device__ __forceinline__ void bulk_wait_all() {
    asm volatile("cp.async.bulk.wait_group 0;" ::: "memory");
}
// generic-proxy smem writes -> visible to the async proxy (the bulk copy)
__device__ __forceinline__ void fence_async_smem() {
    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
}

// ---- TMA tensor stores of the StreamResult (kGeomPlainTmaTs) ---------------
// Each CTA stages kTsRows output rows of its 512-column tile for every plane
// in shared memory (double-buffered), then one thread writes them with six
// cp.async.bulk.tensor stores (gx, gy, gd, gdt as uint64 pairs: one 512-column
// box each; g: two 256-column boxes), coordinates from blockIdx only.
constexpr int kTsBoxCols = kCtaCols;  // 512
constexpr int kTsRows = 2;            // output rows per staged box
constexpr int kTsIntBytes = kTsRows * kTsBoxCols * 4;        // one int32 plane
constexpr int kTsGBytes = kTsRows * (kTsBoxCols / 2) * 8;    // one g half
constexpr int kTsBufBytes = 4 * kTsIntBytes + 2 * kTsGBytes;  // 24 KB
constexpr int kTsSmemBytes = 2 * kTsBufBytes;                 // dynamic shared memory
constexpr int kTsBandRows = 12;  // shared-memory input rows: bands <= 8
__device__ __forceinline__ void tma_store_3d(const CUtensorMap* tm, const void* ssrc, int x, int y,
                                             int z) {
    asm volatile(
        "cp.async.bulk.tensor.3d.global.shared::cta.bulk_group [%0, {%2, %3, %4}], [%1];" ::"l"(tm),
        "r"(smem_addr(ssrc)), "r"(x), "r"(y), "r"(z)
        : "memory");
}
__device__ __forceinline__ void named_bar_sync(int id, int n) {
    asm volatile("bar.sync %0, %1;" ::"r"(id), "r"(n) : "memory");
}

// Four bytes (each < 256) packed little-endian with two byte permutes.
__device__ __forceinline__ uint32_t pack_u8x4(uint32_t a, uint32_t b, uint32_t c, uint32_t d) {
    return __byte_perm(__byte_perm(a, b, 0x0040), __byte_perm(c, d, 0x0040), 0x5410);
}

__device__ __forceinline__ int32_t lane_lo(uint32_t v) {
    return static_cast<int32_t>(static_cast<int16_t>(v & 0xffffu));
}
__device__ __forceinline__ int32_t lane_hi(uint32_t v) {
    return static_cast<int32_t>(v + 0x8000u) >> 16;
}

// Exact normalize export of an integer sum of squares (image_io.hpp:242-255,
// pass 2): u = lround((sqrt(S) - lo) * 255 / span) is non-decreasing in S
// (each IEEE step is monotone), so it equals max{k : thr[k] <= S} for the
// thresholds built by norm_table_kernel (sobel5_detect.cu).  A float estimate
// seeds the lookup; two table probes confirm it, else an 8-step binary
// search decides, so the result is exact whatever the seed.
__device__ __forceinline__ uint32_t u8_normalize_s(uint32_t S, const uint32_t* thr, float lo_f,
                                                   float scale_f) {
    const float f = __uint2float_rn(S);
    const float est = (f * rsqrtf(fmaxf(f, 1.0f)) - lo_f) * scale_f;
    int e = min(255, max(0, __float2int_rn(est)));
    if (thr[e] <= S && S < thr[e + 1]) return static_cast<uint32_t>(e);
    // seed off by more than the table says (tiny spans): binary search
    e = 0;
#pragma unroll
    for (int step = 128; step >= 1; step >>= 1)
        if (thr[e + step] <= S) e += step;
    return static_cast<uint32_t>(e);
}

// Default taps, packed.  PF = number of input rows whose loads are in flight
// ahead of the row being processed (0 = Prefetch::off, >= 1 = on).
// GEOM = Geom (plain image / stacked row band / fused replicate padding).
// OUTS = output-set bits; kOutMinMax adds the per-frame min/max of g
// (normalize pass 1), kOutNorm makes the u8 plane the normalize export
// (pass 2) instead of clamp_abs.
#ifndef SOBEL5_U8_MIN_CTAS
#define SOBEL5_U8_MIN_CTAS kMinCtasPerSm
#endif
#ifndef SOBEL5_TMA_MIN_CTAS
#define SOBEL5_TMA_MIN_CTAS kMinCtasPerSm
#endif
template <int PF, int GEOM, int OUTS, bool RTAPS = false>
__global__ void __launch_bounds__(kCtaThreads,
                                  (OUTS == kOutU8 && !RTAPS) ? SOBEL5_U8_MIN_CTAS
                                  : (GEOM == kGeomPlainTma || GEOM == kGeomPadTma ||
                                     GEOM == kGeomSegTma || GEOM == kGeomPlainTmaTs ||
                                     GEOM == kGeomPlainTmaTw)
                                      ? SOBEL5_TMA_MIN_CTAS
                                      : kMinCtasPerSm)
    sobel5_packed_default_kernel(const __grid_constant__ KernelParams p) {
    pdl_enter();
    __shared__ OddSlot s_odd[RTAPS ? kCtaThreads : 1];  // ParityViolation (runtime taps)
    if constexpr (RTAPS) {
        if (p.diag) odd_init(s_odd);
    }
    constexpr bool SEG = GEOM == kGeomSeg || GEOM == kGeomSegTma;
    constexpr bool PAD = GEOM == kGeomPad || GEOM == kGeomPadTma;
    // TMAL: band rows by TMA into shared memory (tma_band_issue); the
    // launchers instantiate it with PF = 0, so each row is read from shared
    // memory when it is consumed
    // TS: the StreamResult leaves through TMA tensor stores (shared-memory
    // staging, sobel5_tmap.cu builds the maps)
    constexpr bool TS = GEOM == kGeomPlainTmaTs || GEOM == kGeomPlainTmaTw;
    constexpr bool TW = GEOM == kGeomPlainTmaTw;  // per-warp boxes, no CTA barrier
    static_assert(!TS || OUTS == kOutSR, "tensor stores: StreamResult only");
    constexpr bool TMAL = GEOM == kGeomPlainTma || GEOM == kGeomPadTma || GEOM == kGeomSegTma || TS;
    __shared__ __align__(128)
        uint8_t s_band[TS ? kTsBandRows * TmaBand<false>::kRowBytes : TMAL ? TmaBand<PAD>::kBytes : 16];
    extern __shared__ __align__(128) uint8_t s_dyn[];  // TS staging (kTsSmemBytes)
    __shared__ __align__(8) uint64_t s_bar[2];
    // StreamResult on the TMA-row kernel: write-back stores instead of .cs
#ifndef SOBEL5_SR_WB
#define SOBEL5_SR_WB 1
#endif
    constexpr bool WB = (SOBEL5_SR_WB == 2 || (SOBEL5_SR_WB == 1 && TMAL)) && OUTS == kOutSR && !TS;
    // which planes this instantiation writes (compile-time unless kOutRuntime)
    constexpr bool RT = OUTS == kOutRuntime;
    const bool w_gx = RT ? p.gx != nullptr : (OUTS & kOutGx) != 0;
    const bool w_gy = RT ? p.gy != nullptr : (OUTS & kOutGy) != 0;
    const bool w_gd = RT ? p.gd != nullptr : (OUTS & kOutGd) != 0;
    const bool w_gdt = RT ? p.gdt != nullptr : (OUTS & kOutGdt) != 0;
    const bool w_g = RT ? p.g != nullptr : (OUTS & kOutG) != 0;
    const bool w_g32 = RT ? p.g32 != nullptr : (OUTS & kOutG32) != 0;
    const bool w_u8 = RT ? p.u8 != nullptr : (OUTS & kOutU8) != 0;
    const bool w_mm = RT ? p.minmax != nullptr : (OUTS & kOutMinMax) != 0;
    const bool u8_norm = RT ? p.u8_norm != 0 : (OUTS & kOutNorm) != 0;
    const bool w_s = RT ? p.s32 != nullptr : (OUTS & kOutS32) != 0;
    const bool need_g = w_g || w_g32;
    constexpr bool N16 = !RT && (OUTS & kOutN16) != 0;
    static_assert(!N16 || !RTAPS, "int16 wire: default taps only");
    // the clamp_abs edge map alone: packed-float epilogue (u8_from_sf2)
    constexpr bool FU8 = !RTAPS && OUTS == kOutU8;
    const int lane = threadIdx.x & 31;
    const int warp = threadIdx.x >> 5;
    const int warp_x0 = (blockIdx.x * kCtaWarps + warp) * kWarpCols;
    const int x0 = warp_x0 + lane * 4;

    // TMA bulk stores of the wide planes (compile-time output sets only)
    // Opt-in (-DSOBEL5_TMA_STORE, best with -DSOBEL5_CTA_WARPS=1 so the bulk
    // addresses are warp-uniform): measured no faster than register stores
    // in this kernel (145 vs 144 us at 8K SR) although a store-only probe
    // gains 12% (profiles/r1/store_probes.txt), so register stores are the
    // default.
#ifdef SOBEL5_TMA_STORE
    constexpr bool TMA = !RT && (OUTS & (kOutGx | kOutGy | kOutGd | kOutGdt | kOutG | kOutG32)) != 0;
#else
    constexpr bool TMA = false;
#endif
    constexpr int kOffGx = 0;
    constexpr int kOffGy = kOffGx + ((OUTS & kOutGx) ? 512 : 0);
    constexpr int kOffGd = kOffGy + ((OUTS & kOutGy) ? 512 : 0);
    constexpr int kOffGdt = kOffGd + ((OUTS & kOutGd) ? 512 : 0);
    constexpr int kOffG = kOffGdt + ((OUTS & kOutGdt) ? 512 : 0);
    constexpr int kOffG32 = kOffG + ((OUTS & kOutG) ? 1024 : 0);
    constexpr int kStageBytes = kOffG32 + ((OUTS & kOutG32) ? 512 : 0);
#ifndef SOBEL5_STAGE_BUFS
#define SOBEL5_STAGE_BUFS 3
#endif
    constexpr int kBufs = SOBEL5_STAGE_BUFS;  // rows of staging per warp in flight
    __shared__ __align__(128) unsigned char s_stage[TMA ? kCtaWarps * kBufs * kStageBytes : 16];
    int stage_row = 0;

    // normalize pass 2: the frame's threshold table, staged in shared memory
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
    bool cta_tma = false;  // SEG: CTAs touching a halo row load from global
    if constexpr (TMAL) cta_tma = tma_band_issue<PAD, SEG>(p, s_band, s_bar);
    // whole warp right of the image (TS: it still joins the staging barriers;
    // its columns are clipped by the tensor stores)
    if ((!TS || TW) && warp_x0 >= p.out_w) return;
    const int oy0 = blockIdx.y * p.band;
    const int n_out = min(p.band, p.out_h - oy0);
    const int n_in = n_out + 4;
    const int64_t in_frame = static_cast<int64_t>(blockIdx.z) * p.in_frame_stride;
    const int64_t out_frame = static_cast<int64_t>(blockIdx.z) * p.out_frame_stride;
    const bool load_a = x0 < p.width;
    // the one extra word: lane 31's right neighbour; in pad mode lane 0's left
    const int xoff = (PAD && lane == 0) ? -4 : 4;
    // Column sharing (the paper's idea 1).  Ablation builds only
    // (-DSOBEL5_COLSHARE, plain geometry): 0 = warp shuffle (default),
    // 1 = every lane loads its right neighbour word itself (redundant global
    // loads, L1 hits), 2 = each warp stages its row words in shared memory.
#ifndef SOBEL5_COLSHARE
#define SOBEL5_COLSHARE 0
#endif
    constexpr int CS = PAD ? 0 : SOBEL5_COLSHARE;
    const bool load_b = CS == 1 ? (x0 + 4 < p.width)
                                : (lane == 31 && x0 + 4 < p.width) || (PAD && lane == 0 && x0 > 0);
    const bool full = x0 + 3 < p.out_w;
    const bool warp_full = warp_x0 + kWarpCols <= p.out_w;  // warp-uniform
    const PadEdge pe = PAD ? pad_edge_setup(p.width, warp_x0) : PadEdge{0, 0, 0, 0u};
    __shared__ uint32_t s_cols[CS == 2 ? kCtaWarps * 2 * 33 : 1];
    int cs_buf = 0;
    auto window = [&](uint32_t own, uint32_t xtra, uint32_t& wa, uint32_t& wb) {
        if constexpr (CS == 0) {
            row_window<PAD>(own, xtra, lane, x0, p.width, pe, wa, wb);
        } else if constexpr (CS == 1) {
            wa = own;
            wb = xtra;
        } else {  // double-buffered per warp; the next call's syncwarp orders reuse
            uint32_t* row = s_cols + (warp * 2 + cs_buf) * 33;
            row[lane] = own;
            if (lane == 31) row[32] = xtra;
            __syncwarp();
            wa = own;
            wb = row[lane + 1];
            cs_buf ^= 1;
        }
    };

    // Plain images: rows are loaded strictly in order, so one running
    // pointer advanced by the pitch replaces the 64-bit address arithmetic
    // per row (it is never dereferenced past the band's last row).
    const uint8_t* plain = p.mid + in_frame + static_cast<int64_t>(oy0) * p.in_pitch + x0;
    auto row_ptr = [&](int r) -> const uint8_t* {
        if (SEG) return stacked_row(p, in_frame, oy0 + r) + x0;
        // PAD: padded row oy0 + r is image row clamp(oy0 + r - 2, 0, H - 1)
        const int y = min(max(oy0 + r - 2, 0), p.mid_rows - 1);
        return p.mid + in_frame + static_cast<int64_t>(y) * p.in_pitch + x0;
    };
    auto load_row = [&](int r, uint32_t& a, uint32_t& b) {
        if constexpr (TMAL) {
            if (!SEG || cta_tma) {
                const uint8_t* sr = tma_band_row<PAD>(s_band, s_bar, r, x0);
                a = load_a ? *reinterpret_cast<const uint32_t*>(sr) : 0u;
                b = load_b ? *reinterpret_cast<const uint32_t*>(sr + xoff) : 0u;
                return;
            }
        }
        const uint8_t* rp;
        if (!SEG && !PAD) {
            rp = plain;
            plain += p.in_pitch;
        } else {
            rp = row_ptr(r);
        }
        a = load_a ? ld_row_word(rp) : 0u;
        b = load_b ? ld_row_word(rp + xoff) : 0u;
    };
    // element offset of the next output row (running, one pitch per row)
    int64_t out_off = out_frame + static_cast<int64_t>(oy0) * p.pitch + x0;

    // pending accumulators [slot = output row mod 5][pair]
    uint32_t ax[5][2], ay[5][2], an[5][2], aq[5][2];
    uint32_t s_min = 0xffffffffu, s_max = 0u;

    // Prefetch ring: with PF > 0 the loads of the next 5 input rows are in
    // flight while a row is processed.  The ring slot is the unrolled row
    // index s (static), so a row's registers are consumed in place; shifting
    // a queue instead would make the register move wait on the younger load.
    uint32_t qa[5], qb[5];
    // (cur_a, cur_b): the next row's 8-byte window, already shuffled.  The
    // shuffle for row r+1 is issued while row r is computed, so its latency
    // is off the critical path (profiled: SHFL + SEL were 26% of stalls).
    uint32_t cur_a = 0u, cur_b = 0u;
    if (PF > 0) {
#pragma unroll
        for (int k = 0; k < 5; ++k) {
            if (k < n_in) load_row(k, qa[k], qb[k]);
            else qa[k] = qb[k] = 0u;
        }
        window(qa[0], qb[0], cur_a, cur_b);
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
            } else {
                uint32_t o, x;
                load_row(r, o, x);
                window(o, x, wa, wb);
            }

            // E_k = byte k | byte k+2 << 16
            const uint32_t mid = __byte_perm(wa, wb, 0x5432);  // bytes 2,3,4,5
            uint32_t e[6];
            e[0] = __byte_perm(wa, 0u, 0x4240);
            e[1] = __byte_perm(wa, 0u, 0x4341);
            e[2] = __byte_perm(mid, 0u, 0x4240);
            e[3] = __byte_perm(mid, 0u, 0x4341);
            e[4] = __byte_perm(wb, 0u, 0x4240);
            e[5] = __byte_perm(wb, 0u, 0x4341);
            // refill the ring slot only after its word has been consumed, so
            // the load can target the same registers (no move, no early wait)
            if (PF > 0) {
                if (r + 5 < n_in) load_row(r + 5, qa[s], qb[s]);
                // warp-shuffle column sharing for row r+1
                const int sn = (s + 1) % 5;
                window(qa[sn], qb[sn], cur_a, cur_b);
            }

            uint32_t F[2], H[2], D[2], K0[2], K1[2];
#pragma unroll
            for (int q = 0; q < 2; ++q) {
                const uint32_t p0 = e[q], p1 = e[q + 1], p2 = e[q + 2], p3 = e[q + 3],
                               p4 = e[q + 4];
                const uint32_t d = p3 - p1;  // row_diff (pipeline.hpp:124-127)
                D[q] = d;
                if constexpr (RTAPS) {
                    // row_conv5 (pipeline.hpp:117-122) with the caller's taps;
                    // the multiplies act on both packed pixels at once
                    const uint32_t pv[5] = {p0, p1, p2, p3, p4};
                    uint32_t f = 0u, hh = 0u, k0 = 0u, k1 = 0u;
#pragma unroll
                    for (int t = 0; t < 5; ++t) {
                        f += static_cast<uint32_t>(p.f[t]) * pv[t];
                        hh += static_cast<uint32_t>(p.h[t]) * pv[t];
                        k0 += static_cast<uint32_t>(p.k0[t]) * pv[t];
                        k1 += static_cast<uint32_t>(p.k1[t]) * pv[t];
                    }
                    F[q] = f;
                    H[q] = hh;
                    K0[q] = k0;
                    K1[q] = k1;
                } else {
                    const uint32_t s04 = p0 + p4, s13 = p1 + p3;
                    const uint32_t d04 = p4 - p0;
                    F[q] = d04 + 2u * d;
                    H[q] = s04 + 4u * s13 + 6u * p2;
                    K0[q] = 3u * (s04 + s13) + p2;
                    K1[q] = s04 + 6u * s13 + 8u * p2;
                }
            }

            if constexpr (RTAPS) {
                // vagg5 / vagg_gd_minus / vagg_gd_plus (pipeline.hpp:136-189)
                // as running sums: ax = gx, ay = gy, an = M, aq = P
#pragma unroll
                for (int q = 0; q < 2; ++q) {
                    const uint32_t f = F[q], hh = H[q], d = D[q];
#pragma unroll
                    for (int i = 0; i < 5; ++i) {
                        const int sl_i = (s - i + 5) % 5;
                        const uint32_t vx = static_cast<uint32_t>(p.gx_v[i]) * f;
                        const uint32_t vy = static_cast<uint32_t>(p.gy_v[i]) * hh;
                        const uint32_t vm = static_cast<uint32_t>(p.gdm_f[i]) * f -
                                            static_cast<uint32_t>(p.gdm_d[i]) * d;
                        if (i == 0) {
                            ax[sl_i][q] = vx;
                            ay[sl_i][q] = vy;
                            an[sl_i][q] = vm;
                            aq[sl_i][q] = K0[q];
                        } else {
                            ax[sl_i][q] += vx;
                            ay[sl_i][q] += vy;
                            an[sl_i][q] += vm;
                            if (i == 1) aq[sl_i][q] += K1[q];
                            if (i == 3) aq[sl_i][q] -= K1[q];
                            if (i == 4) aq[sl_i][q] -= K0[q];
                        }
                    }
                }
            } else {
#pragma unroll
                for (int q = 0; q < 2; ++q) {
                    const uint32_t f = F[q], hh = H[q], d = D[q];
                    const uint32_t f3 = 3u * f;
                    const uint32_t na = f3 - 5u * d;  // i = 0, 4
                    const uint32_t nc = f + 6u * d;   // i = 2
                    // i = 0: open output row r
                    const int s0 = s;
                    ax[s0][q] = f;
                    ay[s0][q] = 0u - hh;
                    an[s0][q] = na;
                    aq[s0][q] = K0[q];
                    // i = 1
                    const int s1 = (s + 4) % 5;
                    ax[s1][q] += 4u * f;
                    ay[s1][q] -= 2u * hh;
                    an[s1][q] += f3;
                    aq[s1][q] += K1[q];
                    // i = 2
                    const int s2 = (s + 3) % 5;
                    ax[s2][q] += 6u * f;
                    an[s2][q] += nc;
                    // i = 3
                    const int s3 = (s + 2) % 5;
                    ax[s3][q] += 4u * f;
                    ay[s3][q] += 2u * hh;
                    an[s3][q] += f3;
                    aq[s3][q] -= K1[q];
                    // i = 4: closes output row r - 4
                    const int s4 = (s + 1) % 5;
                    ax[s4][q] += f;
                    ay[s4][q] += hh;
                    an[s4][q] += na;
                    aq[s4][q] -= K0[q];
                }
            }

            if (FU8 && r >= 4) {
                // u8 clamp_abs only: packed-float epilogue, no lane extraction
                const int sl = (s + 1) % 5;
                const int64_t row_off = out_off;
                out_off += p.pitch;
                uint32_t u[4];
#pragma unroll
                for (int q = 0; q < 2; ++q) {  // pair q holds pixels (q, q + 2)
                    const float2 fx = pair_to_float2(ax[sl][q] + kPairBias);
                    const float2 fy = pair_to_float2(ay[sl][q] + kPairBias);
                    const float2 fd = pair_to_float2(an[sl][q] - aq[sl][q] + kPairBias);
                    const float2 ft = pair_to_float2(0u - an[sl][q] - aq[sl][q] + kPairBias);
                    u8_from_sf2(sumsq4(fx, fy, fd, ft), u[q], u[q + 2]);
                }
                if (full) {
                    st_cs_u32(p.u8 + row_off, pack_u8x4(u[0], u[1], u[2], u[3]));
                } else {
#pragma unroll
                    for (int j = 0; j < 4; ++j)
                        if (x0 + j < p.out_w) p.u8[row_off + j] = static_cast<uint8_t>(u[j]);
                }
            } else if (r >= 4) {
                const int sl = (s + 1) % 5;
                int32_t gx[4], gy[4], gd[4], gdt[4];
                if constexpr (RTAPS) {
                    // P = aq, M = an extracted per pixel; recover_diag
                    // (pipeline.hpp:268-282): gd = (P+M)/2, gdt = (P-M)/2
                    int32_t P[4], M[4];
                    bool odd_any = false;
                    int32_t odd_p = 0, odd_m = 0, odd_j = 0;
#pragma unroll
                    for (int q = 0; q < 2; ++q) {
                        gx[q] = lane_lo(ax[sl][q]);
                        gx[q + 2] = lane_hi(ax[sl][q]);
                        gy[q] = lane_lo(ay[sl][q]);
                        gy[q + 2] = lane_hi(ay[sl][q]);
                        P[q] = lane_lo(aq[sl][q]);
                        P[q + 2] = lane_hi(aq[sl][q]);
                        M[q] = lane_lo(an[sl][q]);
                        M[q + 2] = lane_hi(an[sl][q]);
                    }
#pragma unroll
                    for (int j = 0; j < 4; ++j) {
                        const int32_t sum = P[j] + M[j];
                        const bool odd = (sum & 1) != 0 && x0 + j < p.out_w;
                        if (odd && !odd_any) {  // pixels x0 + j in column order
                            odd_p = P[j];
                            odd_m = M[j];
                            odd_j = j;
                        }
                        odd_any |= odd;
                        gd[j] = sum >> 1;
                        gdt[j] = (P[j] - M[j]) >> 1;
                    }
                    // ParityViolation (pipeline.hpp:269-271): counted once per
                    // warp, the reported pair is the reference's first one
                    const unsigned odd_mask = __ballot_sync(0xffffffffu, odd_any);
                    if (odd_mask && p.diag) {
                        if (lane == __ffs(odd_mask) - 1) atomicAdd(&p.diag->violations, 1);
                        if (odd_any)
                            odd_note(s_odd, p.diag, blockIdx.z + p.diag_frame0, p.diag_row0 + oy0 + r - 4,
                                     x0 + odd_j, odd_p, odd_m);
                    }
                } else {
#pragma unroll
                    for (int q = 0; q < 2; ++q) {
                        const uint32_t vd = an[sl][q] - aq[sl][q];
                        const uint32_t vt = 0u - an[sl][q] - aq[sl][q];
                        // pair q holds pixels (q, q + 2)
                        gx[q] = lane_lo(ax[sl][q]);
                        gx[q + 2] = lane_hi(ax[sl][q]);
                        gy[q] = lane_lo(ay[sl][q]);
                        gy[q + 2] = lane_hi(ay[sl][q]);
                        gd[q] = lane_lo(vd);
                        gd[q + 2] = lane_hi(vd);
                        gdt[q] = lane_lo(vt);
                        gdt[q + 2] = lane_hi(vt);
                    }
                }
                const int64_t row_off = out_off;
                out_off += p.pitch;
                uint32_t S[4] = {0u, 0u, 0u, 0u};
                double g[4] = {0.0, 0.0, 0.0, 0.0};
                uint32_t u[4] = {0u, 0u, 0u, 0u};
                if (need_g || w_u8 || w_mm || w_s) {
                    // exact: every square < 2^28 and the sum < 2^30, so
                    // double(S) equals the reference's double sum of squares
#pragma unroll
                    for (int j = 0; j < 4; ++j)
                        S[j] = static_cast<uint32_t>(gx[j] * gx[j]) +
                               static_cast<uint32_t>(gy[j] * gy[j]) +
                               static_cast<uint32_t>(gd[j] * gd[j]) +
                               static_cast<uint32_t>(gdt[j] * gdt[j]);
                    if (w_mm) {
#pragma unroll
                        for (int j = 0; j < 4; ++j) {
                            if (full || x0 + j < p.out_w) {
                                s_min = min(s_min, S[j]);
                                s_max = max(s_max, S[j]);
                            }
                        }
                    }
                    if (need_g) {
#pragma unroll
                        for (int j = 0; j < 4; ++j) g[j] = sqrt_u30(S[j]);
                    }
                    if (w_u8) {
#pragma unroll
                        for (int j = 0; j < 4; ++j)
                            u[j] = u8_norm ? u8_normalize_s(S[j], s_thr, n_lo, n_scale)
                                           : u8_from_s(S[j]);
                    }
                }
                if constexpr (TW) {
                    // per-warp staging: [gx gy gd gdt: kTsRows x 128 int32][g: kTsRows x 128]
                    const int rv = r - 4;
                    const int k = rv % kTsRows;
                    constexpr int kI = kTsRows * kWarpCols * 4, kWarpBuf = 4 * kI + 2 * kI;
                    uint8_t* sb = s_dyn + (warp * 2 + ((rv / kTsRows) & 1)) * kWarpBuf;
                    uint8_t* si = sb + k * (kWarpCols * 4) + lane * 16;
                    *reinterpret_cast<int4*>(si) = make_int4(gx[0], gx[1], gx[2], gx[3]);
                    *reinterpret_cast<int4*>(si + kI) = make_int4(gy[0], gy[1], gy[2], gy[3]);
                    *reinterpret_cast<int4*>(si + 2 * kI) = make_int4(gd[0], gd[1], gd[2], gd[3]);
                    *reinterpret_cast<int4*>(si + 3 * kI) = make_int4(gdt[0], gdt[1], gdt[2], gdt[3]);
                    double2* sg = reinterpret_cast<double2*>(sb + 4 * kI + k * (kWarpCols * 8) + lane * 32);
                    sg[0] = make_double2(g[0], g[1]);
                    sg[1] = make_double2(g[2], g[3]);
                    if (k == kTsRows - 1 || rv == n_out - 1) {
                        fence_async_smem();
                        __syncwarp();
                        if (lane == 0) {
                            const int y = oy0 + rv - k, z = blockIdx.z;
                            tma_store_3d(&p.tmap[0], sb, warp_x0 / 2, y, z);
                            tma_store_3d(&p.tmap[1], sb + kI, warp_x0 / 2, y, z);
                            tma_store_3d(&p.tmap[2], sb + 2 * kI, warp_x0 / 2, y, z);
                            tma_store_3d(&p.tmap[3], sb + 3 * kI, warp_x0 / 2, y, z);
                            tma_store_3d(&p.tmap[4], sb + 4 * kI, warp_x0, y, z);
                            bulk_commit();
                            bulk_wait_read<1>();  // the other buffer is free for the next stage
                        }
                        __syncwarp();
                    }
                } else if constexpr (TS) {
                    // stage row rv of the band in buffer (rv / kTsRows) & 1
                    const int rv = r - 4;
                    const int k = rv % kTsRows;
                    uint8_t* sb = s_dyn + ((rv / kTsRows) & 1) * kTsBufBytes;
                    const int col = warp * kWarpCols + lane * 4;
                    uint8_t* si = sb + k * (kTsBoxCols * 4) + col * 4;
                    *reinterpret_cast<int4*>(si) = make_int4(gx[0], gx[1], gx[2], gx[3]);
                    *reinterpret_cast<int4*>(si + kTsIntBytes) = make_int4(gy[0], gy[1], gy[2], gy[3]);
                    *reinterpret_cast<int4*>(si + 2 * kTsIntBytes) = make_int4(gd[0], gd[1], gd[2], gd[3]);
                    *reinterpret_cast<int4*>(si + 3 * kTsIntBytes) =
                        make_int4(gdt[0], gdt[1], gdt[2], gdt[3]);
                    double* sg = reinterpret_cast<double*>(
                        sb + 4 * kTsIntBytes + (warp >> 1) * kTsGBytes + k * (kTsBoxCols / 2) * 8) +
                        (col & (kTsBoxCols / 2 - 1));
                    reinterpret_cast<double2*>(sg)[0] = make_double2(g[0], g[1]);
                    reinterpret_cast<double2*>(sg)[1] = make_double2(g[2], g[3]);
                    if (k == kTsRows - 1 || rv == n_out - 1) {
                        fence_async_smem();  // this thread's staging -> async proxy
                        if (threadIdx.x == 0) bulk_wait_read<0>();  // the other buffer is free
                        named_bar_sync(1, kCtaThreads);
                        if (threadIdx.x == 0) {
                            const int y = oy0 + rv - k, z = blockIdx.z;
                            const int x2 = blockIdx.x * (kTsBoxCols / 2);  // uint64 columns
                            tma_store_3d(&p.tmap[0], sb, x2, y, z);
                            tma_store_3d(&p.tmap[1], sb + kTsIntBytes, x2, y, z);
                            tma_store_3d(&p.tmap[2], sb + 2 * kTsIntBytes, x2, y, z);
                            tma_store_3d(&p.tmap[3], sb + 3 * kTsIntBytes, x2, y, z);
                            tma_store_3d(&p.tmap[4], sb + 4 * kTsIntBytes, blockIdx.x * kTsBoxCols, y, z);
                            tma_store_3d(&p.tmap[4], sb + 4 * kTsIntBytes + kTsGBytes,
                                         blockIdx.x * kTsBoxCols + kTsBoxCols / 2, y, z);
                            bulk_commit();
                        }
                    }
                } else if (TMA && warp_full) {
                    // Stage the warp's row of every wide plane in shared
                    // memory; lane 0 writes each as one bulk copy (TMA,
                    // cp.async.bulk.global.shared::cta).
                    unsigned char* st = s_stage + (warp * kBufs + stage_row % kBufs) * kStageBytes;
                    if (stage_row >= kBufs) {
                        if (lane == 0) bulk_wait_read<kBufs - 1>();
                        __syncwarp();
                    }
                    if (w_gx) reinterpret_cast<int4*>(st + kOffGx)[lane] = make_int4(gx[0], gx[1], gx[2], gx[3]);
                    if (w_gy) reinterpret_cast<int4*>(st + kOffGy)[lane] = make_int4(gy[0], gy[1], gy[2], gy[3]);
                    if (w_gd) reinterpret_cast<int4*>(st + kOffGd)[lane] = make_int4(gd[0], gd[1], gd[2], gd[3]);
                    if (w_gdt)
                        reinterpret_cast<int4*>(st + kOffGdt)[lane] = make_int4(gdt[0], gdt[1], gdt[2], gdt[3]);
                    if (w_g) {
                        reinterpret_cast<double2*>(st + kOffG)[2 * lane] = make_double2(g[0], g[1]);
                        reinterpret_cast<double2*>(st + kOffG)[2 * lane + 1] = make_double2(g[2], g[3]);
                    }
                    if (w_g32)
                        reinterpret_cast<float4*>(st + kOffG32)[lane] =
                            make_float4(__double2float_rn(g[0]), __double2float_rn(g[1]),
                                        __double2float_rn(g[2]), __double2float_rn(g[3]));
                    fence_async_smem();
                    __syncwarp();
                    if (lane == 0) {
                        // from warp-uniform values only (uniform datapath, no
                        // per-lane address to convert)
                        const int64_t wo = out_frame + static_cast<int64_t>(oy0 + r - 4) * p.pitch +
                                           warp_x0;
                        if (w_gx) bulk_store(p.gx + wo, st + kOffGx, 512);
                        if (w_gy) bulk_store(p.gy + wo, st + kOffGy, 512);
                        if (w_gd) bulk_store(p.gd + wo, st + kOffGd, 512);
                        if (w_gdt) bulk_store(p.gdt + wo, st + kOffGdt, 512);
                        if (w_g) bulk_store(p.g + wo, st + kOffG, 1024);
                        if (w_g32) bulk_store(p.g32 + wo, st + kOffG32, 512);
                        bulk_commit();
                    }
                    ++stage_row;
                } else if constexpr (N16) {
                    // int16 wire: 4 columns = 8 bytes per plane and lane
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
                    st16(p.gd, gd);
                    st16(p.gdt, gdt);
                    if (w_g) {  // (without g: the host rebuilds it from the wire)
                        if (full) {
                            st_wb_v4d(p.g + row_off, g[0], g[1], g[2], g[3]);
                        } else {
#pragma unroll
                            for (int j = 0; j < 4; ++j)
                                if (x0 + j < p.out_w) p.g[row_off + j] = g[j];
                        }
                    }
                } else if (full && WB) {
                    st_wb_v4(p.gx + row_off, gx[0], gx[1], gx[2], gx[3]);
                    st_wb_v4(p.gy + row_off, gy[0], gy[1], gy[2], gy[3]);
                    st_wb_v4(p.gd + row_off, gd[0], gd[1], gd[2], gd[3]);
                    st_wb_v4(p.gdt + row_off, gdt[0], gdt[1], gdt[2], gdt[3]);
                    st_wb_v4d(p.g + row_off, g[0], g[1], g[2], g[3]);
                } else if (full) {
                    if (w_gx) st_cs_v4(p.gx + row_off, gx[0], gx[1], gx[2], gx[3]);
                    if (w_gy) st_cs_v4(p.gy + row_off, gy[0], gy[1], gy[2], gy[3]);
                    if (w_gd) st_cs_v4(p.gd + row_off, gd[0], gd[1], gd[2], gd[3]);
                    if (w_gdt) st_cs_v4(p.gdt + row_off, gdt[0], gdt[1], gdt[2], gdt[3]);
                    if (w_g) st_cs_v4d(p.g + row_off, g[0], g[1], g[2], g[3]);
                    if (w_g32)
                        st_cs_v4f(p.g32 + row_off, __double2float_rn(g[0]), __double2float_rn(g[1]),
                                  __double2float_rn(g[2]), __double2float_rn(g[3]));
                } else {
#pragma unroll
                    for (int j = 0; j < 4; ++j) {
                        if (x0 + j < p.out_w) {
                            if (w_gx) p.gx[row_off + j] = gx[j];
                            if (w_gy) p.gy[row_off + j] = gy[j];
                            if (w_gd) p.gd[row_off + j] = gd[j];
                            if (w_gdt) p.gdt[row_off + j] = gdt[j];
                            if (w_g) p.g[row_off + j] = g[j];
                            if (w_g32) p.g32[row_off + j] = __double2float_rn(g[j]);
                        }
                    }
                }
                // narrow planes: register stores
                if (full) {
                    if (w_u8) st_cs_u32(p.u8 + row_off, pack_u8x4(u[0], u[1], u[2], u[3]));
                    if (w_s)  // kept in L2 where it fits: the normalize map reads it next
                        *reinterpret_cast<uint4*>(p.s32 + row_off) = make_uint4(S[0], S[1], S[2], S[3]);
                } else {
#pragma unroll
                    for (int j = 0; j < 4; ++j) {
                        if (x0 + j < p.out_w) {
                            if (w_u8) p.u8[row_off + j] = static_cast<uint8_t>(u[j]);
                            if (w_s) p.s32[row_off + j] = S[j];
                        }
                    }
                }
            }
        }
    }
    if (TMA && warp_full && lane == 0) bulk_wait_all();  // smem must outlive the copies
    if (TS && !TW && threadIdx.x == 0) bulk_wait_read<0>();  // staging read before the CTA exits
    if (TW && lane == 0) bulk_wait_read<0>();
    if (w_mm) {  // normalize pass 1: frame min / max of g = sqrt(S), monotone in S
        s_min = __reduce_min_sync(0xffffffffu, s_min);
        s_max = __reduce_max_sync(0xffffffffu, s_max);
        if (lane == 0 && s_min <= s_max) {
            sobel5_minmax* mm = p.minmax + blockIdx.z;
            atomicMin(reinterpret_cast<unsigned long long*>(&mm->lo_key),
                      dkey(sqrt_u30(s_min)));
            atomicMax(reinterpret_cast<unsigned long long*>(&mm->hi_key),
                      dkey(sqrt_u30(s_max)));
        }
    }
    if constexpr (RTAPS) {
        if (p.diag) odd_flush(s_odd, p.diag);
    }
}

}  // namespace sobel5_b200
